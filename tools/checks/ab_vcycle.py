"""Bitwise A/B of the V-cycle output between two library configurations.

Run twice with different environment switches (e.g. VTS_NO_PAIR=1) and
compare the saved arrays: python tools/checks/ab_vcycle.py out.npy
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1904_06556_b200 as vts  # noqa: E402

out = sys.argv[1]
key = sys.argv[2] if len(sys.argv) > 2 else "C3"
prob = vts.build_config(key)
n, m = prob.n, prob.m
rng = np.random.default_rng(0)
host = dict(u=rng.normal(0.0, 1e-2, n), alpha=1e-3, nu_lo=rng.uniform(0, 1e-2, m), nu_up=rng.uniform(0, 1e-2, m),
            rho=rng.uniform(0.5, 2.0, m), mu_lo=np.ones(m), mu_up=np.ones(m), p=np.full(m, 1e-2),
            q_lo=np.ones(m), q_up=np.ones(m))
st = vts.PbmState(**{k: (v if k == "alpha" else torch.as_tensor(v, device="cuda")) for k, v in host.items()})
ops = vts.ElementOps(prob.fine)
ev = vts.eval_lagrangian(st, ops, prob.f, vts.DensityBounds.for_problem(m, prob.volume, 0.0), vts.PenaltyBarrier())
mat, rhs = vts.schur_system(ev, ops)
mg = vts.MgPreconditioner(mat, prob.transfers)
z = mg.apply(rhs).cpu().numpy()
res = vts.minres_solve(mat, rhs, vts.MinresConfig(tol=1e-10, max_iters=300), mg.apply)
np.save(out, np.concatenate([z, res.x.cpu().numpy(), [res.iterations]]))
print("saved", out, "minres its", res.iterations)
