"""Stress determinism of the device MINRES + V-cycle: solve one fixed Newton
system many times and compare every solution bit for bit.

Usage: python tools/checks/repeat_minres.py [config] [reps] [tol]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1904_06556_b200 as vts  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "C1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
tol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-8
prob = vts.build_config(key)
n, m = prob.n, prob.m
rng = np.random.default_rng(0)
host = dict(u=rng.normal(0.0, 1e-2, n), alpha=1e-3, nu_lo=rng.uniform(0, 1e-2, m), nu_up=rng.uniform(0, 1e-2, m),
            rho=rng.uniform(0.5, 2.0, m), mu_lo=np.ones(m), mu_up=np.ones(m), p=np.full(m, 1e-2),
            q_lo=np.ones(m), q_up=np.ones(m))
st = vts.PbmState(**{k: (v if k == "alpha" else torch.as_tensor(v, device="cuda")) for k, v in host.items()})
ops = vts.ElementOps(prob.fine)
bounds = vts.DensityBounds.for_problem(m, prob.volume, 0.0)
ev = vts.eval_lagrangian(st, ops, prob.f, bounds, vts.PenaltyBarrier())
mat, rhs = vts.schur_system(ev, ops)
mg = vts.MgPreconditioner(mat, prob.transfers)
cfg = vts.MinresConfig(tol=tol, max_iters=1000)
ref = vts.minres_solve(mat, rhs, cfg, mg.apply)
x0 = ref.x.cpu().numpy()
print("ref:", ref.iterations, ref.relres, flush=True)
bad = 0
t0 = time.time()
for r in range(reps):
    try:
        res = vts.minres_solve(mat, rhs, cfg, mg.apply)
        x = res.x.cpu().numpy()
        if res.iterations != ref.iterations or not np.array_equal(x, x0):
            bad += 1
            print(f"rep {r}: DIFFERENT its {res.iterations} max|dx| {np.abs(x - x0).max():.3e}", flush=True)
    except Exception as e:
        bad += 1
        print(f"rep {r}: ERROR {e}", flush=True)
print(f"{bad} of {reps} solves differ ({time.time() - t0:.1f} s)", flush=True)
