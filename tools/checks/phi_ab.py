"""eval_lagrangian A/B (VTS_PHI_SPLIT=1: two-kernel pass; default: fused k_phi_tile) on C3 with a
both-branch state: dumps the outputs to /tmp for a bitwise comparison and times the call.
python tools/checks/phi_ab.py LABEL"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1904_06556_b200 as vts  # noqa: E402

label = sys.argv[1]
prob = vts.build_config("C3")
st_h, _ = bench.microbench_inputs(prob.n, prob.m, seed=0)
rng = np.random.default_rng(5)
st_h["nu_lo"] = rng.uniform(0, 1e-2, prob.m)
st_h["nu_up"] = rng.uniform(0, 1e-2, prob.m)
st = vts.PbmState(**{k: (v if k == "alpha" else torch.as_tensor(v, device="cuda")) for k, v in st_h.items()})
ops = vts.ElementOps(prob.fine)
bounds = vts.DensityBounds.for_problem(prob.m, prob.volume, 0.0)
pen = vts.PenaltyBarrier()
ev = vts.eval_lagrangian(st, ops, prob.f, bounds, pen)
torch.cuda.synchronize()
out = {k: getattr(ev, k).cpu().numpy() for k in ("res_u", "res_lo", "res_up", "q", "mu_hat_lo", "mu_hat_up")}
out.update({k: getattr(ev.blocks, k).cpu().numpy() for k in ("a", "b_lo", "b_up", "rho_hat")})
out["scal"] = np.array([ev.value, ev.res_alpha, ev.tau_res])
np.savez(f"/tmp/phi_{label}.npz", **out)
for _ in range(3):
    vts.eval_lagrangian(st, ops, prob.f, bounds, pen)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    vts.eval_lagrangian(st, ops, prob.f, bounds, pen)
torch.cuda.synchronize()
print(json.dumps(dict(label=label, call_ms=(time.perf_counter() - t0) / 20 * 1e3, value=ev.value, tau=ev.tau_res)))
