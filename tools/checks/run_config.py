"""Full PBM solve of a BASELINE config on the GPU: wall time, counts, optimality checks.

Usage: python tools/checks/run_config.py C5
"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1904_06556_b200 as vts  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "C4"
prob = vts.build_config(key)
print(key, "n", prob.n, "m", prob.m, "levels", len(prob.levels), flush=True)
t0 = time.perf_counter()
rep = vts.solve_pbm(prob)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
rho = rep.rho
print("wall_s", round(wall, 3), "converged", rep.converged, "outer", rep.outer_iterations, rep.totals(), flush=True)
print("compliance", repr(rep.objective), flush=True)
print("volume", float(rho.sum()), "target", prob.volume, "rho range", float(rho.min()), float(rho.max()), flush=True)
print("extras", {k: v for k, v in rep.extras.items() if k != "minres_per_newton"}, flush=True)

# where does rho exceed its upper bound (1)?  (the reference's tau_res omits res_up, pbm.py:181-186)
lvl = prob.fine
over = torch.nonzero(rho > 1.0 + 1e-3).flatten().cpu().numpy()
print("elements with rho > 1.001:", over.size, "of", prob.m, flush=True)
if over.size:
    ex = lvl.ex
    xs, ys = over % ex, over // ex
    print("  x range", int(xs.min()), int(xs.max()), " y range", int(ys.min()), int(ys.max()), flush=True)
    top = torch.topk(rho, 5)
    for v, i in zip(top.values.tolist(), top.indices.tolist()):
        print("  rho", round(v, 4), "at element", (i % ex, i // ex), flush=True)
