"""Where a full PBM solve spends its wall time (host-side cProfile, GPU synchronous calls included).

Runs the solve `reps` times (wall time each), then once more under cProfile.
Usage: python tools/checks/profile_pbm.py [config] [reps]
"""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1904_06556_b200 as vts  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "C4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
prob = vts.build_config(key)
for i in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = vts.solve_pbm(prob)
    torch.cuda.synchronize()
    print(f"solve {i}: {time.perf_counter() - t0:.3f} s", flush=True)
pr = cProfile.Profile()
pr.enable()
rep = vts.solve_pbm(prob)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
