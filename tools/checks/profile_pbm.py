"""Where a full PBM solve spends its wall time (host-side cProfile, GPU synchronous calls included).

Usage: python tools/checks/profile_pbm.py [config]
"""
import cProfile
import pstats
import sys

import torch

sys.path.insert(0, ".")
import paper_1904_06556_b200 as vts  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "C4"
prob = vts.build_config(key)
vts.solve_pbm(prob)  # warm (library load, tensor maps, JIT-free but first-touch)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
rep = vts.solve_pbm(prob)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(28)
