"""Coordinate search over the overlap passes' per-level block counts (VTS_DOVL_BLOCKS /
VTS_OVL_BLOCKS, read at every V-cycle launch) on C3: MINRES iterations/s, median of
`reps` timings of 30 iterations per setting.  python tools/checks/tune_overlap.py"""
import ctypes
import itertools
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1904_06556_b200 as vts  # noqa: E402
from paper_1904_06556_b200 import _lib  # noqa: E402
from paper_1904_06556_b200.fem import ptr  # noqa: E402

lib = _lib.load()
prob = vts.build_config("C3")
st_h, rhs_h = bench.microbench_inputs(prob.n, prob.m, seed=0)
st = vts.PbmState(**{k: (v if k == "alpha" else torch.as_tensor(v, device="cuda")) for k, v in st_h.items()})
ops = vts.ElementOps(prob.fine)
ev = vts.eval_lagrangian(st, ops, prob.f, vts.DensityBounds.for_problem(prob.m, prob.volume, 0.0), vts.PenaltyBarrier())
mat, _ = vts.schur_system(ev, ops)
mg = vts.MgPreconditioner(mat, prob.transfers)
rhs = torch.as_tensor(rhs_h, device="cuda")
x = torch.empty(prob.n + 1, dtype=torch.float64, device="cuda")
itv, rel, conv = ctypes.c_int32(), ctypes.c_double(), ctypes.c_int32()


def its_per_s(reps=5, k=30):
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        _lib.check(lib.vts_minres(ops.handle, ptr(rhs), ptr(x), 1e-14, k, 1e-9, 1, ctypes.byref(itv),
                                  ctypes.byref(rel), ctypes.byref(conv), None), "vts_minres")
        e1.record()
        torch.cuda.synchronize()
        out.append(itv.value / (e0.elapsed_time(e1) * 1e-3))
    return statistics.median(out)


def setting(d, o):
    os.environ["VTS_DOVL_BLOCKS"] = ",".join(str(v) for v in d)
    os.environ["VTS_OVL_BLOCKS"] = ",".join(str(v) for v in o)
    return its_per_s()


its_per_s(2)
dov = [48, 27, 15, 9]  # descent: residual/restriction of levels 8, 7, 6, 5
ov = [16, 16, 6, 2]    # ascent: prolongation into levels 8, 7, 6, 5
best = setting(dov, ov)
print(json.dumps({"start": best, "dovl": dov, "ovl": ov}), flush=True)
grid_d = [[40, 44, 48], [18, 22, 27, 32, 36, 44], [8, 12, 15, 20, 26], [4, 6, 9, 12]]
grid_o = [[12, 16, 20], [4, 8, 12, 16], [2, 4, 6, 10], [1, 2, 4]]
for rnd in range(2):
    for which, grid in (("d", grid_d), ("o", grid_o)):
        for i, vals in enumerate(grid):
            for v in vals:
                d, o = list(dov), list(ov)
                (d if which == "d" else o)[i] = v
                r = setting(d, o)
                if r > best * 1.003:
                    best, dov, ov = r, d, o
                    print(json.dumps({"improved": r, "dovl": dov, "ovl": ov}), flush=True)
    print(json.dumps({"round": rnd, "best": best, "dovl": dov, "ovl": ov}), flush=True)
# confirm against the defaults
os.environ.pop("VTS_DOVL_BLOCKS")
os.environ.pop("VTS_OVL_BLOCKS")
dflt = its_per_s(9)
tuned = setting(dov, ov)
print(json.dumps({"final_default": dflt, "final_tuned": tuned, "dovl": dov, "ovl": ov}), flush=True)
