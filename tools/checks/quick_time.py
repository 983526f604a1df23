"""Quick timing of one library build (VTS_LIB) on C3: V-cycle, finest sweep, pair launches, MINRES it/s.

python tools/checks/quick_time.py [label]   -- one JSON line
"""
import ctypes
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1904_06556_b200 as vts  # noqa: E402
from paper_1904_06556_b200 import _lib  # noqa: E402
from paper_1904_06556_b200.fem import ptr  # noqa: E402

label = sys.argv[1] if len(sys.argv) > 1 else "lib"
key = sys.argv[2] if len(sys.argv) > 2 else "C3"
lib = _lib.load()
prob = vts.build_config(key)
st_h, rhs_h = bench.microbench_inputs(prob.n, prob.m, seed=0)
st = vts.PbmState(**{k: (v if k == "alpha" else torch.as_tensor(v, device="cuda")) for k, v in st_h.items()})
ops = vts.ElementOps(prob.fine)
ev = vts.eval_lagrangian(st, ops, prob.f, vts.DensityBounds.for_problem(prob.m, prob.volume, 0.0), vts.PenaltyBarrier())
mat, _ = vts.schur_system(ev, ops)
mg = vts.MgPreconditioner(mat, prob.transfers)
rhs = torch.as_tensor(rhs_h, device="cuda")
x = torch.empty(prob.n + 1, dtype=torch.float64, device="cuda")
itv, rel, conv = ctypes.c_int32(), ctypes.c_double(), ctypes.c_int32()


def minres(k):
    _lib.check(lib.vts_minres(ops.handle, ptr(rhs), ptr(x), 1e-14, k, 1e-9, 1, ctypes.byref(itv), ctypes.byref(rel),
                              ctypes.byref(conv), None), "vts_minres")
    return itv.value


kms = (ctypes.c_double * 6)()
_lib.check(lib.vts_time_kernels(ops.handle, 50, kms), "vts_time_kernels")
minres(5)
s = torch.cuda.current_stream()
best = 1e9
for _ in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    its = minres(50)
    b.record(s)
    torch.cuda.synchronize()
    best = min(best, a.elapsed_time(b) / its)
prof = (ctypes.c_double * 8)()
_lib.check(lib.vts_profile_begin(ops.handle), "p")
minres(20)
_lib.check(lib.vts_profile_end(ops.handle, prof), "p")
p = list(prof)
out = dict(label=label, key=key, minres_ms=best, its_per_s=1e3 / best, vcycle_ms=kms[1], fine_sweep_ms=kms[2],
           pair_desc_ms=p[4] / max(p[5], 1), pair_asc_ms=p[6] / max(p[7], 1), xsum=float(x.double().sum()))
print(json.dumps(out))
