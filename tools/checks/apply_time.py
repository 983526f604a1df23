"""Newton-apply device time of one library build (VTS_LIB) on C3: python tools/checks/apply_time.py [label]."""
import ctypes
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1904_06556_b200 as vts  # noqa: E402
from paper_1904_06556_b200 import _lib  # noqa: E402

label = sys.argv[1] if len(sys.argv) > 1 else "lib"
lib = _lib.load()
prob = vts.build_config("C3")
st_h, _ = bench.microbench_inputs(prob.n, prob.m, seed=0)
st = vts.PbmState(**{k: (v if k == "alpha" else torch.as_tensor(v, device="cuda")) for k, v in st_h.items()})
ops = vts.ElementOps(prob.fine)
ev = vts.eval_lagrangian(st, ops, prob.f, vts.DensityBounds.for_problem(prob.m, prob.volume, 0.0), vts.PenaltyBarrier())
mat, _ = vts.schur_system(ev, ops)
mg = vts.MgPreconditioner(mat, prob.transfers)
kms = (ctypes.c_double * 6)()
best = 1e9
for _ in range(5):
    _lib.check(lib.vts_time_kernels(ops.handle, 200, kms), "vts_time_kernels")
    best = min(best, kms[0])
nbytes = bench.algorithmic_bytes(prob)["apply"]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
cold = (ctypes.c_double * 2)()
_lib.check(lib.vts_time_cold(ops.handle, 50, flush.data_ptr(), flush.numel(), cold), "vts_time_cold")
print(json.dumps(dict(label=label, apply_us=best * 1e3, GBs=nbytes / (best * 1e-3) / 1e9, cold_us=cold[0] * 1e3,
                      cold_GBs=nbytes / (cold[0] * 1e-3) / 1e9, resid_cold_us=cold[1] * 1e3)))
