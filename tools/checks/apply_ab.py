"""A/B of Newton-apply kernel variants on C3 (run once per variant, env selects it):
python tools/checks/apply_ab.py LABEL OUTDIR -- times the apply cold/warm, dumps y = S x
and MINRES(20) iterates for a seeded x so that variants can be compared bitwise."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1904_06556_b200 as vts  # noqa: E402
from paper_1904_06556_b200 import _lib  # noqa: E402

label, outdir = sys.argv[1], sys.argv[2]
cfg = sys.argv[3] if len(sys.argv) > 3 else "C3"
lib = _lib.load()
prob = vts.build_config(cfg)
st_h, rhs_h = bench.microbench_inputs(prob.n, prob.m, seed=0)
st = vts.PbmState(**{k: (v if k == "alpha" else torch.as_tensor(v, device="cuda")) for k, v in st_h.items()})
ops = vts.ElementOps(prob.fine)
ev = vts.eval_lagrangian(st, ops, prob.f, vts.DensityBounds.for_problem(prob.m, prob.volume, 0.0), vts.PenaltyBarrier())
mat, _ = vts.schur_system(ev, ops)
mg = vts.MgPreconditioner(mat, prob.transfers)
x = torch.as_tensor(np.random.default_rng(1).standard_normal(prob.n + 1), device="cuda")
y = mat.matvec(x)
rhs = torch.as_tensor(rhs_h, device="cuda")
res = vts.minres_solve(mat, rhs, vts.MinresConfig(tol=1e-14, max_iters=20), mg.apply)
torch.cuda.synchronize()
np.savez(os.path.join("/tmp", f"apply_{label}.npz"), y=y.cpu().numpy(), x=res.x.cpu().numpy())
out = dict(label=label, minres_relres=res.relres)
if cfg == "C3":
    kms = (ctypes.c_double * 6)()
    best = 1e9
    for _ in range(5):
        _lib.check(lib.vts_time_kernels(ops.handle, 200, kms), "vts_time_kernels")
        best = min(best, kms[0])
    nbytes = bench.algorithmic_bytes(prob)["apply"]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    cold = (ctypes.c_double * 2)()
    _lib.check(lib.vts_time_cold(ops.handle, 50, flush.data_ptr(), flush.numel(), cold), "vts_time_cold")
    out.update(apply_us=best * 1e3, GBs=nbytes / (best * 1e-3) / 1e9, cold_us=cold[0] * 1e3,
               cold_GBs=nbytes / (cold[0] * 1e-3) / 1e9, cold1_us=cold[1] * 1e3)
print(json.dumps(out))
if cfg == "C3" and os.environ.get("VTS_FLOOR"):
    # the same byte count as one apply through a plain streaming torch kernel: the floor of this harness
    n = prob.n + 1
    a, b, d = (torch.randn(n, dtype=torch.float64, device="cuda") for _ in range(3))
    c = torch.empty_like(a)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for r in range(50):
        flush.fill_(r & 0xFF)
        e0.record(); torch.addcmul(d, a, b, out=c); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    warm = []
    for r in range(50):
        e0.record()
        for _ in range(20):
            torch.addcmul(d, a, b, out=c)
        e1.record(); e1.synchronize()
        warm.append(e0.elapsed_time(e1) / 20)
    print(json.dumps(dict(label="torch_addcmul_floor", bytes=4 * 8 * n, cold_us=1e3 * sum(ts) / len(ts),
                          warm_us=1e3 * min(warm))))
