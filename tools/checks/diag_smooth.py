"""GPU smoothing step vs the oracle's lexicographic GS, level by level (diagnostic, GPU box).

python tools/checks/diag_smooth.py mx my levels
"""
import ctypes
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
import oracle  # noqa: E402
import paper_1904_06556_b200 as vts  # noqa: E402
from paper_1904_06556_b200 import _lib  # noqa: E402
from paper_1904_06556_b200.fem import ptr  # noqa: E402

mx, my, levels = (int(a) for a in sys.argv[1:4])
prob = vts.build_problem("cantilever", mx, my, levels, 0.5)
oprob = oracle.build_problem2d("cantilever", mx, my, levels, 0.5)
n, m = prob.n, prob.m
rng = np.random.default_rng(0)
u = rng.normal(0.0, 1e-2, n)
rho = rng.uniform(0.5, 2.0, m)
one = np.ones(m)
st = dict(u=u, alpha=1e-3, nu_lo=one.copy(), nu_up=one.copy(), rho=rho, mu_lo=one.copy(), mu_up=one.copy(),
          p=np.full(m, 1e-2), q_lo=one.copy(), q_up=one.copy())
dst = vts.PbmState(**{k: (v if k == "alpha" else torch.as_tensor(v, device="cuda")) for k, v in st.items()})
ops = vts.ElementOps(prob.fine)
ev = vts.eval_lagrangian(dst, ops, prob.f, vts.DensityBounds.for_problem(m, prob.volume, 0.0), vts.PenaltyBarrier())
mat, _ = vts.schur_system(ev, ops)
mg = vts.MgPreconditioner(mat, prob.transfers)
oops = oracle.ElementOps2D(oprob.fine)
oev = oracle.eval_lagrangian(oracle.PbmState(**st), oops, oprob.f, oracle.DensityBounds.for_problem(m, oprob.volume, 0.0),
                             oracle.PenaltyBarrier())
omat, _ = oracle.schur_system(oev, oops)
omg = oracle.MgPreconditioner(omat, oprob.transfers)
lib = _lib.load()
for k in range(1, levels):
    a = omg.mats[k]
    nk = a.core_dim
    r = np.random.default_rng(50 + k)
    b = r.standard_normal(nk + 1)
    for forward, zero in ((True, True), (True, False), (False, False)):
        x = np.zeros(nk + 1) if zero else r.standard_normal(nk + 1)
        x[-1] = 0.3 * r.standard_normal()
        xo = x.copy()
        omg._csr[k].sweep(xo[:-1], b[:-1] - a.border * xo[-1], 2, forward)
        xd = torch.as_tensor(x, device="cuda")
        _lib.check(lib.vts_debug_smooth(ops.handle, k, int(forward), int(zero), ptr(torch.as_tensor(b, device="cuda")),
                                        ptr(xd)), "vts_debug_smooth")
        xg = xd.cpu().numpy()
        d = np.abs(xg - xo)
        print(f"level {k} ({nk} dofs) fwd={forward} zero={zero}: max|dx|/max|x| = {d.max() / np.abs(xo).max():.2e} "
              f"at {int(d.argmax())}", flush=True)
