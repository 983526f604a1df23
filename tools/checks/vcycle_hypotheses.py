"""Which arithmetic choice separates the GPU V-cycle from the reference's? (diagnostic, CPU)

Re-implements the reference V-cycle (multigrid.py:109-154) on the oracle's
matrices with switchable variants and compares each against a GPU V-cycle
output saved by `tools/checks/diag_vcycle_levels.py --small --save`:

    python tools/checks/vcycle_hypotheses.py gpurun_out/vc_gpu_4x2_L4_0.npy 4 2 4
"""

from __future__ import annotations

import os
import sys

import numpy as np
import scipy.linalg as sla

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
import oracle  # noqa: E402


def gs(a, x, b, forward, recip=False, split=False):
    """Lexicographic GS on CSR a (multigrid.py:35-64) with arithmetic variants."""
    ip, ix, dv = a.indptr, a.indices, a.data
    n = x.size
    order = range(n) if forward else range(n - 1, -1, -1)
    for _ in range(2):
        for i in order:
            cols = ix[ip[i]:ip[i + 1]]
            vals = dv[ip[i]:ip[i + 1]]
            d = vals[cols == i][0]
            if split:  # the not-yet-updated side first, then the updated side (the GPU's split sweep)
                later = cols > i if forward else cols < i
                earlier = cols < i if forward else cols > i
                s = b[i]
                for c, v in zip(cols[later], vals[later]):
                    s -= v * x[c]
                for c, v in zip(cols[earlier], vals[earlier]):
                    s -= v * x[c]
            else:
                s = b[i]
                for c, v in zip(cols, vals):
                    if c != i:
                        s -= v * x[c]
            x[i] = s * (1.0 / d) if recip else s / d


def vcycle(mg, b, **opt):
    mats, tr = mg.mats, mg.transfers
    top = len(mats) - 1

    def cycle(k, bb):
        if k == 0:
            return sla.cho_solve(mg.coarse, bb, check_finite=False)
        a = mats[k]
        finest = k == top
        x = np.zeros_like(bb)
        if finest:
            x[-1] = bb[-1] / a.corner
        badj = bb[:-1] - a.border * x[-1]
        xc = x[:-1].copy()
        gs(a.core, xc, badj, True, opt.get("recip", False), opt.get("split", False))
        x[:-1] = xc
        r = bb - a.matvec(x)
        p = tr[k - 1]
        rc = np.empty(p.shape[1] + 1)
        rc[:-1] = p.T @ r[:-1]
        rc[-1] = r[-1]
        e = cycle(k - 1, rc)
        x[:-1] += p @ e[:-1]
        if finest or not opt.get("drop_ealpha", False):
            x[-1] += e[-1]
        xa = x[-1] if (finest or not opt.get("post_alpha0", False)) else 0.0
        badj = bb[:-1] - a.border * xa
        xc = x[:-1].copy()
        gs(a.core, xc, badj, False, opt.get("recip", False), opt.get("split", False))
        x[:-1] = xc
        if finest:
            x[-1] += (bb[-1] - a.border @ x[:-1] - a.corner * x[-1]) / a.corner
        return x

    return cycle(top, b)


def main():
    path, mx, my, levels = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    zg = np.load(path)
    prob = oracle.build_problem2d("cantilever", mx, my, levels, 0.5)
    n, m = prob.n, prob.m
    rng = np.random.default_rng(0)
    u = rng.normal(0.0, 1e-2, n)
    rho = rng.uniform(0.5, 2.0, m)
    rng.standard_normal(n + 1)
    one = np.ones(m)
    st = oracle.PbmState(u=u, alpha=1e-3, nu_lo=one.copy(), nu_up=one.copy(), rho=rho, mu_lo=one.copy(),
                         mu_up=one.copy(), p=np.full(m, 1e-2), q_lo=one.copy(), q_up=one.copy())
    ops = oracle.ElementOps2D(prob.fine)
    ev = oracle.eval_lagrangian(st, ops, prob.f, oracle.DensityBounds.for_problem(m, prob.volume, 0.0),
                                oracle.PenaltyBarrier())
    mat, _ = oracle.schur_system(ev, ops)
    mg = oracle.MgPreconditioner(mat, prob.transfers)
    x = np.random.default_rng(1000).standard_normal(n + 1)
    z0 = mg.apply(x)
    print("oracle vs GPU", np.abs(z0 - zg).max() / np.abs(z0).max())
    for name, opt in (("plain", {}), ("recip", {"recip": True}), ("split", {"split": True}),
                      ("drop_ealpha", {"drop_ealpha": True}), ("post_alpha0", {"post_alpha0": True}),
                      ("recip+split", {"recip": True, "split": True})):
        z = vcycle(mg, x, **opt)
        print(f"{name:14s} vs oracle {np.abs(z - z0).max() / np.abs(z0).max():.2e}   "
              f"vs GPU {np.abs(z - zg).max() / np.abs(z0).max():.2e}")


if __name__ == "__main__":
    main()
