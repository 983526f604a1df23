"""Where does the GPU V-cycle leave the oracle?  (diagnostic, GPU box)

For cantilever hierarchies of growing depth (coarse grid fixed) and for the
1024x512 grid over different coarse grids, print the max-norm relative
distance between the GPU and the oracle (bitwise equal to the reference on
C3, tests/golden/c3_ref_samples.npz) for every level apply and the V-cycle.

python tools/checks/diag_vcycle_levels.py [--quick]
"""

from __future__ import annotations

import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)

import oracle  # noqa: E402
import paper_1904_06556_b200 as vts  # noqa: E402


def rel(a, b):
    a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a
    return float(np.abs(a - b).max() / np.abs(b).max())


def run(mx, my, levels, both=False):
    prob = vts.build_problem("cantilever", mx, my, levels, 0.5)
    oprob = oracle.build_problem2d("cantilever", mx, my, levels, 0.5)
    n, m = prob.n, prob.m
    rng = np.random.default_rng(0)
    u = rng.normal(0.0, 1e-2, n)
    rho = rng.uniform(0.5, 2.0, m)
    rng.standard_normal(n + 1)
    one = np.ones(m)
    nl, nu = one.copy(), one.copy()
    if both:
        nl, nu = rng.uniform(0, 1e-2, m), rng.uniform(0, 1e-2, m)
    st = dict(u=u, alpha=1e-3, nu_lo=nl, nu_up=nu, rho=rho, mu_lo=one.copy(), mu_up=one.copy(),
              p=np.full(m, 1e-2), q_lo=one.copy(), q_up=one.copy())
    dst = vts.PbmState(**{k: (v if k == "alpha" else torch.as_tensor(v, device="cuda")) for k, v in st.items()})
    ops = vts.ElementOps(prob.fine)
    ev = vts.eval_lagrangian(dst, ops, prob.f, vts.DensityBounds.for_problem(m, prob.volume, 0.0),
                             vts.PenaltyBarrier())
    mat, rhs = vts.schur_system(ev, ops)
    mg = vts.MgPreconditioner(mat, prob.transfers)
    oops = oracle.ElementOps2D(oprob.fine)
    oev = oracle.eval_lagrangian(oracle.PbmState(**st), oops, oprob.f,
                                 oracle.DensityBounds.for_problem(m, oprob.volume, 0.0), oracle.PenaltyBarrier())
    omat, orhs = oracle.schur_system(oev, oops)
    omg = oracle.MgPreconditioner(omat, oprob.transfers)
    lv = []
    for k, (a, oa) in enumerate(zip(mg.mats, omg.mats)):
        v = np.random.default_rng(2000 + k).standard_normal(oa.core_dim + 1)
        lv.append(rel(a.matvec(torch.as_tensor(v, device="cuda")), oa.matvec(v)))
    x = np.random.default_rng(1000).standard_normal(n + 1)
    zg = mg.apply(torch.as_tensor(x, device="cuda")).cpu().numpy()
    vc = rel(zg, omg.apply(x))
    if SAVE:
        os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
        np.save(os.path.join(REPO, "gpurun_out", f"vc_gpu_{mx}x{my}_L{levels}_{int(both)}.npy"), zg)
    vr = rel(mg.apply(rhs), omg.apply(orhs))
    print(f"{prob.fine.ex}x{prob.fine.ey} coarse {mx}x{my} L={levels} both={both}: V-cycle(x) {vc:.2e} "
          f"V-cycle(rhs) {vr:.2e} | level applies " + " ".join(f"{e:.1e}" for e in lv), flush=True)


SAVE = "--save" in sys.argv


def main():
    quick = "--quick" in sys.argv
    if "--small" in sys.argv:
        for mx, my, levels in ((4, 2, 2), (8, 4, 2), (16, 8, 2), (4, 2, 3), (8, 4, 3), (4, 2, 4), (4, 2, 9)):
            run(mx, my, levels)
        return
    for levels in range(3, 10):
        run(4, 2, levels)
    if quick:
        return
    for mx, my, levels in ((8, 4, 8), (16, 8, 7), (32, 16, 6)):
        run(mx, my, levels)
    run(4, 2, 9, both=True)


if __name__ == "__main__":
    main()
