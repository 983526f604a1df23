"""The reference V-cycle's own rounding sensitivity at the target size (C3, 9 levels).

Run HERE (the build container, where /root/reference is mounted):

    NUMBA_CACHE_DIR=/tmp/numba_vtsopt python tests/golden/vcycle_sensitivity.py

On the C3 states of `make_golden_fullsize.py` it applies the unmodified
reference `MgPreconditioner` (multigrid.py:82-154) twice to the same vectors:
once stock, once with only its two numba Gauss-Seidel loops recompiled with
floating-point contraction (one fused multiply-add per `s -= v * x[j]`, as
the GPU smoother computes; `fma_sensitivity.py`), and once with the Galerkin
triple product's inner sums (A P, linalg.py:78) taken in reverse column
order, and once with every V-cycle residual r = b - A x
(multigrid.py:125) summing each row's products in reverse column order --
all last-bit reorderings of the same arithmetic.  The max-norm distance
between the two, relative to max|z|, is the size of a rounding-level
perturbation of the reference V-cycle itself.  Measured: the Gauss-Seidel
and residual reorderings move it by ~1e-15, the Galerkin reordering by
~1e-12 -- small entries of the coarse operators are sums that cancel, and
their last-bit differences are amplified through the 9-level hierarchy.  `tests/test_gpu_target.py` bounds the GPU V-cycle's distance to the
reference by this measured figure (x2).  Output: `vcycle_sensitivity.npz`.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import fma_sensitivity as fs  # noqa: E402  (reference + 2D glue + the FMA loops)
import make_golden_fullsize as mgf  # noqa: E402

mg_ = fs.mg_


def _galerkin_reversed_sums(self, p):
    """linalg.py:76-81 with each row of A's products summed in reverse column order
    inside A P (P's weights are powers of two: only the order of the sums changes)."""
    core = (p.T @ (_reversed_rows(self.core) @ p)).tocsr()
    core = ((core + core.T) * 0.5).tocsr()
    border = None if self.border is None else p.T @ self.border
    return mg_.rlinalg.BorderedMatrix(core, border, self.corner)


def _reversed_rows(a):
    """The same CSR matrix with every row's entries stored in reverse column order."""
    import scipy.sparse as sp

    indices = a.indices.copy()
    data = a.data.copy()
    for i in range(a.shape[0]):
        lo, hi = a.indptr[i], a.indptr[i + 1]
        indices[lo:hi] = a.indices[lo:hi][::-1]
        data[lo:hi] = a.data[lo:hi][::-1]
    out = sp.csr_matrix((data, indices, a.indptr.copy()), shape=a.shape)
    out.has_sorted_indices = False
    return out


_STOCK_MATVEC = None
_REV_CACHE = {}


def _matvec_reversed_sums(self, x):
    """linalg.py:56-62 with each row's products summed in reverse column order."""
    key = id(self.core)
    if key not in _REV_CACHE:
        _REV_CACHE[key] = (self.core, _reversed_rows(self.core))
    core = _REV_CACHE[key][1]
    if self.border is None:
        return core @ x
    y = np.empty_like(x)
    y[:-1] = core @ x[:-1] + self.border * x[-1]
    y[-1] = self.border @ x[:-1] + self.corner * x[-1]
    return y


def main() -> None:
    prob = mg_.build_config("C3")
    stock_gs = (mg_.rmg._gs_forward, mg_.rmg._gs_backward)
    stock_gal = mg_.rlinalg.BorderedMatrix.galerkin
    variants = {
        "fma": (( fs._gs_forward_fma, fs._gs_backward_fma), stock_gal),
        "rap_order": (stock_gs, _galerkin_reversed_sums),
        "fma+rap_order": ((fs._gs_forward_fma, fs._gs_backward_fma), _galerkin_reversed_sums),
    }

    stock_mv = mg_.rlinalg.BorderedMatrix.matvec
    variants["resid_order"] = (stock_gs, stock_gal)  # residual sums in reverse column order

    def vcycle(s_mat, b, gs, gal, reversed_residual=False):
        mg_.rmg._gs_forward, mg_.rmg._gs_backward = gs
        mg_.rlinalg.BorderedMatrix.galerkin = gal
        try:
            pre = mg_.rmg.MgPreconditioner(s_mat, prob.transfers)
            if reversed_residual:  # only the V-cycle's residuals r = b - A x (multigrid.py:125)
                mg_.rlinalg.BorderedMatrix.matvec = _matvec_reversed_sums
            return pre.apply(b)
        finally:
            mg_.rmg._gs_forward, mg_.rmg._gs_backward = stock_gs
            mg_.rlinalg.BorderedMatrix.galerkin = stock_gal
            mg_.rlinalg.BorderedMatrix.matvec = stock_mv

    out = {}
    for tag, both in (("ref", False), ("br", True)):
        st, bench_rhs = mgf.c3_state(prob, 0, both)
        ops = mg_.ElementOps2DGlue(prob.fine)
        bounds = mg_.rfem.DensityBounds.for_problem(prob.m, prob.volume, 0.0)
        ev = mg_.rpbm.eval_lagrangian(st, ops, prob.f, bounds, mg_.PEN)
        s_mat, rhs = mg_.rpbm.schur_system(ev, ops)
        x = np.random.default_rng(1000).standard_normal(prob.n + 1)
        for name, b in (("x", x), ("rhs", rhs), ("bench_rhs", bench_rhs)):
            z0 = vcycle(s_mat, b, stock_gs, stock_gal)
            for var, (gs, gal) in variants.items():
                z1 = vcycle(s_mat, b, gs, gal, reversed_residual=(var == "resid_order"))
                rel = float(np.abs(z1 - z0).max() / np.abs(z0).max())
                out[f"{tag}_{name}_{var}_maxrel"] = rel
                print(f"[{tag}] V-cycle({name}) stock vs {var}: max|dz|/max|z| = {rel:.3e}", flush=True)
    for var in variants:
        out[f"worst_{var}"] = max(v for k, v in out.items() if k.endswith(f"_{var}_maxrel"))
    out["fma_instructions"] = fs.fused_instructions()
    np.savez_compressed(os.path.join(HERE, "vcycle_sensitivity.npz"), **out)
    print({k: v for k, v in out.items() if k.startswith("worst")})


if __name__ == "__main__":
    main()
