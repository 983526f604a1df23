"""The reference's own rounding sensitivity on the MBB runs: FMA Gauss-Seidel.

Run HERE (the build container, where /root/reference is mounted):

    NUMBA_CACHE_DIR=/tmp/numba_vtsopt python tests/golden/fma_sensitivity.py

It re-runs the unmodified reference `solve_pbm` on C2 (2D glue of
`make_golden.py`) with exactly one change: the two numba Gauss-Seidel loops
(`multigrid.py:35-64`) are recompiled with floating-point contraction allowed
(`fastmath={"contract"}`), so each `s -= v * x[j]` becomes one fused
multiply-add, as on the GPU.  Everything else -- the operation order, every
other module -- is the reference.  The GPU smoother fuses the same products,
so the distance between this run and the stock run is the size of a
rounding-level perturbation of the reference itself.

It does the same for the 32x16 MBB of `pbm_mbb32.npz` (~140 MINRES iterations
per late Newton step, where single per-Newton counts move under rounding) and,
with the argument `c4`, for the full 1024x512 solve of `pbm_c4.npz`.

Output `fma_sensitivity.npz`: for both runs the FMA run's counts, objective
and thickness field (C2: at `pbm_c2.npz`'s 512 sample positions), plus the
max / 2-norm distance to the stock run.  `tests/test_gpu_parity.py` bounds
the GPU's own distance to the stock run by this measured sensitivity.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as mg_  # noqa: E402  (reference + 2D glue)
from numba import njit  # noqa: E402


@njit(fastmath={"contract"})
def _gs_forward_fma(indptr, indices, data, x, b, sweeps):
    for _ in range(sweeps):
        for i in range(x.size):
            acc = b[i]
            d = 0.0
            for k in range(indptr[i], indptr[i + 1]):
                col = indices[k]
                if col == i:
                    d = data[k]
                else:
                    acc -= data[k] * x[col]
            x[i] = acc / d


@njit(fastmath={"contract"})
def _gs_backward_fma(indptr, indices, data, x, b, sweeps):
    for _ in range(sweeps):
        for i in range(x.size - 1, -1, -1):
            acc = b[i]
            d = 0.0
            for k in range(indptr[i], indptr[i + 1]):
                col = indices[k]
                if col == i:
                    d = data[k]
                else:
                    acc -= data[k] * x[col]
            x[i] = acc / d


def fused_instructions() -> int:
    """Count fused multiply-add instructions in the compiled forward loop (proof of contraction)."""
    asm = "".join(_gs_forward_fma.inspect_asm().values())
    return sum(asm.count(op) for op in ("vfmadd", "vfnmadd", "vfmsub", "vfnmsub"))


def run(prob, stock: dict, with_vectors: bool) -> dict:
    out, rep = mg_.pbm_fixture(prob, with_vectors=with_vectors)
    key = "rho" if with_vectors else "rho_sample"  # whole field, or pbm_c2.npz's 512 samples
    sample, ref = out[key], stock[key]
    d = sample - ref
    res = {
        "objective": rep.objective, "outer": rep.outer_iterations,
        "minres_per_newton": out["minres_per_newton"], "rho_sample": sample,
        "max_abs_diff_vs_stock": float(np.abs(d).max()),
        "l2_rel_diff_vs_stock": float(np.linalg.norm(d) / np.linalg.norm(ref)),
        "objective_rel_diff_vs_stock": float(abs(rep.objective - float(stock["objective"])) / float(stock["objective"])),
        "volume_rel_diff_vs_stock": float(abs(rep.volume - float(stock["volume"])) / abs(float(stock["volume"]))),
        "same_counts": bool(np.array_equal(out["minres_per_newton"], stock["minres_per_newton"])),
        "minres_total_diff": int(out["minres_per_newton"].sum() - stock["minres_per_newton"].sum()),
    }
    if not with_vectors:
        res["rho_sample_idx"] = out["rho_sample_idx"]
    return res


def main(argv) -> None:
    mg_.rmg._gs_forward = _gs_forward_fma
    mg_.rmg._gs_backward = _gs_backward_fma
    path = os.path.join(HERE, "fma_sensitivity.npz")
    out = dict(np.load(path)) if os.path.exists(path) else {}
    which = set(argv) or {"c2", "mbb32"}
    if "c2" in which:
        c2 = run(mg_.build_config("C2"), dict(np.load(os.path.join(HERE, "pbm_c2.npz"))), with_vectors=False)
        out.update({f"c2_{k}": v for k, v in c2.items()})
    if "mbb32" in which:
        mbb = run(mg_.build_problem2d("mbb", 4, 2, 4, 0.4), dict(np.load(os.path.join(HERE, "pbm_mbb32.npz"))),
                  with_vectors=True)
        out.update({f"mbb32_{k}": v for k, v in mbb.items()})
    if "c4" in which:  # the north_star target (~6 min): the thickness field's own sensitivity
        c4 = run(mg_.build_config("C4"), dict(np.load(os.path.join(HERE, "pbm_c4.npz"))), with_vectors=True)
        c4.pop("rho_sample")  # 4 MB; the distances are what the tests use
        out.update({f"c4_{k}": v for k, v in c4.items()})
    nfma = fused_instructions()
    assert nfma > 0, "the host compiler did not contract the Gauss-Seidel products"
    out["fma_instructions"] = nfma
    np.savez_compressed(path, **out)
    print({k: v for k, v in out.items() if np.ndim(v) == 0})


if __name__ == "__main__":
    main(sys.argv[1:])
