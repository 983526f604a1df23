"""Galerkin V(2,2) multigrid preconditioner (oracle side).

Restates `multigrid.py:67-154` of the reference: Galerkin chain built at
construction (`:88-90`), dense Cholesky of the coarsest bordered matrix with
a trace-scaled shift fallback (`:92-103`), V-cycle from a zero guess with
two forward lexicographic Gauss-Seidel sweeps before and two backward sweeps
after the coarse correction on the core unknowns (`:113-154`), the border
unknown transferred by identity, and the finest-level diagonal relaxation of
the border unknown on both sides (`:121-122,141-142`).

The sequential sweeps run in `csrc/gs_oracle.c` (restating the reference's
numba loops `multigrid.py:35-64`), loaded through ctypes and built on demand.
"""

from __future__ import annotations

import ctypes
import logging
import os
import subprocess

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from .krylov import BorderedMatrix

log = logging.getLogger("oracle.vcycle")

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libvts_oracle_gs.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            subprocess.run(["make", "-s", "-C", _HERE], check=True)
        lib = ctypes.CDLL(_LIB_PATH)
        ptr = ctypes.c_void_p
        for name in ("vts_oracle_gs_forward", "vts_oracle_gs_backward"):
            fn = getattr(lib, name)
            fn.argtypes = [ptr, ptr, ptr, ptr, ptr, ctypes.c_int64, ctypes.c_int32]
            fn.restype = None
        _lib = lib
    return _lib


class _CsrView:
    """int64 copies of a CSR structure for the C sweeps."""

    def __init__(self, a: sp.csr_matrix):
        self.indptr = np.ascontiguousarray(a.indptr, dtype=np.int64)
        self.indices = np.ascontiguousarray(a.indices, dtype=np.int64)
        self.data = np.ascontiguousarray(a.data, dtype=np.float64)
        self.n = a.shape[0]

    def sweep(self, x: np.ndarray, b: np.ndarray, sweeps: int, forward: bool) -> None:
        lib = _load()
        fn = lib.vts_oracle_gs_forward if forward else lib.vts_oracle_gs_backward
        assert x.flags.c_contiguous and x.dtype == np.float64
        b = np.ascontiguousarray(b, dtype=np.float64)
        fn(
            self.indptr.ctypes.data,
            self.indices.ctypes.data,
            self.data.ctypes.data,
            x.ctypes.data,
            b.ctypes.data,
            self.n,
            sweeps,
        )


class MgPreconditioner:
    def __init__(self, fine, transfers, sweeps: int = 2, shift_scale: float = 1e-12):
        if sp.issparse(fine):
            fine = BorderedMatrix(fine.tocsr(), None, 0.0)
        self.transfers = list(transfers)
        self.sweeps = sweeps
        chain = [fine]
        for p in reversed(self.transfers):
            chain.append(chain[-1].galerkin(p))
        chain.reverse()
        self.mats = chain  # coarsest first
        self._csr = [_CsrView(m.core) for m in chain]
        self.shifted = False
        dense = chain[0].to_dense()
        try:
            self.coarse = sla.cho_factor(dense, check_finite=False)
        except np.linalg.LinAlgError:
            shift = shift_scale * np.trace(dense) / dense.shape[0]
            log.warning(
                "coarse matrix is not positive definite; retrying Cholesky with shift %.3e", shift
            )
            self.coarse = sla.cho_factor(dense + shift * np.eye(dense.shape[0]), check_finite=False)
            self.shifted = True

    @property
    def levels(self) -> int:
        return len(self.mats)

    def apply(self, v: np.ndarray) -> np.ndarray:
        return self._cycle(self.levels - 1, v)

    def _smooth(self, k: int, x: np.ndarray, b: np.ndarray, forward: bool) -> None:
        a = self.mats[k]
        if a.border is not None:
            rhs = b[:-1] - a.border * x[-1]
            core = x[:-1]  # a view: the C sweep writes through it
        else:
            rhs, core = b, x
        self._csr[k].sweep(core, rhs, self.sweeps, forward)

    def _cycle(self, k: int, b: np.ndarray) -> np.ndarray:
        if k == 0:
            return sla.cho_solve(self.coarse, b, check_finite=False)
        a = self.mats[k]
        has_border = a.border is not None
        top = k == self.levels - 1
        x = np.zeros_like(b)
        if has_border and top:
            x[-1] = b[-1] / a.corner
        self._smooth(k, x, b, forward=True)
        r = b - a.matvec(x)
        p = self.transfers[k - 1]
        if has_border:
            rc = np.empty(p.shape[1] + 1)
            rc[:-1] = p.T @ r[:-1]
            rc[-1] = r[-1]
        else:
            rc = p.T @ r
        e = self._cycle(k - 1, rc)
        if has_border:
            x[:-1] += p @ e[:-1]
            x[-1] += e[-1]
        else:
            x += p @ e
        self._smooth(k, x, b, forward=False)
        if has_border and top:
            x[-1] += (b[-1] - a.border @ x[:-1] - a.corner * x[-1]) / a.corner
        return x
