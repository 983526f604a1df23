"""Galerkin V(2,2) multigrid preconditioner on the device (multigrid.py of the reference).

`MgPreconditioner(fine, transfers)` builds, for the bound Newton matrix (or
the unbordered stiffness K(rho) of the DOC state solves, multigrid.py:85-86), the
finest-level block stencil, every coarse operator P^T A P (symmetrised), the
restricted borders and the dense Cholesky factor of the coarsest bordered
matrix with the reference's trace-scaled shift fallback
(multigrid.py:82-103).  `apply(v)` runs one V-cycle from a zero guess with
the reference's exact lexicographic Gauss-Seidel order (multigrid.py:35-64,
109-154).
"""

from __future__ import annotations

import ctypes
import logging

import torch

from . import _lib
from .fem import ptr
from .linalg import NewtonMatrix

log = logging.getLogger("paper_1904_06556_b200.multigrid")


class LevelOperator:
    """Probe handle for one level operator (MgPreconditioner.mats[k]): bordered
    (core_dim + 1 entries) over a Newton matrix, plain (core_dim) over K(rho)."""

    def __init__(self, pre: "MgPreconditioner", k: int):
        self._pre = pre
        self.level = k
        self.core_dim = pre.ops.level_size(k)
        self.bordered = pre.bordered
        self.dim = self.core_dim + (1 if self.bordered else 0)

    def matvec(self, x: torch.Tensor) -> torch.Tensor:
        self._pre._check_current()
        ops = self._pre.ops
        x = ops.check_vec(x, self.dim, "x")
        y = ops.vec(self.dim)
        _lib.check(_lib.load().vts_level_apply(ops.handle, self.level, ptr(x), ptr(y)), "vts_level_apply")
        return y


class MgPreconditioner:
    def __init__(self, fine: NewtonMatrix, transfers, sweeps: int = 2, shift_scale: float = 1e-12):
        if not isinstance(fine, NewtonMatrix):
            raise TypeError("MgPreconditioner takes a matrix bound in the device context: the NewtonMatrix of "
                            "schur_system or the StiffnessMatrix of ElementOps.assemble_stiffness")
        if sweeps != 2:
            raise ValueError("the device V-cycle implements the reference's V(2,2) (sweeps=2)")
        fine._check_current()
        self.ops = fine.ops
        self.transfers = list(transfers)
        hier = self.ops.problem
        if len(self.transfers) != len(hier.levels) - 1:
            raise ValueError("transfers must chain every level of the problem hierarchy")
        for k, t in enumerate(self.transfers):
            if tuple(t.shape) != (hier.levels[k + 1].n, hier.levels[k].n):
                raise ValueError(f"transfer {k} does not match the hierarchy")
        self.sweeps = sweeps
        self.bordered = fine.bordered  # multigrid.py:85-86: a plain matrix gets no border
        self.dim = fine.dim
        self._version = fine._version
        shifted = ctypes.c_int32(0)
        rc = _lib.load().vts_mg_setup(self.ops.handle, shift_scale, ctypes.byref(shifted))
        if rc == _lib.VTS_E_CHOLESKY:  # the shifted retry failed too: cho_factor's error (multigrid.py:102)
            import numpy as np

            raise np.linalg.LinAlgError(_lib.last_error())
        _lib.check(rc, "vts_mg_setup")
        self.shifted = bool(shifted.value)
        if self.shifted:
            log.warning("coarse matrix is not positive definite; retrying Cholesky with a trace-scaled shift")
        self.mats = [LevelOperator(self, k) for k in range(len(hier.levels))]

    @property
    def levels(self) -> int:
        return len(self.mats)

    def _check_current(self) -> None:
        if self.ops._system_version != self._version:
            raise RuntimeError("this preconditioner was built for a superseded Newton matrix")

    def apply(self, v: torch.Tensor) -> torch.Tensor:
        self._check_current()
        v = self.ops.check_vec(v, self.dim, "v")
        z = self.ops.vec(self.dim)
        _lib.check(_lib.load().vts_vcycle(self.ops.handle, ptr(v), ptr(z)), "vts_vcycle")
        return z
