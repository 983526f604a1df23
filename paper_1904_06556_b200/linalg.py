"""Bordered Newton operator, MINRES and tolerance policy (linalg.py of the reference).

* `NewtonMatrix` — the bordered Schur matrix [[A, c], [c^T, d]] of
  `schur_system` held matrix-free in the device context; `matvec` is
  `BorderedMatrix.matvec` (linalg.py:56-62) without the CSR.
* `minres_solve` — `linalg.py:128-242` run entirely on the device (vector
  recurrences and Givens scalars), same contract: convergence means the true
  relative residual is <= tol; errors raise `MinresError` carrying the last
  sound iterate.
* `MinresConfig`, `MinresResult`, `MinresError`, `StagnationTolerance` keep
  the reference's fields and semantics (linalg.py:84-115, 260-286).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import torch

from . import _lib
from .fem import ptr


class NewtonMatrix:
    """Matrix-free bordered Schur matrix bound in an `ElementOps` context."""

    def __init__(self, ops, border: torch.Tensor, corner: float, version: int):
        self.ops = ops
        self.border = border
        self.corner = corner
        self._version = version

    @property
    def shape(self):
        return (self.ops.n + 1, self.ops.n + 1)

    @property
    def core_dim(self) -> int:
        return self.ops.n

    def _check_current(self) -> None:
        if self.ops._system_version != self._version:
            raise RuntimeError("this Newton matrix was superseded by a later schur_system call")

    def matvec(self, x: torch.Tensor) -> torch.Tensor:
        self._check_current()
        x = self.ops.check_vec(x, self.ops.n + 1, "x")
        y = self.ops.vec(self.ops.n + 1)
        _lib.check(_lib.load().vts_newton_apply(self.ops.handle, ptr(x), ptr(y)), "vts_newton_apply")
        return y

    __matmul__ = matvec


@dataclass
class MinresConfig:
    tol: float = 1e-4
    max_iters: int = 0  # 0 -> 3 * system dimension
    floor: float = 1e-9

    def __post_init__(self) -> None:
        if not 0.0 < self.tol < 1.0:
            raise ValueError(f"tol must lie in (0, 1), got {self.tol}")
        if self.max_iters < 0:
            raise ValueError("max_iters must be non-negative")


@dataclass
class MinresResult:
    x: torch.Tensor
    iterations: int
    relres: float
    converged: bool


class MinresError(RuntimeError):
    """Breakdown, NaN recurrence, or indefinite preconditioner (linalg.py:107-115)."""

    def __init__(self, message: str, x=None):
        super().__init__(message)
        self.x = x


_ERRORS = {
    _lib.VTS_E_INDEFINITE: "preconditioner is indefinite: <M r, r> < 0",
    _lib.VTS_E_BREAKDOWN: "MINRES recurrence broke down",
    _lib.VTS_E_NONFINITE: "NaN/inf encountered in MINRES recurrences",
}


def minres_solve(a, b: torch.Tensor, config: MinresConfig, precond=None, x0=None, history: list | None = None
                 ) -> MinresResult:
    """Preconditioned MINRES for the bound Newton matrix (linalg.py:128-242).

    `a` must be the `NewtonMatrix` returned by `schur_system`; `precond` is
    None or the `apply` of an `MgPreconditioner` built on it.  `history`, when
    a list, receives the true relative residual after every iteration.
    """
    if not isinstance(a, NewtonMatrix):
        raise TypeError("minres_solve runs on the device Newton matrix returned by schur_system")
    if x0 is not None:
        raise NotImplementedError("warm starts are not used on the PBM path (pbm.py:282-285)")
    a._check_current()
    ops = a.ops
    use_mg = 0
    if precond is not None:
        owner = getattr(precond, "__self__", None)
        from .multigrid import MgPreconditioner

        if not isinstance(owner, MgPreconditioner) or owner.ops is not ops or precond.__func__ is not MgPreconditioner.apply:
            raise TypeError("precond must be MgPreconditioner.apply of a preconditioner built on this matrix")
        owner._check_current()
        use_mg = 1
    b = ops.check_vec(b, ops.n + 1, "b")
    x = ops.vec(ops.n + 1)
    cap = config.max_iters if config.max_iters > 0 else 3 * (ops.n + 1)
    hist = (ctypes.c_double * cap)() if history is not None else None
    it = ctypes.c_int32(0)
    rel = ctypes.c_double(0.0)
    conv = ctypes.c_int32(0)
    rc = _lib.load().vts_minres(ops.handle, ptr(b), ptr(x), config.tol, cap, config.floor, use_mg,
                                ctypes.byref(it), ctypes.byref(rel), ctypes.byref(conv), hist)
    if history is not None:
        history.extend(hist[: it.value])
    if rc in _ERRORS:
        raise MinresError(_ERRORS[rc], x)
    _lib.check(rc, "vts_minres")
    return MinresResult(x, it.value, rel.value, bool(conv.value))


@dataclass
class ComplementarityTolerance:
    """MINRES tolerance tied to the largest complementarity product (linalg.py:289-309):
    the monotone running minimum of max(scale * comp_max, floor)."""

    tol: float = 1e-2
    floor: float = 1e-9
    scale: float = 100.0

    def current(self) -> float:
        return self.tol

    def observe(self, comp_max: float) -> None:
        cand = max(self.scale * comp_max, self.floor)
        if cand < self.tol:
            self.tol = cand


@dataclass
class StagnationTolerance:
    """Tenfold shrink of the inner tolerance on stagnating Newton residuals."""

    tol: float
    floor: float = 1e-9
    shrink: float = 0.1
    trigger: float = 0.9
    _prev: float | None = field(default=None, init=False, repr=False)

    def current(self) -> float:
        return self.tol

    def reset(self) -> None:
        self._prev = None

    def observe(self, residual: float) -> None:
        if self._prev is not None and residual > self.trigger * self._prev:
            self.tol = max(self.shrink * self.tol, self.floor)
        self._prev = residual
