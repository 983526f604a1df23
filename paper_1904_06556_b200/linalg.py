"""Bordered Newton operator, MINRES and tolerance policy (linalg.py of the reference).

* `NewtonMatrix` — the bordered Schur matrix [[A, c], [c^T, d]] of
  `schur_system` held matrix-free in the device context; `matvec` is
  `BorderedMatrix.matvec` (linalg.py:56-62) without the CSR.
  `StiffnessMatrix` — the unbordered K(rho) of the DOC state solves.
* `minres_solve` — `linalg.py:128-242` run entirely on the device (vector
  recurrences and Givens scalars), same contract: convergence means the true
  relative residual is <= tol; errors raise `MinresError` carrying the last
  sound iterate.
* `MinresConfig`, `MinresResult`, `MinresError`, `FixedTolerance`,
  `StagnationTolerance`, `ComplementarityTolerance` keep the reference's
  fields and semantics (linalg.py:84-115, 250-308).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import torch

from . import _lib
from .fem import ptr


class NewtonMatrix:
    """Matrix-free bordered Schur matrix bound in an `ElementOps` context."""

    bordered = True

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

    @property
    def dim(self) -> int:
        return self.shape[0]

    def _check_current(self) -> None:
        if self.ops._system_version != self._version:
            raise RuntimeError("this matrix was superseded by a later system bound in the same context")

    def matvec(self, x: torch.Tensor) -> torch.Tensor:
        self._check_current()
        x = self.ops.check_vec(x, self.dim, "x")
        y = self.ops.vec(self.dim)
        _lib.check(_lib.load().vts_newton_apply(self.ops.handle, ptr(x), ptr(y)), "vts_newton_apply")
        return y

    __matmul__ = matvec


class StiffnessMatrix(NewtonMatrix):
    """K(rho) = sum_e rho_e K_e on the free dofs, matrix-free in the context
    (`ElementOps.assemble_stiffness`, fem.py:211-219): the unbordered operator of
    the DOC state solves (doc.py:137-146).  `border` is None like the
    reference's plain CSR matrix (linalg.py:49-53)."""

    bordered = False

    def __init__(self, ops, version: int):
        super().__init__(ops, None, 0.0, version)

    @property
    def shape(self):
        return (self.ops.n, self.ops.n)


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


def _own_mg(precond, a) -> bool:
    """precond is the `apply` of an MgPreconditioner built on the bound matrix `a`."""
    from .multigrid import MgPreconditioner

    owner = getattr(precond, "__self__", None)
    return (isinstance(owner, MgPreconditioner) and owner.ops is a.ops
            and getattr(precond, "__func__", None) is MgPreconditioner.apply and owner._version == a._version)


def _dev_view(addr: int, length: int) -> torch.Tensor:
    """A torch view of `length` doubles of device memory owned by the library."""

    class _Buf:
        __cuda_array_interface__ = {"shape": (length,), "typestr": "<f8", "data": (addr, False), "version": 3}

    return torch.as_tensor(_Buf(), device="cuda")


def _as_operator(a):
    """_as_matvec (linalg.py:118-125): bound matrices, dense / sparse tensors, callables."""
    if isinstance(a, NewtonMatrix):
        return a.matvec, a.dim
    if isinstance(a, torch.Tensor):
        if a.dim() != 2 or a.shape[0] != a.shape[1]:
            raise ValueError("the operator must be a square matrix")
        mat = a if a.is_cuda else a.to("cuda")
        return (lambda v: mat @ v), a.shape[0]
    if hasattr(a, "tocsr") or hasattr(a, "__array__"):  # scipy sparse / numpy: move to the device once
        import numpy as np
        import scipy.sparse as sp

        if sp.issparse(a):
            c = a.tocsr()
            mat = torch.sparse_csr_tensor(torch.as_tensor(c.indptr, dtype=torch.int64),
                                          torch.as_tensor(c.indices, dtype=torch.int64),
                                          torch.as_tensor(c.data, dtype=torch.float64), size=c.shape).to("cuda")
        else:
            mat = torch.as_tensor(np.asarray(a, dtype=np.float64), device="cuda")
        return (lambda v: mat @ v), mat.shape[0]
    if callable(a):
        return a, None
    raise TypeError(f"cannot use {type(a).__name__} as a MINRES operator")


def minres_solve(a, b: torch.Tensor, config: MinresConfig, precond=None, x0=None, history: list | None = None
                 ) -> MinresResult:
    """Preconditioned MINRES (linalg.py:128-242), same contract: convergence means
    the true relative residual is <= tol; errors raise `MinresError` carrying the
    last sound iterate.

    `a` is the bound Newton matrix of `schur_system` or the bound stiffness of
    `ElementOps.assemble_stiffness` (then with `precond` None or its own
    `MgPreconditioner.apply` the whole solve runs in the context: vts_minres_warm),
    or any operator the reference accepts (linalg.py:118-125) -- a dense or
    sparse matrix, or a callable on device vectors -- with any callable
    preconditioner (vts_minres_generic: the same device recurrences, the
    operator applied through a callback).  `x0` warm-starts (linalg.py:144-154).
    `history`, when a list, receives the true relative residual after every
    iteration.
    """
    lib = _lib.load()
    if isinstance(a, NewtonMatrix) and (precond is None or _own_mg(precond, a)):
        a._check_current()
        ops = a.ops
        if precond is not None:
            precond.__self__._check_current()
        b = ops.check_vec(b, a.dim, "b")
        if x0 is not None:
            x0 = ops.check_vec(torch.as_tensor(x0, dtype=torch.float64, device="cuda").contiguous(), a.dim, "x0")
        x = ops.vec(a.dim)
        cap = config.max_iters if config.max_iters > 0 else 3 * a.dim
        hist = (ctypes.c_double * cap)() if history is not None else None
        it, rel, conv = ctypes.c_int32(0), ctypes.c_double(0.0), ctypes.c_int32(0)
        rc = lib.vts_minres_warm(ops.handle, ptr(b), ptr(x), ptr(x0), config.tol, cap, config.floor,
                                 1 if precond is not None else 0, ctypes.byref(it), ctypes.byref(rel),
                                 ctypes.byref(conv), hist)
        if history is not None:
            history.extend(hist[: it.value])
        if rc in _ERRORS:
            raise MinresError(_ERRORS[rc], x)
        _lib.check(rc, "vts_minres_warm")
        return MinresResult(x, it.value, rel.value, bool(conv.value))
    return _minres_generic(a, b, config, precond, x0, history)


def _minres_generic(a, b, config, precond, x0, history):
    from .fem import ElementOps

    op, dim = _as_operator(a)
    if not (isinstance(b, torch.Tensor) and b.is_cuda and b.dtype == torch.float64):
        b = torch.as_tensor(b, dtype=torch.float64, device="cuda")
    b = b.contiguous()
    n = b.numel()
    if dim is not None and dim != n:
        raise ValueError(f"b has {n} entries, the operator {dim}")
    if x0 is not None:
        x0 = torch.as_tensor(x0, dtype=torch.float64, device="cuda").contiguous()
        if x0.numel() != n:
            raise ValueError(f"x0 has {x0.numel()} entries, expected {n}")
    ops = a.ops if isinstance(a, NewtonMatrix) else ElementOps.scratch()
    errors: list = []

    def wrap(fn):
        def cb(_user, pin, pout):
            try:
                res = fn(_dev_view(pin, n))
                out = _dev_view(pout, n)
                out.copy_(torch.as_tensor(res, dtype=torch.float64, device="cuda").reshape(-1))
                torch.cuda.current_stream().synchronize()
                return 0
            except Exception as exc:  # re-raised after the library returns
                errors.append(exc)
                return 1
        return _lib.APPLY_FN(cb)

    op_cb = wrap(op)
    pre_cb = wrap(precond) if precond is not None else None
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    cap = config.max_iters if config.max_iters > 0 else 3 * n
    hist = (ctypes.c_double * cap)() if history is not None else None
    it, rel, conv = ctypes.c_int32(0), ctypes.c_double(0.0), ctypes.c_int32(0)
    torch.cuda.current_stream().synchronize()
    rc = _lib.load().vts_minres_generic(ops.handle, n, ptr(b), ptr(x), ptr(x0), config.tol, cap, config.floor,
                                        ctypes.cast(op_cb, ctypes.c_void_p),
                                        ctypes.cast(pre_cb, ctypes.c_void_p) if pre_cb is not None else None, None,
                                        ctypes.byref(it), ctypes.byref(rel), ctypes.byref(conv), hist)
    if errors:
        raise errors[0]
    if history is not None:
        history.extend(hist[: it.value])
    if rc in _ERRORS:
        raise MinresError(_ERRORS[rc], x)
    _lib.check(rc, "vts_minres_generic")
    return MinresResult(x, it.value, rel.value, bool(conv.value))


@dataclass
class FixedTolerance:
    """Constant inner tolerance (linalg.py:250-257), the DOC state solves' policy."""

    tol: float = 1e-4

    def current(self) -> float:
        return self.tol

    def observe(self, *_args) -> None:
        pass


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
