"""Penalty/barrier kernel phi (penalty.py:27-99 of the reference).

`PenaltyBarrier` keeps the reference's interface: `branch` in (-1, 0) is
validated at construction, and `value`/`deriv`/`deriv2` evaluate phi, phi',
phi'' of a CUDA tensor on the device (the same inlined device function the
fused element passes use), with the reference's saturation RuntimeWarning.
"""

from __future__ import annotations

import ctypes
import warnings
from dataclasses import dataclass

import torch

from . import _lib
from .fem import as_dev, ptr

_SAT_MSG = "penalty kernel input saturated at +/-1e150; the iterate is far outside the useful range of the kernel"


def warn_saturated(flags: int) -> None:
    if flags & _lib.VTS_W_SATURATED:
        warnings.warn(_SAT_MSG, RuntimeWarning, stacklevel=3)


@dataclass(frozen=True)
class PenaltyBarrier:
    branch: float = -0.5

    def __post_init__(self) -> None:
        if not -1.0 < self.branch < 0.0:
            raise ValueError(f"branch point must lie in (-1, 0), got {self.branch}")

    def _eval(self, tau, which: int, ops):
        scalar = not isinstance(tau, torch.Tensor) and not hasattr(tau, "__len__")
        t = as_dev([tau] if scalar else tau).reshape(-1)
        out = torch.empty_like(t)
        outs = [None, None, None]
        outs[which] = out
        flags = ctypes.c_uint32(0)
        handle = ops.handle if ops is not None else _scratch_ctx().handle
        rc = _lib.load().vts_penalty_eval(handle, t.numel(), ptr(t), self.branch, ptr(outs[0]), ptr(outs[1]),
                                          ptr(outs[2]), ctypes.byref(flags))
        _lib.check(rc, "vts_penalty_eval")
        warn_saturated(flags.value)
        return float(out[0]) if scalar else out

    def value(self, tau, ops=None):
        return self._eval(tau, 0, ops)

    def deriv(self, tau, ops=None):
        return self._eval(tau, 1, ops)

    def deriv2(self, tau, ops=None):
        return self._eval(tau, 2, ops)


_SCRATCH = None


def _scratch_ctx():
    """A one-element context used only for stand-alone phi evaluations."""
    global _SCRATCH
    if _SCRATCH is None:
        from .fem import ElementOps
        from .problem import build_problem

        _SCRATCH = ElementOps(build_problem("cantilever", 1, 1, 1, 0.5).fine)
    return _SCRATCH
