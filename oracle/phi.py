"""Two-branch penalty/barrier kernel phi (oracle side).

Restates `penalty.py:27-99` of the reference: quadratic tau + tau^2/2 for
tau >= t (branch t in (-1, 0), default -1/2), and the C^2 logarithmic
extension  -c log((1 + 2t - tau)/(1 + t)) + t + t^2/2,  c = (1 + t)^2, below it
(`penalty.py:49-60`); derivatives `penalty.py:62-82`.  Inputs beyond 1e150 in
magnitude, NaN or inf are saturated with a RuntimeWarning
(`penalty.py:85-95`).
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np

SATURATION = 1e150
_HUGE = 1e300


def saturate(tau: np.ndarray) -> np.ndarray:
    if np.any(~np.isfinite(tau)) or np.any(np.abs(tau) > SATURATION):
        warnings.warn(
            "penalty kernel input saturated at +/-1e150; the iterate is far "
            "outside the useful range of the kernel",
            RuntimeWarning,
            stacklevel=3,
        )
        tau = np.clip(np.nan_to_num(tau, nan=0.0, posinf=_HUGE, neginf=-_HUGE), -SATURATION, SATURATION)
    return tau


def _scalar_or_array(x: np.ndarray):
    return x.item() if x.ndim == 0 else x


@dataclass(frozen=True)
class PenaltyBarrier:
    branch: float = -0.5

    def __post_init__(self) -> None:
        if not -1.0 < self.branch < 0.0:
            raise ValueError(f"branch point must lie in (-1, 0), got {self.branch}")

    def _split(self, tau):
        tau = saturate(np.asarray(tau, dtype=float))
        t = self.branch
        return tau, t, (1.0 + t) ** 2, tau >= t

    def value(self, tau):
        tau, t, c, quad = self._split(tau)
        out = np.empty_like(tau)
        out[quad] = tau[quad] + 0.5 * tau[quad] * tau[quad]
        lo = tau[~quad]
        out[~quad] = -c * np.log((1.0 + 2.0 * t - lo) / (1.0 + t)) + t + 0.5 * t * t
        return _scalar_or_array(out)

    def deriv(self, tau):
        tau, t, c, quad = self._split(tau)
        out = np.empty_like(tau)
        out[quad] = 1.0 + tau[quad]
        out[~quad] = c / (1.0 + 2.0 * t - tau[~quad])
        return _scalar_or_array(out)

    def deriv2(self, tau):
        tau, t, c, quad = self._split(tau)
        out = np.empty_like(tau)
        out[quad] = 1.0
        out[~quad] = c / (1.0 + 2.0 * t - tau[~quad]) ** 2
        return _scalar_or_array(out)
