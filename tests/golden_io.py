"""Loading helpers for the committed golden fixtures (tests/golden/*.npz)."""

from __future__ import annotations

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# fixture name -> oracle problem arguments (family, mx, my, levels, vol_frac)
KERNEL_FIXTURES = {
    "c1_random_state": ("cantilever", 16, 8, 3, 0.5),
    "c1_microbench_state": ("cantilever", 16, 8, 3, 0.5),
    "mbb32_random_state": ("mbb", 4, 2, 4, 0.4),
    "bridge32_random_state": ("bridge", 4, 2, 4, 0.3),
}

STATE_KEYS = ("u", "alpha", "nu_lo", "nu_up", "rho", "mu_lo", "mu_up", "p", "q_lo", "q_up")


def load(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def state_dict(fx: dict) -> dict:
    out = {k: fx["st_" + k] for k in STATE_KEYS}
    out["alpha"] = float(out["alpha"])
    return out
