"""Shared pytest configuration.

`-m gpu` tests need a B200 (they call the CUDA path through the C-ABI
library); everything else runs on CPU.  The CPU oracle (`oracle/`) is test
infrastructure: tests use it only as the checker.
"""

from __future__ import annotations

import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")
    config.addinivalue_line("markers", "slow: long-running CPU oracle work")


@pytest.fixture(scope="session")
def problems():
    """Memoised oracle problem builder (configs and small ad-hoc instances)."""
    from oracle.mesh2d import build_config, build_problem2d

    cache = {}

    def get(key, *args):
        k = (key,) + tuple(args)
        if k not in cache:
            cache[k] = build_config(key) if not args else build_problem2d(key, *args)
        return cache[k]

    return get
