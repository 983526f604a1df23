"""The C-ABI boundary on CPU: the library loads and exports exactly what
include/vts_b200.h declares; argument validation and the status-code mapping
work without a GPU (no compute calls are made here).

The reference has no FFI layer; the boundary replaces the
Python call signatures of pbm.py / linalg.py / multigrid.py, and the error
contract mirrors linalg.py:107-115 (MinresError) and the reference's
ValueError validation (fem.py:39-47).
"""

from __future__ import annotations

import ctypes
import os
import re
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "vts_b200.h")
DECL = re.compile(r"^(?:int|int64_t|const char\s*\*)\s*(vts_\w+)\(", re.M)


def header_symbols() -> set[str]:
    with open(HEADER) as fh:
        return set(DECL.findall(fh.read()))


@pytest.fixture(scope="module")
def lib():
    from paper_1904_06556_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        _lib.build()
    return _lib.load()


def test_header_declares_the_boundary():
    syms = header_symbols()
    # the SURVEY §8(b) contract, by function
    for name in ("vts_ctx_create", "vts_ctx_destroy", "vts_eval_lagrangian", "vts_al_value", "vts_newton_apply",
                 "vts_mg_setup", "vts_vcycle", "vts_minres", "vts_reconstruct_nu", "vts_outer_update",
                 "vts_last_error"):
        assert name in syms, name


def test_bindings_match_header():
    from paper_1904_06556_b200 import _lib

    assert set(_lib.SIGNATURES) == header_symbols()


def test_library_exports_every_declared_symbol(lib):
    from paper_1904_06556_b200 import _lib

    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True, check=True)
    exported = {ln.split()[-1] for ln in out.stdout.splitlines() if " T " in ln}
    missing = header_symbols() - exported
    assert not missing, missing
    for name in header_symbols():
        assert getattr(lib, name) is not None


def test_library_is_sm100a_only():
    from paper_1904_06556_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_\w+", out.stdout))
    assert archs == {"sm_100a"}, archs


def test_version_and_error_plumbing(lib):
    assert lib.vts_version() >= 1
    # NULL context -> argument error with a message, no CUDA call
    rc = lib.vts_newton_apply(None, None, None)
    assert rc == 4
    assert b"ctx" in lib.vts_last_error().lower() or len(lib.vts_last_error()) > 0
    assert lib.vts_ctx_destroy(None) in (0, 4)
    assert lib.vts_kernel_launches(None) == 0
    assert lib.vts_profile_begin(None) == 4
    out = (ctypes.c_double * 4)()
    assert lib.vts_profile_end(None, out) == 4


def test_create_rejects_bad_arguments(lib):
    h = ctypes.c_void_p()
    ex = (ctypes.c_int32 * 1)(4)
    ey = (ctypes.c_int32 * 1)(2)
    # zero levels / NULL out pointer are argument errors before any device work
    assert lib.vts_ctx_create(ctypes.byref(h), 0, ex, ey, None, None, 0) == 4
    assert lib.vts_ctx_create(None, 1, ex, ey, None, None, 0) == 4


def test_status_codes_map_to_reference_exceptions():
    from paper_1904_06556_b200 import _lib, linalg

    with pytest.raises(ValueError):
        _lib.check(_lib.VTS_E_ARGUMENT, "probe")
    with pytest.raises(_lib.VtsError):
        _lib.check(_lib.VTS_E_CUDA, "probe")
    _lib.check(_lib.VTS_OK, "probe")
    # MINRES failures surface as the reference's MinresError (linalg.py:107-115)
    assert issubclass(linalg.MinresError, RuntimeError) or issubclass(linalg.MinresError, Exception)


def test_product_path_has_no_fallback(monkeypatch, tmp_path):
    """With the library missing, loading raises instead of falling back to CPU."""
    from paper_1904_06556_b200 import _lib

    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(RuntimeError, match="no fallback"):
        _lib.load()


def test_product_package_does_not_import_the_oracle():
    """The shipped package never routes through oracle/ (test infrastructure)."""
    pkg = os.path.join(REPO, "paper_1904_06556_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                with open(os.path.join(root, f)) as fh:
                    src = fh.read()
                assert not re.search(r"^\s*(import oracle|from oracle)", src, re.M), f
