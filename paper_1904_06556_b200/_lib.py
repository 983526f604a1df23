"""ctypes binding of the in-tree C-ABI library `_build/libvts_b200.so`.

This is the reference-side stub INTEGRATION.md describes: every entry point of
`include/vts_b200.h` with its argument types, plus the status-code mapping to
the reference's exception classes (`linalg.py:107-115` MinresError,
`ValueError` for bad arguments).  There is no fallback: if the library is
missing or fails to load, importing the product path raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
# VTS_LIB overrides the library path (A/B comparisons of two builds; tools/checks)
LIB_PATH = os.environ.get("VTS_LIB") or os.path.join(_HERE, "_build", "libvts_b200.so")

VTS_OK = 0
VTS_E_INDEFINITE = 1
VTS_E_BREAKDOWN = 2
VTS_E_NONFINITE = 3
VTS_E_ARGUMENT = 4
VTS_E_CUDA = 5
VTS_E_CHOLESKY = 6
VTS_W_SATURATED = 1
VTS_W_SHIFTED = 2

_P = ctypes.c_void_p
_D = ctypes.c_double
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_PD = ctypes.POINTER(ctypes.c_double)
_PI32 = ctypes.POINTER(ctypes.c_int32)
_PI64 = ctypes.POINTER(ctypes.c_int64)
_PU32 = ctypes.POINTER(ctypes.c_uint32)

# name -> (restype, argtypes); mirrors include/vts_b200.h
SIGNATURES = {
    "vts_last_error": (ctypes.c_char_p, []),
    "vts_version": (ctypes.c_int, []),
    "vts_ctx_create": (ctypes.c_int, [ctypes.POINTER(_P), _I32, _PI32, _PI32, ctypes.POINTER(_PI64), _PD, _I64]),
    "vts_ctx_create3": (ctypes.c_int, [ctypes.POINTER(_P), _I32, _PI32, _PI32, _PI32, ctypes.POINTER(_PI64), _PD,
                                       _I64]),
    "vts_ctx_dim": (ctypes.c_int, [_P]),
    "vts_ctx_destroy": (ctypes.c_int, [_P]),
    "vts_ctx_sizes": (ctypes.c_int, [_P, _PI64, _PI64]),
    "vts_eval_lagrangian": (ctypes.c_int, [_P, _P, _D] + [_P] * 11 + [_D, _D, _D, _D] + [_P] * 11 + [_PD, _PU32]),
    "vts_schur_system": (ctypes.c_int, [_P, _P, _P, _D] + [_P] * 6 + [_P, _P, _P, _PD]),
    "vts_newton_apply": (ctypes.c_int, [_P, _P, _P]),
    "vts_mg_setup": (ctypes.c_int, [_P, _D, _PI32]),
    "vts_vcycle": (ctypes.c_int, [_P, _P, _P]),
    "vts_level_apply": (ctypes.c_int, [_P, _I32, _P, _P]),
    "vts_level_size": (ctypes.c_int, [_P, _I32, _PI64]),
    "vts_minres": (ctypes.c_int, [_P, _P, _P, _D, _I32, _D, _I32, _PI32, _PD, _PI32, _PD]),
    "vts_reconstruct_nu": (ctypes.c_int, [_P, _P, _P, _D, _P, _D] + [_P] * 5 + [_P, _P, _PD]),
    "vts_al_value": (ctypes.c_int, [_P, _P, _D, _P, _P, _P, _D, _P, _P, _D] + [_P] * 9 + [_D, _D, _PD, _PU32]),
    "vts_axpy": (ctypes.c_int, [_P, _I64, _D, _P, _P]),
    "vts_outer_update": (ctypes.c_int, [_P, _D, _D, _D] + [_P] * 9 + [_I32]),
    "vts_gap": (ctypes.c_int, [_P, _P, _D] + [_P] * 6 + [_D, _P, _PD, _PD, _PD, _PD]),
    "vts_penalty_eval": (ctypes.c_int, [_P, _I64, _P, _D, _P, _P, _P, _PU32]),
    "vts_time_kernels": (ctypes.c_int, [_P, _I32, _PD]),
    "vts_time_cold": (ctypes.c_int, [_P, _I32, _P, ctypes.c_int64, _PD]),
    "vts_ip_residual": (ctypes.c_int, [_P, _P, _D, _P, _P, _P, _D, _D, _P, _P, _D, _P, _D, _P, _P, _P, _P, _P, _PD]),
    "vts_ip_schur_system": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _D, _P, _P, _P, _PD]),
    "vts_ip_reconstruct": (ctypes.c_int, [_P, _P, _P, _D, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "vts_ip_step_bounds": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _PD]),
    "vts_debug_smooth": (ctypes.c_int, [_P, _I32, _I32, _I32, _P, _P]),
    "vts_minres_warm": (ctypes.c_int, [_P, _P, _P, _P, _D, _I32, _D, _I32, _PI32, _PD, _PI32, _PD]),
    "vts_minres_generic": (ctypes.c_int, [_P, _I64, _P, _P, _P, _D, _I32, _D, _P, _P, _P, _PI32, _PD, _PI32, _PD]),
    "vts_bind_stiffness": (ctypes.c_int, [_P, _P, _PU32]),
    "vts_element_products": (ctypes.c_int, [_P, _P, _P, _P]),
    "vts_doc_update": (ctypes.c_int, [_P, _P, _P, _D, _D, _D, _P, _P, _P]),
    "vts_doc_bisect": (ctypes.c_int, [_P, _P, _P, _D, _P, _P, _D, _D, _D, _D, _I32, _P, _PD, _PI32]),
    "vts_doc_measure": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _D, _PD]),
    "vts_kernel_launches": (ctypes.c_int64, [_P]),
    "vts_profile_begin": (ctypes.c_int, [_P]),
    "vts_profile_end": (ctypes.c_int, [_P, _PD]),
}


class NewtonStepArgs(ctypes.Structure):
    """vts_newton_step_args (include/vts_b200.h): device pointers, scalars, controls."""

    _fields_ = ([("u", _P), ("nu_lo", _P), ("nu_up", _P), ("alpha", _D)]
                + [(k, _P) for k in ("rho", "p", "mu_lo", "mu_up", "q_lo", "q_up", "f", "lower", "upper")]
                + [(k, _D) for k in ("volume", "norm_f", "norm_bounds", "branch")]
                + [(k, _P) for k in ("res_u", "res_lo", "res_up", "q", "mu_hat_lo", "mu_hat_up", "a", "b_lo", "b_up",
                                     "rho_hat")]
                + [("value", _D), ("res_alpha", _D)]
                + [(k, _P) for k in ("chat", "rhs", "border", "du", "dnu_lo", "dnu_up")]
                + [("minres_tol", _D), ("minres_floor", _D), ("minres_cap", _I32), ("armijo_c1", _D),
                   ("armijo_shrink", _D), ("armijo_max_halvings", _I32), ("shift_scale", _D)])


class NewtonStepResult(ctypes.Structure):
    """vts_newton_step_result (include/vts_b200.h)."""

    _fields_ = [("status", _I32), ("minres_iterations", _I32), ("minres_converged", _I32), ("minres_relres", _D),
                ("kappa", _D), ("slope", _D), ("dalpha", _D), ("alpha", _D), ("scalars", _D * 8),
                ("warnings", ctypes.c_uint32), ("trials", _I32), ("host_syncs", _I32), ("graphs", _I32)]


SIGNATURES["vts_newton_step"] = (ctypes.c_int, [_P, ctypes.POINTER(NewtonStepArgs), ctypes.POINTER(NewtonStepResult)])

# int (*vts_apply_fn)(void* user, const double* in, double* out): device vectors
APPLY_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)

_lib = None


def build(force: bool = False) -> str:
    """Compile the library in-tree with nvcc for sm_100a (see Makefile)."""
    cmd = ["make", "-s", "-C", _HERE]
    if force:
        subprocess.run(["make", "-s", "-C", _HERE, "clean"], check=True)
    subprocess.run(cmd, check=True)
    return LIB_PATH


def load():
    """Load the library; raises if it is missing (no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `make -C {_HERE}` "
            "(or __graft_entry__.build()); the B200 path has no fallback"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class VtsError(RuntimeError):
    """CUDA failure or internal error inside the library."""


def last_error() -> str:
    return load().vts_last_error().decode("utf-8", "replace")


def check(rc: int, where: str) -> None:
    if rc == VTS_OK:
        return
    msg = last_error()
    if rc == VTS_E_ARGUMENT:
        raise ValueError(f"{where}: {msg}")
    raise VtsError(f"{where} failed (code {rc}): {msg}")
