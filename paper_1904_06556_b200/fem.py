"""Q1 element data, density bounds and the device context (`ElementOps`).

* `quad_stiffness` — 8x8 plane-stress stiffness of the unit square by 2x2 Gauss
  quadrature, symmetrised (2D counterpart of `hex_stiffness`, fem.py:31-97);
  host-side setup, uploaded once into the context's constant memory.
* `DensityBounds` — `fem.py:100-116`, with CUDA tensors.
* `ElementOps` — the reference's per-level element plumbing (`fem.py:142-219`)
  is, on B200, a handle to a C-ABI context (`vts_ctx`) over the whole level
  hierarchy: grid layouts, free-dof maps, the bound Newton matrix and the
  multigrid workspace live on the device.  Construct it from the finest
  `MeshLevel` exactly like the reference (`ElementOps(problem.fine)`).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


def quad_stiffness(e_mod: float = 1.0, nu: float = 0.3) -> np.ndarray:
    if e_mod <= 0.0:
        raise ValueError("Young's modulus must be positive")
    if not 0.0 <= nu < 0.5:
        raise ValueError(f"Poisson ratio must lie in [0, 0.5), got {nu}")
    d = (e_mod / (1.0 - nu * nu)) * np.array([[1.0, nu, 0.0], [nu, 1.0, 0.0], [0.0, 0.0, 0.5 * (1.0 - nu)]])
    g = 1.0 / np.sqrt(3.0)
    jac = 0.5
    xi_c = np.array([-1.0, 1.0, 1.0, -1.0])
    eta_c = np.array([-1.0, -1.0, 1.0, 1.0])
    k = np.zeros((8, 8))
    for eta in (-g, g):
        for xi in (-g, g):
            dxi = 0.25 * xi_c * (1.0 + eta_c * eta) / jac
            deta = 0.25 * eta_c * (1.0 + xi_c * xi) / jac
            b = np.zeros((3, 8))
            b[0, 0::2] = dxi
            b[1, 1::2] = deta
            b[2, 0::2] = deta
            b[2, 1::2] = dxi
            k += (jac * jac) * (b.T @ d @ b)
    return 0.5 * (k + k.T)


def as_dev(x, name: str = "array") -> torch.Tensor:
    """fp64 contiguous CUDA tensor view/copy of `x` (host arrays are uploaded)."""
    t = torch.as_tensor(x, dtype=torch.float64)
    if not t.is_cuda:
        t = t.to("cuda")
    if not t.is_contiguous():
        t = t.contiguous()
    return t


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


@dataclass(frozen=True)
class DensityBounds:
    """Density box and volume budget (fem.py:100-116)."""

    lower: torch.Tensor
    upper: torch.Tensor
    volume: float
    norm: float  # ||lower|| + ||upper||, the tau_res weight (pbm.py:181)

    @classmethod
    def for_problem(cls, m: int, volume: float, rho_lower: float) -> "DensityBounds":
        lo = np.full(m, rho_lower)
        up = np.ones(m)
        if np.any(lo < 0.0) or np.any(up <= lo):
            raise ValueError("density bounds must satisfy 0 <= lower < upper")
        if not lo.sum() <= volume <= up.sum():
            raise ValueError("volume budget is outside the density box")
        return cls(as_dev(lo), as_dev(up), volume, float(np.linalg.norm(lo) + np.linalg.norm(up)))


class ElementOps:
    """Device context over a level hierarchy (stands in for fem.ElementOps)."""

    def __init__(self, level, e_mod: float = 1.0, nu: float = 0.3, stream: torch.cuda.Stream | None = None):
        hier = getattr(level, "hierarchy", None)
        if hier is None or hier.fine is not level:
            raise ValueError("ElementOps needs the finest MeshLevel of a build_problem hierarchy")
        from .mesh3d import HexLevel, hex_stiffness

        self.level = level
        self.problem = hier
        self.n = level.n
        self.m = level.m
        self.dim = 3 if isinstance(level, HexLevel) else 2
        self.nodes_per_elem = 8 if self.dim == 3 else 4
        self.dofs_per_elem = self.dim * self.nodes_per_elem  # 24 (fem.py:154) or 8
        # K_e of the finest level (the only one PBM uses; coarse operators are Galerkin)
        self.ke = hex_stiffness(e_mod, nu, level.edge) if self.dim == 3 else quad_stiffness(e_mod, nu)
        self._lib = _lib.load()
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        levels = hier.levels
        nl = len(levels)
        ex = (ctypes.c_int32 * nl)(*[lv.ex for lv in levels])
        ey = (ctypes.c_int32 * nl)(*[lv.ey for lv in levels])
        self._dofs = [np.ascontiguousarray(lv.dof.reshape(-1), dtype=np.int64) for lv in levels]
        maps = (ctypes.POINTER(ctypes.c_int64) * nl)(
            *[d.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)) for d in self._dofs]
        )
        ke = np.ascontiguousarray(self.ke, dtype=np.float64)
        kep = ke.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        handle = ctypes.c_void_p()
        if self.dim == 3:
            ez = (ctypes.c_int32 * nl)(*[lv.ez for lv in levels])
            rc = self._lib.vts_ctx_create3(ctypes.byref(handle), nl, ex, ey, ez, maps, kep, self.stream.cuda_stream)
        else:
            rc = self._lib.vts_ctx_create(ctypes.byref(handle), nl, ex, ey, maps, kep, self.stream.cuda_stream)
        _lib.check(rc, "vts_ctx_create3" if self.dim == 3 else "vts_ctx_create")
        self.handle = handle
        self.norm_f = float(np.linalg.norm(level.load))
        self._level_n = [lv.n for lv in levels]

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.vts_ctx_destroy(h)
            except Exception:
                pass
            self.handle = None

    @property
    def kernel_launches(self) -> int:
        return int(self._lib.vts_kernel_launches(self.handle))

    def level_size(self, k: int) -> int:
        return self._level_n[k]

    def vec(self, size: int) -> torch.Tensor:
        return torch.empty(size, dtype=torch.float64, device="cuda")

    # -- element-vector plumbing and assembly (fem.py:175-180, 211-219) --------------

    def element_products(self, u) -> tuple[torch.Tensor, torch.Tensor]:
        """Per-element w_e = u_e K_e (m x 8, local frame) and q_e = u_e . w_e / 2 (fem.py:175-180)."""
        u = self.check_vec(u, self.n, "u")
        w = torch.empty((self.m, self.dofs_per_elem), dtype=torch.float64, device="cuda")
        q = self.vec(self.m)
        _lib.check(self._lib.vts_element_products(self.handle, ptr(u), ptr(w), ptr(q)), "vts_element_products")
        return w, q

    def assemble_stiffness(self, rho):
        """K(rho) = sum_e rho_e K_e on the free dofs (fem.py:211-219), bound matrix-free
        in this context (it supersedes the context's previous system)."""
        import warnings

        from .linalg import StiffnessMatrix

        rho = self.check_vec(rho, self.m, "rho")
        flags = ctypes.c_uint32(0)
        _lib.check(self._lib.vts_bind_stiffness(self.handle, ptr(rho), ctypes.byref(flags)), "vts_bind_stiffness")
        if flags.value & 1:
            warnings.warn("assembling K(rho) with negative densities; the operator may be indefinite",
                          RuntimeWarning, stacklevel=2)
        self._system_version = getattr(self, "_system_version", 0) + 1
        return StiffnessMatrix(self, self._system_version)

    _scratch = None

    @classmethod
    def scratch(cls) -> "ElementOps":
        """A minimal context (one 1x1 cantilever level) for solves that bind no mesh:
        minres_solve on a user operator needs only its device scratch and stream."""
        if cls._scratch is None:
            from .problem import build_problem

            cls._scratch = cls(build_problem("cantilever", 1, 1, 1, 0.5).fine)
        return cls._scratch

    def check_vec(self, t: torch.Tensor, size: int, name: str) -> torch.Tensor:
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
            raise TypeError(f"{name} must be a contiguous CUDA float64 tensor")
        if t.numel() != size:
            raise ValueError(f"{name} has {t.numel()} entries, expected {size}")
        return t
