"""Structured 2D Q1 problem hierarchies (host-side setup, product path).

The reference builds 3D box hierarchies in `mesh.py` (`build_problem`
:216-239, `_build_level` :247-287, `_interpolation` :290-332).  The tier's
configurations are 2D bilinear-Q1 plane-stress grids:

* level k (1-based) of a coarse grid mx x my has (mx 2^(k-1)) x (my 2^(k-1))
  unit squares, nodes and elements numbered x-fastest;
* Dirichlet data per dof (cantilever: left edge clamped; MBB half-beam: u_x = 0
  on the left edge and u_y = 0 at the bottom-right node; bridge: both bottom
  corners pinned); free dofs numbered node-major, x then y;
* unit downward load: cantilever at the right-edge mid node(s), MBB at the
  top-left node, bridge spread evenly over the top edge.

Transfers between levels are implicit in the structure (bilinear
interpolation with Dirichlet endpoints dropped, mesh.py:290-332); the device
kernels apply them without storing P.  `StructuredTransfer` stands in for the
reference's `transfers[k]` CSR matrices in the API.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

FAMILIES = ("cantilever", "mbb", "bridge")
_TAG = {"cantilever": "CANT2D", "mbb": "MBB2D", "bridge": "BRIDGE2D"}

# BASELINE.json configs (family, coarse mx, coarse my, levels, V / m)
CONFIGS = {
    "C1": ("cantilever", 16, 8, 3, 0.5),  # 64 x 32
    "C2": ("mbb", 8, 4, 6, 0.4),  # 256 x 128
    "C3": ("cantilever", 4, 2, 9, 0.5),  # 1024 x 512 operator microbench
    "C4": ("cantilever", 4, 2, 9, 0.5),  # 1024 x 512 full PBM
    "C5": ("bridge", 4, 2, 10, 0.3),  # 2048 x 1024 full PBM
}


def _dirichlet(family: str, ex: int, ey: int) -> np.ndarray:
    nx, ny = ex + 1, ey + 1
    fixed = np.zeros((ny, nx, 2), dtype=bool)
    if family == "cantilever":
        fixed[:, 0, :] = True
    elif family == "mbb":
        fixed[:, 0, 0] = True
        fixed[0, ex, 1] = True
    elif family == "bridge":
        fixed[0, 0, :] = True
        fixed[0, ex, :] = True
    else:
        raise ValueError(f"unknown problem family {family!r}")
    return fixed.reshape(nx * ny, 2)


def _load_nodes(family: str, ex: int, ey: int):
    nx = ex + 1
    if family == "cantilever":
        rows = sorted({ey // 2, (ey + 1) // 2})
        nodes = np.array([ex + nx * r for r in rows], dtype=np.int64)
    elif family == "mbb":
        nodes = np.array([nx * ey], dtype=np.int64)
    else:
        nodes = np.arange(nx * ey, nx * ey + nx, dtype=np.int64)
    return nodes, 1.0 / nodes.size


@dataclass
class MeshLevel:
    """One refinement level (MeshLevel, mesh.py:145-169, in 2D)."""

    index: int
    ex: int
    ey: int
    fixed: np.ndarray  # (n_nodes, 2) bool
    dof: np.ndarray  # (n_nodes, 2) int64 free index or -1
    n: int
    load: np.ndarray  # (n,) host copy of the load vector
    hierarchy: "Problem" = field(default=None, repr=False)

    @property
    def shape(self):
        return (self.ex, self.ey)

    @property
    def m(self) -> int:
        return self.ex * self.ey

    @property
    def nx(self) -> int:
        return self.ex + 1

    @property
    def ny(self) -> int:
        return self.ey + 1

    @property
    def n_nodes(self) -> int:
        return self.nx * self.ny

    @property
    def conn(self) -> np.ndarray:
        """(m, 4) corner node ids, (0,0),(1,0),(1,1),(0,1) (mesh.py:253-259)."""
        e = np.arange(self.m, dtype=np.int64)
        base = e % self.ex + self.nx * (e // self.ex)
        return base[:, None] + np.array([0, 1, self.nx + 1, self.nx])[None, :]


def _level(family: str, mx: int, my: int, k: int) -> MeshLevel:
    ex, ey = mx << (k - 1), my << (k - 1)
    fixed = _dirichlet(family, ex, ey)
    free = ~fixed
    n = int(free.sum())
    if n == 0:
        raise ValueError(f"level {k} has no free degrees of freedom")
    dof = np.full(fixed.shape, -1, dtype=np.int64)
    dof[free] = np.arange(n, dtype=np.int64)
    nodes, weight = _load_nodes(family, ex, ey)
    target = dof[nodes, 1]
    if np.any(target < 0):
        raise ValueError("a loaded dof is fixed; the instance is degenerate")
    load = np.zeros(n)
    np.add.at(load, target, -weight)
    return MeshLevel(k, ex, ey, fixed, dof, n, load)


@dataclass(frozen=True)
class StructuredTransfer:
    """Bilinear prolongation between consecutive levels (mesh.py:290-332).

    Never stored as a matrix: the device restriction/prolongation kernels
    evaluate it from the grid structure.  `shape` matches the reference's
    `transfers[k].shape` = (fine.n, coarse.n).
    """

    coarse: int  # 0-based level index
    fine: int
    shape: tuple


@dataclass
class Problem:
    """A named instance: hierarchy, transfers, load, volume (mesh.py:172-201)."""

    name: str
    family: str
    mx: int
    my: int
    levels: list
    transfers: list
    vol_frac: float
    volume: float = field(init=False)
    _f_dev: object = field(default=None, init=False, repr=False)

    def __post_init__(self) -> None:
        self.volume = self.vol_frac * self.fine.m
        for lv in self.levels:
            lv.hierarchy = self

    @property
    def fine(self) -> MeshLevel:
        return self.levels[-1]

    @property
    def m(self) -> int:
        return self.fine.m

    @property
    def n(self) -> int:
        return self.fine.n

    @property
    def f(self):
        """Finest load vector as a CUDA fp64 tensor (cached)."""
        if self._f_dev is None:
            import torch

            self._f_dev = torch.as_tensor(self.fine.load, dtype=torch.float64, device="cuda")
        return self._f_dev


def build_problem(family: str, mx: int | None = None, my: int | None = None, levels: int | None = None,
                  vol_frac: float | None = None):
    """A 2D Q1 hierarchy `build_problem(family, mx, my, levels, vol_frac)`, or the
    reference's own 3D instances by name: `build_problem("CANT-2-2-2-3",
    vol_frac=0.35, levels=None)` (mesh.py:216-239, mesh3d.build_hex_problem)."""
    if mx is None and isinstance(family, str) and "-" in family:
        from .mesh3d import build_hex_problem

        return build_hex_problem(family, vol_frac=0.35 if vol_frac is None else vol_frac, levels=levels)
    if family not in FAMILIES:
        raise ValueError(f"unknown problem family {family!r}")
    if mx is None or my is None or levels is None or vol_frac is None:
        raise ValueError("a 2D problem needs family, mx, my, levels and vol_frac")
    if min(mx, my, levels) < 1:
        raise ValueError("mx, my and levels must be positive integers")
    if not 0.0 < vol_frac < 1.0:
        raise ValueError(f"vol_frac must lie in (0, 1), got {vol_frac}")
    lv = [_level(family, mx, my, k) for k in range(1, levels + 1)]
    tr = [StructuredTransfer(k, k + 1, (lv[k + 1].n, lv[k].n)) for k in range(levels - 1)]
    return Problem(f"{_TAG[family]}-{mx}-{my}-{levels}", family, mx, my, lv, tr, vol_frac)


def build_config(key: str) -> Problem:
    return build_problem(*CONFIGS[key])
