"""Structured 2D Q1 mesh hierarchies (oracle side; test infrastructure only).

2D restatement of the reference's mesh module:

* level k (1-based) of a coarse grid mx x my has (mx 2^(k-1)) x (my 2^(k-1))
  unit-square elements; nodes are numbered x-fastest, elements likewise
  (reference `mesh.py:247-259`, first four corners of `_CORNERS`
  `mesh.py:47-51`);
* Dirichlet data is per *dof* (the MBB half-beam fixes single components),
  generalising the per-node mask of `mesh.py:90-103,261-267`; free dofs are
  numbered node-major, component-minor (x then y), skipping fixed dofs
  (`mesh.py:266-267`);
* every level carries its own load vector (`mesh.py:269-276`); only the
  finest one is used by PBM (`mesh.py:199-201`);
* the bilinear interpolation between consecutive levels drops every entry
  whose fine or coarse endpoint is fixed (`mesh.py:290-332`, weights
  {1, 1/2, 1/4} in 2D); restriction is its transpose (`mesh.py:335-342`).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

FAMILIES = ("cantilever", "mbb", "bridge")
_TAG = {"cantilever": "CANT2D", "mbb": "MBB2D", "bridge": "BRIDGE2D"}


def fixed_dof_mask(family: str, ex: int, ey: int) -> np.ndarray:
    """(n_nodes, 2) boolean mask of Dirichlet dofs on an ex x ey grid."""
    nx, ny = ex + 1, ey + 1
    mask = np.zeros((nx * ny, 2), dtype=bool)
    ix = np.arange(nx * ny) % nx
    if family == "cantilever":
        mask[ix == 0, :] = True  # whole left edge clamped
    elif family == "mbb":
        mask[ix == 0, 0] = True  # symmetry line: u_x = 0
        mask[ex, 1] = True  # roller at the bottom-right corner node (ex, 0)
    elif family == "bridge":
        mask[0, :] = True  # (0, 0) pinned
        mask[ex, :] = True  # (ex, 0) pinned
    else:
        raise ValueError(f"unknown problem family {family!r}")
    return mask


def load_entries(family: str, ex: int, ey: int) -> tuple[np.ndarray, np.ndarray]:
    """Node ids and -y weights of the unit load (total resultant (0, -1))."""
    nx = ex + 1
    if family == "cantilever":
        ys = np.unique([ey // 2, (ey + 1) // 2])
        ids = ex + nx * ys
    elif family == "mbb":
        ids = np.array([nx * ey])  # top-left node (0, ey)
    elif family == "bridge":
        ids = nx * ey + np.arange(nx)  # every top-edge node
    else:
        raise ValueError(f"unknown problem family {family!r}")
    ids = np.asarray(ids, dtype=np.int64)
    return ids, np.full(ids.size, 1.0 / ids.size)


@dataclass
class Level2D:
    """One refinement level: connectivity, dof numbering and load vector."""

    index: int  # 1-based, 1 = coarsest
    ex: int
    ey: int
    conn: np.ndarray  # (m, 4) node ids, corners (0,0),(1,0),(1,1),(0,1)
    fixed: np.ndarray  # (n_nodes, 2) bool
    dof: np.ndarray  # (n_nodes, 2) free-dof index or -1
    n: int
    load: np.ndarray  # (n,)

    @property
    def m(self) -> int:
        return self.conn.shape[0]

    @property
    def nx(self) -> int:
        return self.ex + 1

    @property
    def ny(self) -> int:
        return self.ey + 1

    @property
    def n_nodes(self) -> int:
        return self.nx * self.ny


def build_level(family: str, mx: int, my: int, k: int) -> Level2D:
    s = 2 ** (k - 1)
    ex, ey = mx * s, my * s
    nx = ex + 1
    m = ex * ey
    e = np.arange(m, dtype=np.int64)
    base = (e % ex) + nx * (e // ex)
    conn = base[:, None] + np.array([0, 1, nx + 1, nx], dtype=np.int64)[None, :]

    fixed = fixed_dof_mask(family, ex, ey)
    n = int((~fixed).sum())
    if n == 0:
        raise ValueError(f"level {k} has no free degrees of freedom")
    dof = np.full(fixed.shape, -1, dtype=np.int64)
    dof[~fixed] = np.arange(n, dtype=np.int64)  # C order: node-major, x then y

    ids, wts = load_entries(family, ex, ey)
    ydofs = dof[ids, 1]
    if np.any(ydofs < 0):
        raise ValueError("a loaded dof is fixed; the instance is degenerate")
    load = np.zeros(n)
    np.add.at(load, ydofs, -wts)
    return Level2D(k, ex, ey, conn, fixed, dof, n, load)


def interpolation2d(coarse: Level2D, fine: Level2D) -> sp.csr_matrix:
    """Bilinear prolongation (fine.n x coarse.n), fixed endpoints dropped."""
    ids = np.arange(fine.n_nodes, dtype=np.int64)
    fx, fy = ids % fine.nx, ids // fine.nx
    odd_x, odd_y = (fx & 1) == 1, (fy & 1) == 1
    weight = np.where(odd_x, 0.5, 1.0) * np.where(odd_y, 0.5, 1.0)
    r_all, c_all, v_all = [], [], []
    for dy in (0, 1):
        for dx in (0, 1):
            ok = (odd_x | (dx == 0)) & (odd_y | (dy == 0))
            cx = np.where(odd_x, (fx - 1) // 2 + dx, fx // 2)
            cy = np.where(odd_y, (fy - 1) // 2 + dy, fy // 2)
            parent = cx + coarse.nx * cy
            f_sel, c_sel = ids[ok], parent[ok]
            for comp in (0, 1):
                r = fine.dof[f_sel, comp]
                c = coarse.dof[c_sel, comp]
                keep = (r >= 0) & (c >= 0)
                r_all.append(r[keep])
                c_all.append(c[keep])
                v_all.append(weight[f_sel][keep])
    p = sp.csr_matrix(
        (np.concatenate(v_all), (np.concatenate(r_all), np.concatenate(c_all))),
        shape=(fine.n, coarse.n),
    )
    p.sum_duplicates()
    return p


@dataclass
class Problem2D:
    """Named instance: hierarchy, transfers, load and volume budget."""

    name: str
    family: str
    mx: int
    my: int
    levels: list
    transfers: list  # transfers[k] maps levels[k] -> levels[k+1]
    vol_frac: float
    volume: float = field(init=False)

    def __post_init__(self) -> None:
        self.volume = self.vol_frac * self.fine.m

    @property
    def fine(self) -> Level2D:
        return self.levels[-1]

    @property
    def m(self) -> int:
        return self.fine.m

    @property
    def n(self) -> int:
        return self.fine.n

    @property
    def f(self) -> np.ndarray:
        return self.fine.load


def build_problem2d(family: str, mx: int, my: int, levels: int, vol_frac: float) -> Problem2D:
    if family not in FAMILIES:
        raise ValueError(f"unknown problem family {family!r}")
    if min(mx, my, levels) < 1:
        raise ValueError("mx, my and levels must be positive")
    if not 0.0 < vol_frac < 1.0:
        raise ValueError(f"vol_frac must lie in (0, 1), got {vol_frac}")
    lv = [build_level(family, mx, my, k) for k in range(1, levels + 1)]
    tr = [interpolation2d(lv[k], lv[k + 1]) for k in range(levels - 1)]
    name = f"{_TAG[family]}-{mx}-{my}-{levels}"
    return Problem2D(name, family, mx, my, lv, tr, vol_frac)


# BASELINE.json configs: family, coarse grid, levels, V/m
CONFIGS = {
    "C1": ("cantilever", 16, 8, 3, 0.5),  # 64 x 32
    "C2": ("mbb", 8, 4, 6, 0.4),  # 256 x 128
    "C3": ("cantilever", 4, 2, 9, 0.5),  # 1024 x 512 operator microbench
    "C4": ("cantilever", 4, 2, 9, 0.5),  # 1024 x 512 full PBM
    "C5": ("bridge", 4, 2, 10, 0.3),  # 2048 x 1024 full PBM
}


def build_config(key: str) -> Problem2D:
    family, mx, my, levels, vf = CONFIGS[key]
    return build_problem2d(family, mx, my, levels, vf)
