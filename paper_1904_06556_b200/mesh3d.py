"""Nested hexahedral hierarchies: the reference's own 3D instances.

Host-side restatement of the reference's `mesh.py` (the package's 3D
discretisation), so the unmodified reference is the oracle with no glue:

* instance names `CANT-mx-my-mz-L` / `BRIDGE-mx-my-mz-L` (mesh.py:43,
  204-213); level k (1-based) has (mx, my, mz) * 2^(k-1) elements of edge
  2^(1-k) (mesh.py:59-77); nodes and elements x fastest, then y, then z;
  element corners in VTK order (mesh.py:47-56);
* cantilever: the x = 0 face clamped, a -z load of total 1 split over the
  node(s) nearest the centre of the x = max face; bridge: the four bottom
  corner nodes pinned, the load spread over a centred top-face element patch
  of about half the span per axis (mesh.py:80-142);
* whole nodes are fixed (all three dofs); free dofs numbered node-major,
  x, y, z (mesh.py:261-267);
* transfers are trilinear with weights {1, 1/2, 1/4, 1/8}, Dirichlet
  endpoints dropped (mesh.py:290-332); like the 2D path they are never stored:
  the device kernels apply them from the grid structure.

The element stiffness is `hex_stiffness` (fem.py:31-97) restated: 2x2x2 Gauss,
isotropic D from (lambda, mu), symmetrised, linear in the edge length.
"""

from __future__ import annotations

import re
from dataclasses import dataclass, field

import numpy as np

from .problem import StructuredTransfer

__all__ = ["HexLevel", "HexProblem", "build_hex_problem", "parse_name", "hex_stiffness"]

_NAME = re.compile(r"^(CANT|BRIDGE)-(\d+)-(\d+)-(\d+)-(\d+)$", re.IGNORECASE)
CORNERS = ((0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1))


def hex_stiffness(e_mod: float = 1.0, nu: float = 0.3, edge: float = 1.0) -> np.ndarray:
    """24x24 stiffness of a cube of edge `edge` (the reference's fem.py:31-97)."""
    if edge <= 0.0:
        raise ValueError("edge length must be positive")
    if e_mod <= 0.0:
        raise ValueError("Young's modulus must be positive")
    if not 0.0 <= nu < 0.5:
        raise ValueError(f"Poisson ratio must lie in [0, 0.5), got {nu}")
    lam = e_mod * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    mu = e_mod / (2.0 * (1.0 + nu))
    dmat = np.diag([lam + 2 * mu] * 3 + [mu] * 3)
    dmat[:3, :3] += lam * (1.0 - np.eye(3))
    sgn = np.array([(2 * cx - 1, 2 * cy - 1, 2 * cz - 1) for cx, cy, cz in CORNERS], dtype=float)
    gp = 1.0 / np.sqrt(3.0)
    half = 0.5 * edge
    k = np.zeros((24, 24))
    for zeta in (-gp, gp):
        for eta in (-gp, gp):
            for xi in (-gp, gp):
                pt = (xi, eta, zeta)
                grads = np.empty((8, 3))
                for a in range(8):
                    s = sgn[a]
                    f = [1.0 + s[d] * pt[d] for d in range(3)]
                    grads[a] = [0.125 * s[0] * f[1] * f[2], 0.125 * s[1] * f[0] * f[2], 0.125 * s[2] * f[0] * f[1]]
                grads /= half
                bmat = np.zeros((6, 24))
                for a in range(8):
                    gx, gy, gz = grads[a]
                    col = 3 * a
                    bmat[0, col], bmat[1, col + 1], bmat[2, col + 2] = gx, gy, gz
                    bmat[3, col], bmat[3, col + 1] = gy, gx
                    bmat[4, col + 1], bmat[4, col + 2] = gz, gy
                    bmat[5, col], bmat[5, col + 2] = gz, gx
                k += half ** 3 * (bmat.T @ dmat @ bmat)
    return 0.5 * (k + k.T)


def _patch(n: int) -> int:
    """Loaded-patch extent along one axis (mesh.py:138-142)."""
    p = max(1, round(n / 2))
    if (n - p) % 2 == 1:
        p += 1
    return min(p, n)


def _fixed(family: str, ex: int, ey: int, ez: int) -> np.ndarray:
    nx, ny, nz = ex + 1, ey + 1, ez + 1
    fixed = np.zeros((nz, ny, nx), dtype=bool)
    if family == "cantilever":
        fixed[:, :, 0] = True
    else:
        for ix, iy in ((0, 0), (ex, 0), (0, ey), (ex, ey)):
            fixed[0, iy, ix] = True
    return fixed.reshape(-1)


def _loads(family: str, ex: int, ey: int, ez: int):
    nx, ny = ex + 1, ey + 1
    if family == "cantilever":
        ys = sorted({ey // 2, (ey + 1) // 2})
        zs = sorted({ez // 2, (ez + 1) // 2})
        ids = np.array([ex + nx * (y + ny * z) for y in ys for z in zs], dtype=np.int64)
        return ids, np.full(ids.size, 1.0 / ids.size)
    px, py = _patch(ex), _patch(ey)
    sx, sy = (ex - px) // 2, (ey - py) // 2
    quarter = 0.25 / (px * py)
    acc: dict = {}
    top = nx * ny * ez
    for i in range(sx, sx + px):
        for j in range(sy, sy + py):
            for dx, dy in ((0, 0), (1, 0), (0, 1), (1, 1)):
                node = top + (i + dx) + nx * (j + dy)
                acc[node] = acc.get(node, 0.0) + quarter
    ids = np.array(sorted(acc), dtype=np.int64)
    return ids, np.array([acc[int(i)] for i in ids])


@dataclass
class HexLevel:
    """One refinement level (the reference's MeshLevel, mesh.py:145-169)."""

    index: int
    ex: int
    ey: int
    ez: int
    edge: float
    fixed: np.ndarray  # (n_nodes,) whole-node Dirichlet mask
    dof: np.ndarray  # (n_nodes, 3) free index or -1
    n: int
    load: np.ndarray
    hierarchy: "HexProblem" = field(default=None, repr=False)

    @property
    def shape(self):
        return (self.ex, self.ey, self.ez)

    @property
    def m(self) -> int:
        return self.ex * self.ey * self.ez

    @property
    def node_shape(self):
        return (self.ex + 1, self.ey + 1, self.ez + 1)

    @property
    def n_nodes(self) -> int:
        return (self.ex + 1) * (self.ey + 1) * (self.ez + 1)

    @property
    def conn(self) -> np.ndarray:
        """(m, 8) corner node ids in VTK order (mesh.py:253-259)."""
        nx, ny = self.ex + 1, self.ey + 1
        e = np.arange(self.m, dtype=np.int64)
        base = e % self.ex + nx * ((e // self.ex) % self.ey + ny * (e // (self.ex * self.ey)))
        off = np.array([dx + nx * (dy + ny * dz) for dx, dy, dz in CORNERS], dtype=np.int64)
        return base[:, None] + off[None, :]


def _level(family: str, mx: int, my: int, mz: int, k: int) -> HexLevel:
    s = 1 << (k - 1)
    ex, ey, ez = mx * s, my * s, mz * s
    fixed = _fixed(family, ex, ey, ez)
    nfree_nodes = int((~fixed).sum())
    n = 3 * nfree_nodes
    if n == 0:
        raise ValueError(f"level {k} has no free degrees of freedom")
    dof = np.full((fixed.size, 3), -1, dtype=np.int64)
    dof[~fixed] = np.arange(n, dtype=np.int64).reshape(-1, 3)
    ids, weights = _loads(family, ex, ey, ez)
    zdof = dof[ids, 2]
    if np.any(zdof < 0):
        raise ValueError("a loaded node is fixed; the instance is degenerate")
    load = np.zeros(n)
    np.add.at(load, zdof, -weights)
    return HexLevel(k, ex, ey, ez, 2.0 ** (1 - k), fixed, dof, n, load)


@dataclass
class HexProblem:
    """A named 3D instance (the reference's Problem, mesh.py:172-201)."""

    name: str
    family: str
    mx: int
    my: int
    mz: int
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
    def fine(self) -> HexLevel:
        return self.levels[-1]

    @property
    def m(self) -> int:
        return self.fine.m

    @property
    def n(self) -> int:
        return self.fine.n

    @property
    def f(self):
        if self._f_dev is None:
            import torch

            self._f_dev = torch.as_tensor(self.fine.load, dtype=torch.float64, device="cuda")
        return self._f_dev


def parse_name(name: str):
    """`CANT-mx-my-mz-L` / `BRIDGE-mx-my-mz-L` (mesh.py:204-213)."""
    hit = _NAME.match(name.strip())
    if hit is None:
        raise ValueError(f"malformed problem name {name!r}; expected CANT-mx-my-mz-L or BRIDGE-mx-my-mz-L")
    family = "cantilever" if hit.group(1).upper() == "CANT" else "bridge"
    mx, my, mz, levels = (int(hit.group(i)) for i in range(2, 6))
    if min(mx, my, mz, levels) < 1:
        raise ValueError("mx, my, mz and the level count must be positive integers")
    return family, mx, my, mz, levels


def build_hex_problem(name: str, *, vol_frac: float = 0.35, levels: int | None = None) -> HexProblem:
    """The reference's `build_problem` (mesh.py:216-239) for 3D instance names."""
    family, mx, my, mz, nlev = parse_name(name)
    if levels is not None:
        nlev = int(levels)
    if not 0.0 < vol_frac < 1.0:
        raise ValueError(f"vol_frac must lie in (0, 1), got {vol_frac}")
    lv = [_level(family, mx, my, mz, k) for k in range(1, nlev + 1)]
    tr = [StructuredTransfer(k, k + 1, (lv[k + 1].n, lv[k].n)) for k in range(nlev - 1)]
    tag = "CANT" if family == "cantilever" else "BRIDGE"
    return HexProblem(f"{tag}-{mx}-{my}-{mz}-{nlev}", family, mx, my, mz, lv, tr, vol_frac)
