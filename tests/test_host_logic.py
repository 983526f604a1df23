"""Host-side logic of the B200 package on CPU, checked against the oracle.

The package's Python layer mirrors the reference's interface (pbm.py,
linalg.py, multigrid.py, mesh.py): configuration defaults, the inner
tolerance policy, validation errors and the mesh / dof numbering that the
device layout is built from must be the oracle's exactly.  No device work.
"""

from __future__ import annotations

import dataclasses

import numpy as np
import pytest

import oracle
from oracle import mesh2d
import paper_1904_06556_b200 as vts
from paper_1904_06556_b200 import linalg, pbm, problem


def test_pbm_config_defaults_match_reference():
    ours = dataclasses.asdict(pbm.PbmConfig())
    ref = dataclasses.asdict(oracle.PbmConfig())
    assert ours == ref
    assert dataclasses.asdict(pbm.PbmConfig.large()) == dataclasses.asdict(oracle.PbmConfig.large())


@pytest.mark.parametrize("tol,iters", [(0.0, 1), (1.0, 1), (-1e-3, 1), (1e-3, -1)])
def test_minres_config_validation(tol, iters):
    with pytest.raises(ValueError):
        linalg.MinresConfig(tol=tol, max_iters=iters)
    with pytest.raises(ValueError):
        oracle.MinresConfig(tol=tol, max_iters=iters)


def test_stagnation_tolerance_matches_reference():
    rng = np.random.default_rng(3)
    for _ in range(20):
        a = linalg.StagnationTolerance(tol=10 ** rng.uniform(-4, -1))
        b = oracle.StagnationTolerance(tol=a.tol)
        r = 1.0
        for step in range(30):
            r *= rng.choice([0.5, 0.95, 1.1])
            a.observe(r)
            b.observe(r)
            assert a.current() == b.current()
            if step == 15:
                a.reset()
                b.reset()
        assert a.current() >= 1e-9


@pytest.mark.parametrize("key", ["C1", "C2", "C3"])
def test_mesh_numbering_matches_oracle(key):
    ours = problem.build_config(key)
    ref = mesh2d.build_config(key)
    assert len(ours.levels) == len(ref.levels)
    assert ours.n == ref.n and ours.m == ref.m
    assert ours.volume == ref.volume
    for a, b in zip(ours.levels, ref.levels):
        assert (a.ex, a.ey, a.n) == (b.ex, b.ey, b.n)
        np.testing.assert_array_equal(a.fixed, b.fixed)
        np.testing.assert_array_equal(a.dof, b.dof)
        np.testing.assert_array_equal(a.load, b.load)


@pytest.mark.parametrize("family,mx,my,levels,vf", [("cantilever", 4, 2, 3, 0.5), ("mbb", 4, 2, 3, 0.4),
                                                    ("bridge", 4, 2, 3, 0.3)])
def test_structured_transfers_match_oracle_interpolation(family, mx, my, levels, vf):
    """The device prolongation is the structured form of mesh.py:290-332's P;
    rebuild it densely from the host description and compare with the oracle's CSR."""
    ours = problem.build_problem(family, mx, my, levels, vf)
    ref = mesh2d.build_problem2d(family, mx, my, levels, vf)
    for k, P in enumerate(ref.transfers):
        c, f = ours.levels[k], ours.levels[k + 1]
        dense = np.zeros((f.n, c.n))
        for fy in range(f.ny):
            for fx in range(f.nx):
                xs = [(fx // 2, 1.0)] if fx % 2 == 0 else [(fx // 2, 0.5), (fx // 2 + 1, 0.5)]
                ys = [(fy // 2, 1.0)] if fy % 2 == 0 else [(fy // 2, 0.5), (fy // 2 + 1, 0.5)]
                for comp in range(2):
                    i = f.dof[fy * f.nx + fx, comp]
                    if i < 0:
                        continue
                    for cx, wx in xs:
                        for cy, wy in ys:
                            j = c.dof[cy * c.nx + cx, comp]
                            if j >= 0:
                                dense[i, j] += wx * wy
        np.testing.assert_array_equal(dense, P.toarray())


def test_quad_stiffness_matches_oracle():
    from oracle import fem2d

    from paper_1904_06556_b200 import fem

    np.testing.assert_allclose(fem.quad_stiffness(), fem2d.quad_stiffness(), rtol=0, atol=1e-15)
    ev = np.linalg.eigvalsh(fem.quad_stiffness())
    assert np.sum(np.abs(ev) < 1e-12) == 3  # rigid modes


def test_density_bounds_validation():
    with pytest.raises(ValueError):
        vts.DensityBounds.for_problem(10, 20.0, 0.0)  # volume above m * upper
