"""Validate the 2D discretisation glue before trusting it.

2D analogues of the reference's own invariants: `test_fem.py:25-57,77-218`
(stiffness symmetry/rank/rigid modes, scatter vs assembled matvec,
gather/scatter adjointness, bordered assembly vs dense) and
`test_mesh.py:43-162` (sizes, load resultant, transfer weights, adjointness,
constants preserved away from the clamped edge).  CPU only.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle.fem2d import ElementOps2D, quad_stiffness
from oracle.mesh2d import build_config, build_problem2d

CORNERS = np.array([(0, 0), (1, 0), (1, 1), (0, 1)], dtype=float)


def test_quad_stiffness_spectrum_and_rigid_modes():
    ke = quad_stiffness()
    np.testing.assert_array_equal(ke, ke.T)
    eig = np.linalg.eigvalsh(ke)
    assert np.sum(np.abs(eig) < 1e-12 * eig[-1]) == 3
    np.testing.assert_allclose(eig[3:], [0.4945, 0.4945, 0.7692, 0.7692, 1.4286], atol=1e-4)
    modes = [np.tile([1.0, 0.0], 4), np.tile([0.0, 1.0], 4),
             np.column_stack([-CORNERS[:, 1], CORNERS[:, 0]]).ravel()]
    for mode in modes:
        assert np.linalg.norm(ke @ mode) <= 1e-13


def test_quad_stiffness_scales_with_modulus_and_rejects_bad_input():
    np.testing.assert_allclose(quad_stiffness(e_mod=3.0), 3.0 * quad_stiffness(), rtol=1e-13)
    for kw in ({"nu": 0.5}, {"nu": -0.1}, {"e_mod": 0.0}):
        with pytest.raises(ValueError):
            quad_stiffness(**kw)


@pytest.mark.parametrize("key,n,m", [("C1", 4224, 2048), ("C2", 66176, 32768),
                                     ("C3", 1050624, 524288)])
def test_config_sizes_match_survey(key, n, m):
    prob = build_config(key)
    assert (prob.n, prob.m) == (n, m)


def test_c3_level_sizes_match_survey():
    prob = build_config("C3")
    assert [lv.n for lv in prob.levels] == [24, 80, 288, 1088, 4224, 16640, 66048, 263168, 1050624]


@pytest.mark.parametrize("family", ["cantilever", "mbb", "bridge"])
def test_load_resultant_and_fixed_counts(family):
    prob = build_problem2d(family, 4, 2, 3, 0.4)
    for lv in prob.levels:
        assert lv.load.sum() == pytest.approx(-1.0, abs=1e-14)
        assert lv.load[lv.dof[~lv.fixed.any(axis=1), 0]].sum() == 0.0
        fixed = {"cantilever": 2 * lv.ny, "mbb": lv.ny + 1, "bridge": 4}[family]
        assert lv.fixed.sum() == fixed
        assert lv.n == 2 * lv.n_nodes - fixed


@pytest.mark.parametrize("family", ["cantilever", "mbb", "bridge"])
def test_transfers_weights_and_adjointness(family):
    prob = build_problem2d(family, 4, 2, 4, 0.4)
    rng = np.random.default_rng(7)
    for coarse, fine, p in zip(prob.levels, prob.levels[1:], prob.transfers):
        assert p.shape == (fine.n, coarse.n)
        assert set(np.unique(p.data)).issubset({1.0, 0.5, 0.25})
        uc, uf = rng.standard_normal(coarse.n), rng.standard_normal(fine.n)
        assert (p @ uc) @ uf == pytest.approx(uc @ (p.T @ uf), rel=1e-13)
        colsq = np.asarray(p.multiply(p).sum(axis=0)).ravel()
        assert colsq.max() <= 9.0 / 4.0 + 1e-12


def test_prolongation_preserves_constants_away_from_clamped_edge():
    prob = build_problem2d("cantilever", 4, 2, 3, 0.5)
    coarse, fine = prob.levels[-2], prob.levels[-1]
    ones = prob.transfers[-1] @ np.ones(coarse.n)
    ix = np.arange(fine.n_nodes) % fine.nx
    inner = fine.dof[(ix >= 2)].ravel()
    np.testing.assert_allclose(ones[inner], 1.0, atol=1e-14)
    assert np.all(ones[fine.dof[ix == 1].ravel()] < 1.0)


@pytest.mark.parametrize("family", ["cantilever", "mbb", "bridge"])
def test_scatter_matches_assembled_matvec(family):
    prob = build_problem2d(family, 4, 2, 3, 0.4)
    ops = ElementOps2D(prob.fine)
    rng = np.random.default_rng(17)
    rho = rng.uniform(0.05, 1.0, prob.m)
    u = rng.standard_normal(prob.n)
    w, q = ops.element_products(u)
    via_matrix = ops.assemble_stiffness(rho) @ u
    np.testing.assert_allclose(ops.scatter(rho[:, None] * w), via_matrix, rtol=0,
                               atol=1e-12 * np.abs(via_matrix).max())
    assert q.sum() == pytest.approx(0.5 * u @ (ops.assemble_stiffness(np.ones(prob.m)) @ u), rel=1e-12)
    counts = np.diff(ops.assemble_stiffness(np.ones(prob.m)).indptr)
    assert counts.max() == 18  # 9-point node stencil x 2 components


def test_gather_scatter_adjoint_and_bordered_assembly():
    prob = build_problem2d("mbb", 2, 1, 3, 0.4)
    ops = ElementOps2D(prob.fine)
    rng = np.random.default_rng(31)
    u = rng.standard_normal(prob.n)
    wr = rng.standard_normal((prob.m, 8))
    assert np.sum(ops.gather(u) * wr) == pytest.approx(u @ ops.scatter(wr), rel=1e-13)
    w, _ = ops.element_products(u)
    kc, r1 = rng.uniform(0.1, 1.0, prob.m), rng.uniform(0.01, 0.5, prob.m)
    mat = ops.assemble(kc, r1, w, border_sign=-1.0)
    dense = np.zeros((prob.n + 1, prob.n + 1))
    dense[:-1, :-1] = ops.assemble_stiffness(kc).toarray()
    for i in range(prob.m):
        v = np.zeros(prob.n + 1)
        sel = ops.edof[i] < prob.n
        v[ops.edof[i][sel]] = w[i][sel]
        v[-1] = -1.0
        dense += r1[i] * np.outer(v, v)
    np.testing.assert_allclose(mat.to_dense(), dense, rtol=0, atol=1e-12 * np.abs(dense).max())
