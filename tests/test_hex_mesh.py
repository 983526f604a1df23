"""CPU checks of the 3D hexahedral setup against the reference's own hierarchies.

`tests/golden/hex_mesh.npz` was written by the unmodified reference
(`make_golden_3d.py mesh`: `vtsopt.mesh.build_problem`, `fem.hex_stiffness`).
The package's host-side restatement (`paper_1904_06556_b200.mesh3d`) must
reproduce its dof numbering, loads, connectivity and volume exactly
(mesh.py:216-287), and its element stiffness to rounding (fem.py:31-97).
The trilinear transfer rule the device kernels apply (k3_restrict /
k3_prolong: weight 1/2 per odd fine coordinate, Dirichlet endpoints
dropped) is restated here and compared with the reference's P matrices
(mesh.py:290-332).
"""

from __future__ import annotations

import numpy as np
import pytest

from golden_io import load

from paper_1904_06556_b200 import mesh3d

NAMES = ("CANT-2-2-2-3", "BRIDGE-4-2-2-2", "CANT-3-1-2-2", "BRIDGE-3-3-2-2")


@pytest.fixture(scope="module")
def fx():
    return load("hex_mesh")


@pytest.mark.parametrize("name", NAMES)
def test_hierarchy_matches_reference(fx, name):
    prob = mesh3d.build_hex_problem(name)
    tag = name.replace("-", "_")
    assert prob.volume == float(fx[f"{tag}__volume"])
    for k, lv in enumerate(prob.levels):
        assert lv.shape == tuple(fx[f"{tag}__L{k}_shape"])
        np.testing.assert_array_equal(lv.dof, fx[f"{tag}__L{k}_dof"])
        np.testing.assert_array_equal(lv.load, fx[f"{tag}__L{k}_load"])
        np.testing.assert_array_equal(lv.conn, fx[f"{tag}__L{k}_conn"])


def _trilinear(coarse, fine):
    """The device transfer rule (hex3d.inc.cu k3_prolong) as a dense matrix."""
    fnx, fny, fnz = fine.node_shape
    cnx, cny, _ = coarse.node_shape
    p = np.zeros((fine.n, coarse.n))
    for fz in range(fnz):
        for fy in range(fny):
            for fx_ in range(fnx):
                fi = fx_ + fnx * (fy + fny * fz)
                w = (0.5 if fx_ & 1 else 1.0) * (0.5 if fy & 1 else 1.0) * (0.5 if fz & 1 else 1.0)
                for cz in {fz >> 1, (fz + 1) >> 1}:
                    for cy in {fy >> 1, (fy + 1) >> 1}:
                        for cx in {fx_ >> 1, (fx_ + 1) >> 1}:
                            ci = cx + cnx * (cy + cny * cz)
                            for c in range(3):
                                r, col = fine.dof[fi, c], coarse.dof[ci, c]
                                if r >= 0 and col >= 0:
                                    p[r, col] = w
    return p


@pytest.mark.parametrize("name", ("CANT-2-2-2-3", "BRIDGE-3-3-2-2"))
def test_transfer_rule_matches_reference(fx, name):
    prob = mesh3d.build_hex_problem(name)
    tag = name.replace("-", "_")
    for k in range(len(prob.levels) - 1):
        rows, cols, vals = fx[f"{tag}__P{k}"]
        ref = np.zeros((prob.levels[k + 1].n, prob.levels[k].n))
        ref[rows.astype(int), cols.astype(int)] = vals
        np.testing.assert_array_equal(_trilinear(prob.levels[k], prob.levels[k + 1]), ref)
        assert prob.transfers[k].shape == ref.shape


@pytest.mark.parametrize("edge", (1.0, 0.5, 0.25))
def test_hex_stiffness_matches_reference(fx, edge):
    ke = mesh3d.hex_stiffness(1.0, 0.3, edge)
    ref = fx[f"ke_{edge}"]
    np.testing.assert_allclose(ke, ref, rtol=0, atol=1e-15 * np.abs(ref).max())
    assert np.array_equal(ke, ke.T)


def test_names_and_errors():
    assert mesh3d.parse_name("cant-2-1-1-4") == ("cantilever", 2, 1, 1, 4)
    with pytest.raises(ValueError):
        mesh3d.parse_name("CANT-2-2-3")
    with pytest.raises(ValueError):
        mesh3d.build_hex_problem("CANT-2-2-2-2", vol_frac=1.5)
    with pytest.raises(ValueError):
        mesh3d.hex_stiffness(1.0, 0.5)
    prob = mesh3d.build_hex_problem("BRIDGE-2-2-2-3", levels=2)
    assert prob.name == "BRIDGE-2-2-2-2" and len(prob.levels) == 2
