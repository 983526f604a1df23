"""Report and VTK writers against files written by the reference's serializers.

`tests/golden/make_golden_io.py` wrote `tests/golden/io/*` with the
unmodified `vtsopt.report` / `vtsopt.vtkio` for the reference's C1 PBM run.
The package's writers must reproduce them byte for byte (the VTK DIMENSIONS
line aside: the reference writes 3D slabs, the package 2D grids), and files
must read back bit-exactly (report.py:1-8, vtkio.py:1-9).
"""

from __future__ import annotations

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1904_06556_b200 import report, vtkio  # noqa: E402
from paper_1904_06556_b200.pbm import SolveReport  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
IO = os.path.join(GOLD, "io")


def _c1_report():
    d = np.load(os.path.join(GOLD, "pbm_c1.npz"))
    rows = [(int(r[0]), int(r[1]), int(r[2]), float(r[3]), float(r[4]), float(r[5])) for r in d["rows"]]
    return SolveReport(
        method="pbm", problem="C1", tol=1e-5, converged=bool(d["converged"]),
        columns=("outer", "newton", "minres", "gap_scaled", "tau_res", "volume"), rows=rows,
        count_columns=("newton", "minres"), objective=float(d["objective"]),
        dual_objective=float(d["dual_objective"]), gap_scaled=float(d["gap_scaled"]),
        tau_res=float(d["tau_res"]), volume=float(d["volume"]), rho=torch.as_tensor(d["rho"]), wall_clock=1.25,
        notes="golden", certificate="|duality gap|/|dual objective| = 1.000000e-06 < tol = 1.0e-05")


def test_csv_and_summary_are_byte_identical_to_the_reference(tmp_path):
    rep = _c1_report()
    report.write_csv(rep, tmp_path / "log.csv")
    report.write_summary(rep, tmp_path / "summary.txt")
    assert (tmp_path / "log.csv").read_bytes() == open(os.path.join(IO, "c1_log.csv"), "rb").read()
    assert (tmp_path / "summary.txt").read_bytes() == open(os.path.join(IO, "c1_summary.txt"), "rb").read()
    back = report.read_summary(tmp_path / "summary.txt")
    assert back["total_minres"] == "572" and float(back["objective"]) == rep.objective
    assert rep.totals() == {"newton": 34, "minres": 572} and rep.outer_iterations == 12


def _lines_without_dimensions(path):
    return [ln for ln in open(path).read().splitlines() if not ln.startswith("DIMENSIONS")]


def test_vtk_matches_the_reference_and_reads_back_bit_exactly(tmp_path):
    rep = _c1_report()
    vtkio.write_density_vtk(tmp_path / "rho.vtk", (64, 32), 1.0, rep.rho)
    assert _lines_without_dimensions(tmp_path / "rho.vtk") == _lines_without_dimensions(
        os.path.join(IO, "c1_rho.vtk"))
    assert "DIMENSIONS 65 33 1" in open(tmp_path / "rho.vtk").read()
    shape, spacing, values = vtkio.read_density_vtk(tmp_path / "rho.vtk")
    assert shape == (64, 32) and spacing == 1.0
    assert np.array_equal(values, rep.rho.numpy())
    mask = vtkio.write_filtered_vtk(tmp_path / "cut.vtk", (64, 32, 1), 1.0, rep.rho, rep.volume)
    assert np.array_equal(mask, np.load(os.path.join(IO, "c1_filter_mask.npy")))
    assert _lines_without_dimensions(tmp_path / "cut.vtk") == _lines_without_dimensions(
        os.path.join(IO, "c1_rho_filtered.vtk"))
    kept = rep.rho.numpy()[mask].sum()
    assert 0.8 * rep.volume - rep.rho.max().item() < kept <= 0.8 * rep.volume


def test_vtk_rejects_bad_shapes(tmp_path):
    with pytest.raises(ValueError):
        vtkio.write_density_vtk(tmp_path / "x.vtk", (4, 4), 1.0, np.zeros(15))
    with pytest.raises(ValueError):
        vtkio.write_density_vtk(tmp_path / "x.vtk", (4, 4, 2), 1.0, np.zeros(31))
    with pytest.raises(ValueError):
        vtkio.write_density_vtk(tmp_path / "x.vtk", (4,), 1.0, np.zeros(4))
    # a 3D element grid (the reference's own layout) round-trips
    vtkio.write_density_vtk(tmp_path / "x3.vtk", (4, 4, 2), 0.5, np.arange(32.0))
    assert "DIMENSIONS 5 5 3" in (tmp_path / "x3.vtk").read_text()
    shape, spacing, values = vtkio.read_density_vtk(tmp_path / "x3.vtk")
    assert shape == (4, 4, 2) and spacing == 0.5 and np.array_equal(values, np.arange(32.0))
    (tmp_path / "bad.vtk").write_text("# vtk\nnothing\n")
    with pytest.raises(ValueError):
        vtkio.read_density_vtk(tmp_path / "bad.vtk")


@pytest.mark.gpu
def test_device_solve_writes_and_reads_back(tmp_path):
    if not torch.cuda.is_available():  # pragma: no cover
        pytest.skip("needs a CUDA device")
    import paper_1904_06556_b200 as vts

    rep = vts.solve_pbm(vts.build_config("C1"))
    report.write_csv(rep, tmp_path / "log.csv")
    report.write_summary(rep, tmp_path / "s.txt")
    vtkio.write_density_vtk(tmp_path / "rho.vtk", (64, 32), 1.0, rep.rho)
    _, _, values = vtkio.read_density_vtk(tmp_path / "rho.vtk")
    assert np.array_equal(values, rep.rho.cpu().numpy())
    assert report.read_summary(tmp_path / "s.txt")["outer_iterations"] == str(rep.outer_iterations)
    assert len(open(tmp_path / "log.csv").read().splitlines()) == rep.outer_iterations + 1
