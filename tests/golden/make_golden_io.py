"""Golden output files written by the reference's own serializers.

Run HERE (the build container), where the read-only reference is mounted:

    python tests/golden/make_golden_io.py

It imports the unmodified `vtsopt.report` (report.py:22-105) and
`vtsopt.vtkio` (vtkio.py:26-119) and writes, for the reference C1 PBM run
recorded in `pbm_c1.npz` (made by make_golden.py from the reference solver):
the iteration-log CSV, the key/value summary, the density VTK and the
filtered VTK.  The reference writer is 3D; the 2D fields are written as
(ex, ey, 1) slabs, whose only difference from the package's 2D files is the
DIMENSIONS line (`ex+1 ey+1 2` there, `ex+1 ey+1 1` here).
`tests/test_output_formats.py` checks the package's writers against these
files byte for byte (DIMENSIONS line aside).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from vtsopt import report as ref_report  # noqa: E402
from vtsopt import vtkio as ref_vtk  # noqa: E402

OUT = os.path.join(HERE, "io")


def reference_c1_report():
    d = np.load(os.path.join(HERE, "pbm_c1.npz"))
    rows = [(int(r[0]), int(r[1]), int(r[2]), float(r[3]), float(r[4]), float(r[5])) for r in d["rows"]]
    return ref_report.SolveReport(
        method="pbm", problem="C1", tol=1e-5, converged=bool(d["converged"]),
        columns=("outer", "newton", "minres", "gap_scaled", "tau_res", "volume"), rows=rows,
        count_columns=("newton", "minres"), objective=float(d["objective"]),
        dual_objective=float(d["dual_objective"]), gap_scaled=float(d["gap_scaled"]),
        tau_res=float(d["tau_res"]), volume=float(d["volume"]), rho=d["rho"], wall_clock=1.25,
        notes="golden", certificate="|duality gap|/|dual objective| = 1.000000e-06 < tol = 1.0e-05")


def main() -> None:
    os.makedirs(OUT, exist_ok=True)
    rep = reference_c1_report()
    ref_report.write_csv(rep, os.path.join(OUT, "c1_log.csv"))
    ref_report.write_summary(rep, os.path.join(OUT, "c1_summary.txt"))
    ref_vtk.write_density_vtk(os.path.join(OUT, "c1_rho.vtk"), (64, 32, 1), 1.0, rep.rho)
    mask = ref_vtk.write_filtered_vtk(os.path.join(OUT, "c1_rho_filtered.vtk"), (64, 32, 1), 1.0, rep.rho,
                                      rep.volume)
    np.save(os.path.join(OUT, "c1_filter_mask.npy"), mask)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
