"""Compare the GPU PBM trajectory with a golden fixture (diagnostics)."""
import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_1904_06556_b200 as vts
from golden_io import load
for name, args in [("pbm_mbb32", ("mbb", 4, 2, 4, 0.4)), ("pbm_c2", ("mbb", 8, 4, 6, 0.4)), ("pbm_c1", ("cantilever", 16, 8, 3, 0.5))]:
    fx = load(name)
    tr = {}
    rep = vts.solve_pbm(vts.build_problem(*args), trace=tr)
    mg = np.array(rep.extras["minres_per_newton"]); mr = fx["minres_per_newton"]
    print(name, "outer gpu/ref", rep.outer_iterations, int(fx["outer"]), "newton", rep.totals(), "ref minres sum", mr.sum(), "len", len(mr))
    k = min(len(mg), len(mr)); d = np.nonzero(mg[:k] != mr[:k])[0]
    print("  first minres-count mismatch at newton step", d[:5], "gpu", mg[d[:5]] if d.size else None, "ref", mr[d[:5]] if d.size else None)
    print("  objective rel diff", abs(rep.objective - float(fx["objective"])) / abs(float(fx["objective"])))
    rows_g = np.array(rep.rows); rows_r = fx["rows"]
    for rg, rr in zip(rows_g, rows_r):
        print("   row gpu", rg[:3].astype(int), "%.6e %.6e %.10f" % tuple(rg[3:]), "| ref", rr[:3].astype(int), "%.6e %.6e %.10f" % tuple(rr[3:]))
    if "rho" in fx:
        r = rep.rho.cpu().numpy(); print("  rho max abs diff", np.abs(r - fx["rho"]).max())
    else:
        r = rep.rho.cpu().numpy()[fx["rho_sample_idx"]]; print("  rho sample max abs diff", np.abs(r - fx["rho_sample"]).max())
    print("  kappas", tr.get("kappa")[:60])
