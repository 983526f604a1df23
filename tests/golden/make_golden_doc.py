"""Golden fixtures for the DOC path, from the unmodified reference.

Run HERE (the build container, where /root/reference is mounted):

    NUMBA_CACHE_DIR=/tmp/numba_vtsopt python tests/golden/make_golden_doc.py

Uses `vtsopt.doc` and `vtsopt.model` unchanged, on the 2D glue of
`make_golden.py` (the glue's ElementOps inherits the reference's
`assemble_stiffness` / `element_products`, fem.py:175-219):

* `doc_c1_blocks.npz` -- one state-solve round on C1 at a seeded thickness
  field: K(rho) x (fem.py:211-219), the unbordered Galerkin levels and V-cycle
  (multigrid.py:82-154), a warm-started MINRES solve with its residual history
  (linalg.py:128-242 with x0), element products (fem.py:175-180), doc_update
  and bisect_volume (doc.py:63-108), best_alpha_gap (model.py:82-98);
* `doc_c1_run.npz` -- the full `solve_doc` on C1 (doc.py:111-208): rows,
  objective, counts, final rho and u.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as mg_  # noqa: E402  (reference + 2D glue)
import vtsopt.doc as rdoc  # noqa: E402
import vtsopt.model as rmodel  # noqa: E402

rdoc.ElementOps = mg_.ElementOps2DGlue  # solve_doc builds ElementOps(fine) (doc.py:117)


def blocks_fixture(prob) -> dict:
    cfg = rdoc.DocConfig()
    rng = np.random.default_rng(21)
    ops = mg_.ElementOps2DGlue(prob.fine)
    bounds = mg_.rfem.DensityBounds.for_problem(prob.m, prob.volume, cfg.rho_lower)
    rho = rng.uniform(0.05, 1.0, prob.m)
    rho *= prob.volume / rho.sum()
    rho = np.clip(rho, bounds.lower, bounds.upper)
    k_mat = ops.assemble_stiffness(rho)
    x = rng.standard_normal(prob.n)
    out = {"rho": rho, "x": x, "Kx": k_mat @ x}
    chain = mg_.rmg.MgPreconditioner(k_mat, prob.transfers)
    out["shifted"] = chain.shifted
    for k, mat in enumerate(chain.mats):
        v = np.random.default_rng(3000 + k).standard_normal(mat.core_dim)
        out[f"level{k}_probe"] = v
        out[f"level{k}_apply"] = mat.matvec(v)
    out["vcycle_x"] = chain.apply(x)
    out["vcycle_f"] = chain.apply(prob.f)
    # warm start: a perturbed solution of a looser solve
    rough = mg_.rlinalg.minres_solve(k_mat, prob.f, mg_.rlinalg.MinresConfig(tol=1e-2, max_iters=1000), chain.apply)
    out["x0"] = rough.x
    hist = []
    for k in range(1, 16):
        res = mg_.rlinalg.minres_solve(k_mat, prob.f, mg_.rlinalg.MinresConfig(tol=1e-14, max_iters=k), chain.apply,
                                       x0=rough.x)
        hist.append(res.relres)
    out["warm_hist"] = np.array(hist)
    res = mg_.rlinalg.minres_solve(k_mat, prob.f, mg_.rlinalg.MinresConfig(tol=1e-4, max_iters=1000), chain.apply,
                                   x0=rough.x)
    out["warm_iters"], out["warm_relres"], out["warm_x"] = res.iterations, res.relres, res.x
    res = mg_.rlinalg.minres_solve(k_mat, prob.f, mg_.rlinalg.MinresConfig(tol=1e-4, max_iters=1000, floor=1e-1),
                                   chain.apply, x0=rough.x)
    out["floor_iters"], out["floor_relres"] = res.iterations, res.relres
    u = res.x
    w, q = ops.element_products(u)
    out["u"], out["w"], out["q"] = u, w, q
    z = 2.0 * q
    out["update_alpha"] = 0.37
    out["update"] = rdoc.doc_update(rho, z, 0.37, cfg.exponent, bounds)
    alpha, rho_new = rdoc.bisect_volume(rho, z, bounds, cfg)
    out["bisect_alpha"], out["bisect_rho"] = alpha, rho_new
    fu = float(prob.f @ u)
    gap, ga = rmodel.best_alpha_gap(q, fu, bounds)
    out["fu"], out["gap"], out["gap_alpha"] = fu, gap, ga
    out["step_inf"] = float(np.max(np.abs(rho_new - rho)))
    return out


def main() -> None:
    meta = {"generator": "tests/golden/make_golden_doc.py"}
    c1 = mg_.build_config("C1")
    np.savez_compressed(os.path.join(HERE, "doc_c1_blocks.npz"), **blocks_fixture(c1))
    rep = rdoc.solve_doc(c1)
    np.savez_compressed(os.path.join(HERE, "doc_c1_run.npz"), rows=np.array(rep.rows, dtype=float),
                        objective=rep.objective, converged=rep.converged, volume=rep.volume, rho=rep.rho,
                        u=rep.extras["u"], gap_scaled=rep.gap_scaled, tau_res=rep.tau_res)
    meta["doc_c1"] = {"objective": rep.objective, "iters": rep.outer_iterations, **rep.totals(),
                      "converged": rep.converged, "wall_clock_s": rep.wall_clock, "notes": rep.notes}
    with open(os.path.join(HERE, "golden_meta_doc.json"), "w") as fh:
        json.dump(meta, fh, indent=1, default=float)
    print(json.dumps(meta, indent=1, default=float))


if __name__ == "__main__":
    main()
