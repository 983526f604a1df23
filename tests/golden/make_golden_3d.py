"""Golden fixtures for the 3D hexahedral path, from the UNMODIFIED reference -- no glue.

Run HERE (the build container, where /root/reference is mounted):

    NUMBA_CACHE_DIR=/tmp/numba_vtsopt python tests/golden/make_golden_3d.py [mesh]

The reference is 3D (mesh.py, fem.py:31-97), so these fixtures come from its
own `build_problem`, `ElementOps`, `eval_lagrangian`, `schur_system`,
`MgPreconditioner`, `minres_solve`, `solve_pbm` and `solve_doc` with nothing
replaced:

* `hex_<instance>_kernels.npz` -- a seeded state (the reference's own
  `oracles.random_pbm_state`, pkg/tests/oracles.py:312-330): phi-pass outputs,
  Schur rhs / border / corner, S x, every Galerkin level probed, V-cycles,
  20-iteration MINRES histories, the tol-1e-6 solve, reconstruction, Armijo
  trial value;
* `hex_pbm_cant2223.npz` -- `solve_pbm` on CANT-2-2-2-3 at tol 1e-6, the
  instance of the reference README's run record (pkg/README.md:70-71:
  14 outer, 6460 MINRES, objective 6.4023097317);
* `hex_pbm_bridge2223.npz`, `hex_doc_cant2223.npz` -- default-tolerance PBM on
  BRIDGE-2-2-2-3 and DOC on CANT-2-2-2-3.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_vtsopt")
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)

import oracles as roracles  # noqa: E402  (reference test helpers)
import vtsopt.doc as rdoc  # noqa: E402
import vtsopt.fem as rfem  # noqa: E402
import vtsopt.linalg as rlinalg  # noqa: E402
import vtsopt.mesh as rmesh  # noqa: E402
import vtsopt.multigrid as rmg  # noqa: E402
import vtsopt.pbm as rpbm  # noqa: E402
import vtsopt.penalty as rpen  # noqa: E402

PEN = rpen.PenaltyBarrier()
STATE_KEYS = ("u", "alpha", "nu_lo", "nu_up", "rho", "mu_lo", "mu_up", "p", "q_lo", "q_up")


def kernels(name: str, seed: int) -> dict:
    prob = rmesh.build_problem(name)
    st = roracles.random_pbm_state(prob.n, prob.m, prob.volume, seed=seed)
    ops = rfem.ElementOps(prob.fine)
    bounds = rfem.DensityBounds.for_problem(prob.m, prob.volume, 0.0)
    ev = rpbm.eval_lagrangian(st, ops, prob.f, bounds, PEN)
    s_mat, rhs = rpbm.schur_system(ev, ops)
    rng = np.random.default_rng(1000 + seed)
    x = rng.standard_normal(prob.n + 1)
    du = 1e-2 * rng.standard_normal(prob.n)
    dalpha = float(1e-3 * rng.standard_normal())
    dnu_lo, dnu_up = rpbm.reconstruct_nu(ev, ops, du, dalpha)
    kappa = 0.5
    trial = rpbm._al_value(st.u + kappa * du, st.alpha + kappa * dalpha, st.nu_lo + kappa * dnu_lo,
                           st.nu_up + kappa * dnu_up, st, ops, prob.f, bounds, PEN)
    out = {f"st_{k}": np.asarray(getattr(st, k), dtype=float) for k in STATE_KEYS}
    out.update({
        "value": ev.value, "res_u": ev.res_u, "res_alpha": ev.res_alpha, "res_lo": ev.res_lo, "res_up": ev.res_up,
        "tau_res": ev.tau_res, "q": ev.q, "mu_hat_lo": ev.mu_hat_lo, "mu_hat_up": ev.mu_hat_up, "w": ev.blocks.w,
        "a": ev.blocks.a, "b_lo": ev.blocks.b_lo, "b_up": ev.blocks.b_up, "rho_hat": ev.blocks.rho_hat,
        "rhs": rhs, "border": s_mat.border, "corner": s_mat.corner, "x": x, "Sx": s_mat.matvec(x),
        "du": du, "dalpha": dalpha, "dnu_lo": dnu_lo, "dnu_up": dnu_up, "kappa": kappa, "trial_value": trial,
    })
    mg = rmg.MgPreconditioner(s_mat, prob.transfers)
    out["shifted"] = mg.shifted
    out["vcycle_x"] = mg.apply(x)
    out["vcycle_rhs"] = mg.apply(rhs)
    for k, mat in enumerate(mg.mats):
        v = np.random.default_rng(2000 + k).standard_normal(mat.core_dim + 1)
        out[f"level{k}_probe"] = v
        out[f"level{k}_apply"] = mat.matvec(v)
    hist = []
    for k in range(1, 21):
        res = rlinalg.minres_solve(s_mat, rhs, rlinalg.MinresConfig(tol=1e-14, max_iters=k), mg.apply)
        hist.append(res.relres)
    out["minres_hist"] = np.array(hist)
    res = rlinalg.minres_solve(s_mat, rhs, rlinalg.MinresConfig(tol=1e-6, max_iters=1000), mg.apply)
    out["minres_tol6_x"], out["minres_tol6_iters"] = res.x, res.iterations
    return out


def pbm_run(name: str, tol: float) -> tuple[dict, dict]:
    prob = rmesh.build_problem(name)
    rep = rpbm.solve_pbm(prob, rpbm.PbmConfig(tol=tol))
    out = {"objective": rep.objective, "outer": rep.outer_iterations, "converged": rep.converged,
           "rows": np.array(rep.rows, dtype=float), "minres_per_newton": np.array(rep.extras["minres_per_newton"]),
           "rho": rep.rho, "volume": rep.volume, "gap_scaled": rep.gap_scaled}
    meta = {"objective": rep.objective, "outer": rep.outer_iterations, **rep.totals(), "wall_clock_s": rep.wall_clock}
    return out, meta


def main() -> None:
    meta = {"generator": "tests/golden/make_golden_3d.py", "reference": REF_SRC}
    for name, seed, tag in (("CANT-2-2-2-3", 3, "cant2223"), ("BRIDGE-2-2-2-3", 5, "bridge2223")):
        np.savez_compressed(os.path.join(HERE, f"hex_{tag}_kernels.npz"), **kernels(name, seed))
    out, m = pbm_run("CANT-2-2-2-3", 1e-6)
    np.savez_compressed(os.path.join(HERE, "hex_pbm_cant2223.npz"), **out)
    meta["pbm_cant2223_tol1e-6"] = m
    out, m = pbm_run("BRIDGE-2-2-2-3", 1e-5)
    np.savez_compressed(os.path.join(HERE, "hex_pbm_bridge2223.npz"), **out)
    meta["pbm_bridge2223"] = m
    rep = rdoc.solve_doc(rmesh.build_problem("CANT-2-2-2-3"))
    np.savez_compressed(os.path.join(HERE, "hex_doc_cant2223.npz"), rows=np.array(rep.rows, dtype=float),
                        objective=rep.objective, converged=rep.converged, rho=rep.rho, volume=rep.volume)
    meta["doc_cant2223"] = {"objective": rep.objective, "iters": rep.outer_iterations, **rep.totals()}
    with open(os.path.join(HERE, "golden_meta_3d.json"), "w") as fh:
        json.dump(meta, fh, indent=1, default=float)
    print(json.dumps(meta, indent=1, default=float))


if __name__ == "__main__" and "mesh" not in sys.argv[1:]:
    main()


def mesh_fixture() -> None:
    """`hex_mesh.npz`: the reference's own hierarchies and element stiffness for the CPU mesh test."""
    out = {}
    for name in ("CANT-2-2-2-3", "BRIDGE-4-2-2-2", "CANT-3-1-2-2", "BRIDGE-3-3-2-2"):
        prob = rmesh.build_problem(name)
        tag = name.replace("-", "_")
        out[f"{tag}__volume"] = prob.volume
        for k, lv in enumerate(prob.levels):
            out[f"{tag}__L{k}_dof"] = lv.dof
            out[f"{tag}__L{k}_load"] = lv.load
            out[f"{tag}__L{k}_shape"] = np.array(lv.shape)
            out[f"{tag}__L{k}_conn"] = lv.conn
        for k, p in enumerate(prob.transfers):
            c = p.tocoo()
            out[f"{tag}__P{k}"] = np.stack([c.row.astype(float), c.col.astype(float), c.data])
    for edge in (1.0, 0.5, 0.25):
        out[f"ke_{edge}"] = rfem.hex_stiffness(1.0, 0.3, edge)
    np.savez_compressed(os.path.join(HERE, "hex_mesh.npz"), **out)


if __name__ == "__main__" and "mesh" in sys.argv[1:]:
    mesh_fixture()
