"""Generate the golden fixtures that pin the CPU oracle to the real reference.

Run HERE (the build container), where the read-only reference is mounted:

    NUMBA_CACHE_DIR=/tmp/numba_vtsopt python tests/golden/make_golden.py

It imports the *unmodified* reference solver modules from
`/root/reference/pkg/src/vtsopt` (`pbm`, `linalg`, `multigrid`, `penalty`,
`model`, `fem._AssemblyPattern`) and the reference's own seeded state
generator (`/root/reference/pkg/tests/oracles.py:312-330`).  The reference is
3D-only, so the one new piece on this side is the 2D discretisation glue of
SURVEY.md Appendix A: the Q1 mesh hierarchy of `oracle.mesh2d` and an
`ElementOps` subclass that overrides only `__init__` (the reference's
`fem.py:150-162` hard-codes 24 dofs) with the 8x8 `oracle.fem2d.quad_stiffness`.
Every other line that runs is reference code.  The glue itself is validated
by `tests/test_glue_invariants.py`.

Outputs (small .npz files next to this script) are read by
`tests/test_oracle_golden.py` (oracle vs reference, CPU) and by the GPU parity
tests (GPU vs the same fixtures).  /root/reference does not exist on the GPU
box; nothing else reads it.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_vtsopt")
sys.path.insert(0, REPO)
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)

import vtsopt.fem as rfem  # noqa: E402
import vtsopt.linalg as rlinalg  # noqa: E402
import vtsopt.multigrid as rmg  # noqa: E402
import vtsopt.pbm as rpbm  # noqa: E402
import vtsopt.penalty as rpen  # noqa: E402
import oracles as roracles  # noqa: E402  (reference test helpers)

from oracle.fem2d import quad_stiffness  # noqa: E402
from oracle.mesh2d import build_config, build_problem2d  # noqa: E402


class ElementOps2DGlue(rfem.ElementOps):
    """Reference ElementOps with the 3D constructor replaced by the Q1 one."""

    def __init__(self, level, e_mod: float = 1.0, nu: float = 0.3):  # noqa: D401
        self.level = level
        self.n = level.n
        self.m = level.m
        self.ke = quad_stiffness(e_mod, nu)
        edof = level.dof[level.conn].reshape(self.m, 8)
        self.edof = np.where(edof < 0, self.n, edof).astype(np.int64)
        rows = np.repeat(self.edof, 8, axis=1).ravel()
        cols = np.tile(self.edof, (1, 8)).ravel()
        self._mask = (rows != self.n) & (cols != self.n)
        self._pattern = rfem._AssemblyPattern(rows[self._mask], cols[self._mask], self.n)


rpbm.ElementOps = ElementOps2DGlue  # solve_pbm builds ElementOps(fine) (pbm.py:346)
PEN = rpen.PenaltyBarrier()


def microbench_state(n, m, seed):
    """BASELINE.json configs[2] state: u~N(0,1e-4), rho~U(0.5,2), p=1e-2, alpha=1e-3."""
    rng = np.random.default_rng(seed)
    u = rng.normal(0.0, 1e-2, n)
    rho = rng.uniform(0.5, 2.0, m)
    one = np.ones(m)
    return rpbm.PbmState(u=u, alpha=1e-3, nu_lo=one.copy(), nu_up=one.copy(), rho=rho,
                         mu_lo=one.copy(), mu_up=one.copy(), p=np.full(m, 1e-2),
                         q_lo=one.copy(), q_up=one.copy())


def state_arrays(prefix, st):
    return {f"{prefix}{k}": np.asarray(getattr(st, k), dtype=float) for k in
            ("u", "alpha", "nu_lo", "nu_up", "rho", "mu_lo", "mu_up", "p", "q_lo", "q_up")}


def kernel_fixture(prob, st, seed):
    """phi pass, Schur system, operator applies, V-cycle, MINRES replays, reconstruction."""
    ops = ElementOps2DGlue(prob.fine)
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
    out = {
        **state_arrays("st_", st),
        "value": ev.value, "res_u": ev.res_u, "res_alpha": ev.res_alpha, "res_lo": ev.res_lo,
        "res_up": ev.res_up, "tau_res": ev.tau_res, "q": ev.q, "mu_hat_lo": ev.mu_hat_lo,
        "mu_hat_up": ev.mu_hat_up, "w": ev.blocks.w, "a": ev.blocks.a, "b_lo": ev.blocks.b_lo,
        "b_up": ev.blocks.b_up, "rho_hat": ev.blocks.rho_hat,
        "rhs": rhs, "border": s_mat.border, "corner": s_mat.corner,
        "x": x, "Sx": s_mat.matvec(x),
        "du": du, "dalpha": dalpha, "dnu_lo": dnu_lo, "dnu_up": dnu_up,
        "kappa": kappa, "trial_value": trial,
    }
    mg = rmg.MgPreconditioner(s_mat, prob.transfers)
    out["shifted"] = mg.shifted
    out["vcycle_in"] = x
    out["vcycle_out"] = mg.apply(x)
    out["vcycle_rhs_out"] = mg.apply(rhs)
    # level operators, probed with seeded vectors (mats[k] is coarsest-first)
    for k, mat in enumerate(mg.mats):
        v = np.random.default_rng(2000 + k).standard_normal(mat.core_dim + 1)
        out[f"level{k}_probe"] = v
        out[f"level{k}_apply"] = mat.matvec(v)
    # MINRES residual history by the reference's own max_iters=k replays
    hist, iters = [], []
    for k in range(1, 21):
        res = rlinalg.minres_solve(s_mat, rhs, rlinalg.MinresConfig(tol=1e-14, max_iters=k), mg.apply)
        hist.append(res.relres)
        iters.append(res.iterations)
        if k == 20:
            out["minres20_x"] = res.x
    out["minres_hist"] = np.array(hist)
    out["minres_iters"] = np.array(iters)
    # one Newton-style solve at a realistic tolerance
    res = rlinalg.minres_solve(s_mat, rhs, rlinalg.MinresConfig(tol=1e-6, max_iters=1000), mg.apply)
    out["minres_tol6_x"] = res.x
    out["minres_tol6_iters"] = res.iterations
    out["minres_tol6_relres"] = res.relres
    return out


def pbm_fixture(prob, with_vectors: bool):
    rep = rpbm.solve_pbm(prob)
    out = {
        "objective": rep.objective, "dual_objective": rep.dual_objective,
        "gap_scaled": rep.gap_scaled, "tau_res": rep.tau_res, "volume": rep.volume,
        "converged": rep.converged, "outer": rep.outer_iterations,
        "rows": np.array(rep.rows, dtype=float),
        "minres_per_newton": np.array(rep.extras["minres_per_newton"]),
        "alpha": rep.extras["alpha"], "minres_tol_final": rep.extras["minres_tol_final"],
        "rho_sum": float(rep.rho.sum()), "rho_min": float(rep.rho.min()),
        "rho_max": float(rep.rho.max()), "wall_clock": rep.wall_clock,
    }
    if with_vectors:
        out["rho"] = rep.rho
        out["u"] = rep.extras["u"]
    else:
        idx = np.linspace(0, prob.m - 1, 512).astype(np.int64)
        out["rho_sample_idx"] = idx
        out["rho_sample"] = rep.rho[idx]
    return out, rep


def penalty_fixture():
    taus = np.concatenate([np.linspace(-3.0, 3.0, 61), [-0.5, -0.500000001, -0.49999999,
                           -1e3, -1e6, 1e3, 0.0, -100.0, 7.5]])
    return {"tau": taus, "value": PEN.value(taus), "deriv": PEN.deriv(taus), "deriv2": PEN.deriv2(taus)}


def main():
    meta = {"generator": "tests/golden/make_golden.py", "reference": REF_SRC,
            "numpy": np.__version__}
    np.savez_compressed(os.path.join(HERE, "penalty.npz"), **penalty_fixture())

    c1 = build_config("C1")
    st = roracles.random_pbm_state(c1.n, c1.m, c1.volume, seed=3)
    np.savez_compressed(os.path.join(HERE, "c1_random_state.npz"), **kernel_fixture(c1, st, 3))
    st = microbench_state(c1.n, c1.m, seed=7)
    np.savez_compressed(os.path.join(HERE, "c1_microbench_state.npz"), **kernel_fixture(c1, st, 7))

    mbb = build_problem2d("mbb", 4, 2, 4, 0.4)  # 32 x 16 MBB: per-dof fixing
    st = roracles.random_pbm_state(mbb.n, mbb.m, mbb.volume, seed=5)
    np.savez_compressed(os.path.join(HERE, "mbb32_random_state.npz"), **kernel_fixture(mbb, st, 5))

    br = build_problem2d("bridge", 4, 2, 4, 0.3)  # 32 x 16 bridge: pinned corners
    st = roracles.random_pbm_state(br.n, br.m, br.volume, seed=9)
    np.savez_compressed(os.path.join(HERE, "bridge32_random_state.npz"), **kernel_fixture(br, st, 9))

    out, rep = pbm_fixture(c1, with_vectors=True)
    np.savez_compressed(os.path.join(HERE, "pbm_c1.npz"), **out)
    meta["pbm_c1"] = {"objective": rep.objective, "outer": rep.outer_iterations, **rep.totals(),
                      "wall_clock_s": rep.wall_clock}
    small = build_problem2d("mbb", 4, 2, 4, 0.4)
    out, rep = pbm_fixture(small, with_vectors=True)
    np.savez_compressed(os.path.join(HERE, "pbm_mbb32.npz"), **out)
    meta["pbm_mbb32"] = {"objective": rep.objective, "outer": rep.outer_iterations, **rep.totals()}
    if os.environ.get("VTS_GOLDEN_C2", "1") == "1":
        c2 = build_config("C2")
        out, rep = pbm_fixture(c2, with_vectors=False)
        np.savez_compressed(os.path.join(HERE, "pbm_c2.npz"), **out)
        meta["pbm_c2"] = {"objective": rep.objective, "outer": rep.outer_iterations, **rep.totals(),
                          "wall_clock_s": rep.wall_clock}
    with open(os.path.join(HERE, "golden_meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1, default=float)
    print(json.dumps(meta, indent=1, default=float))


if __name__ == "__main__":
    main()
