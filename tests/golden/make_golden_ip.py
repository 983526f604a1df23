"""Golden fixtures for the interior-point path, produced by the unmodified reference.

Run HERE (the build container), where the read-only reference is mounted:

    NUMBA_CACHE_DIR=/tmp/numba_vtsopt python tests/golden/make_golden_ip.py

It reuses the 2D glue of make_golden.py (the reference `ElementOps` with the
Q1 constructor) and runs the reference's own
`vtsopt.ip` functions: `kkt_residual`, `schur_system` (border_sign=+1),
`MgPreconditioner`, `minres_solve`, `reconstruct`, `step_lengths` on a seeded
interior state of C1, and a full `solve_ip` on C1.  Outputs: `ip_c1_state.npz`,
`ip_c1_run.npz`, read by tests/test_gpu_ip.py.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as mg  # noqa: E402  (2D glue + reference imports)

import vtsopt.ip as rip  # noqa: E402
import vtsopt.linalg as rlinalg  # noqa: E402
import vtsopt.multigrid as rmgmod  # noqa: E402
import vtsopt.fem as rfem  # noqa: E402

rip.ElementOps = mg.ElementOps2DGlue  # solve_ip builds ElementOps(fine) (ip.py:229)


def state_fixture(prob, seed=0):
    rng = np.random.default_rng(seed)
    n, m = prob.n, prob.m
    st = rip.IpState(u=0.3 * rng.standard_normal(n) * 1e-1, alpha=float(rng.uniform(0.5, 4.0)),
                     rho=rng.uniform(0.1, 1.0, m), nu_lo=rng.uniform(0.05, 1.5, m),
                     nu_up=rng.uniform(0.05, 1.5, m), r=float(rng.uniform(0.05, 1.0)),
                     s=float(rng.uniform(0.05, 1.0)))
    ops = mg.ElementOps2DGlue(prob.fine)
    bounds = rfem.DensityBounds.for_problem(m, prob.volume, 1e-7)
    res = rip.kkt_residual(st, ops, prob.f, bounds)
    s_mat, rhs, dcoef, g = rip.schur_system(st, res, ops, bounds)
    x = np.random.default_rng(100 + seed).standard_normal(n + 1)
    pre = rmgmod.MgPreconditioner(s_mat, prob.transfers)
    sol = rlinalg.minres_solve(s_mat, rhs, rlinalg.MinresConfig(tol=1e-8, max_iters=1000), pre.apply)
    du, dalpha = sol.x[:-1], float(sol.x[-1])
    drho, dnu_up, dnu_lo = rip.reconstruct(st, res, ops, bounds, du, dalpha, dcoef, g)
    kp, klo, kup = rip.step_lengths(st, drho, dnu_lo, dnu_up, bounds, 0.9)
    comp_max = max(float(np.max(np.abs((st.rho - bounds.lower) * st.nu_lo))),
                   float(np.max(np.abs((bounds.upper - st.rho) * st.nu_up))))
    return dict(
        u=st.u, alpha=st.alpha, rho=st.rho, nu_lo=st.nu_lo, nu_up=st.nu_up, r=st.r, s=st.s,
        res_u=res.res_u, res_alpha=res.res_alpha, res_c=res.res_c, res_lo=res.res_lo, res_up=res.res_up, q=res.q,
        tau_res=res.tau_res, comp_max=comp_max, rhs=rhs, dcoef=dcoef, g=g, corner=s_mat.corner,
        x=x, Sx=s_mat.matvec(x), Mx=pre.apply(x), minres_x=sol.x, minres_iters=sol.iterations,
        minres_relres=sol.relres, drho=drho, dnu_up=dnu_up, dnu_lo=dnu_lo, kappa=np.array([kp, klo, kup]))


def run_fixture(prob):
    rep = rip.solve_ip(prob)
    return dict(rows=np.array(rep.rows, dtype=float), objective=rep.objective, gap_scaled=rep.gap_scaled,
                tau_res=rep.tau_res, volume=rep.volume, converged=rep.converged, rho=rep.rho,
                alpha=rep.extras["alpha"], minres_tol_final=rep.extras["minres_tol_final"], notes=rep.notes)


def main() -> None:
    prob = mg.build_config("C1")
    np.savez_compressed(os.path.join(HERE, "ip_c1_state.npz"), **state_fixture(prob))
    np.savez_compressed(os.path.join(HERE, "ip_c1_run.npz"), **run_fixture(prob))
    print("wrote ip_c1_state.npz, ip_c1_run.npz")


if __name__ == "__main__":
    main()
