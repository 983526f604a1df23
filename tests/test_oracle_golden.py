"""Pin the CPU oracle to the real reference through the committed fixtures.

The fixtures in tests/golden/ were produced by tests/golden/make_golden.py from
the unmodified reference solver modules (+ the validated 2D glue).  These
tests check that the oracle restatement (`oracle/`) reproduces them with the
reference's own tolerance styles (`test_pbm.py:64-79`, `test_fem.py:149-158`,
`test_linalg_multigrid.py:261-271`).  CPU only.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from golden_io import KERNEL_FIXTURES, load, state_dict
from oracle.fem2d import DensityBounds, ElementOps2D
from oracle.mesh2d import build_problem2d
from oracle.newton import schur_coefficients

PEN = oracle.PenaltyBarrier()


def close(a, b, rtol=1e-12):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    scale = max(float(np.abs(b).max()), 1e-300)
    np.testing.assert_allclose(a, b, rtol=rtol, atol=rtol * scale)


def test_penalty_known_answers():
    fx = load("penalty")
    close(PEN.value(fx["tau"]), fx["value"], 1e-15)
    close(PEN.deriv(fx["tau"]), fx["deriv"], 1e-15)
    close(PEN.deriv2(fx["tau"]), fx["deriv2"], 1e-15)


def test_penalty_saturation_warns():
    with pytest.warns(RuntimeWarning, match="saturated"):
        v = PEN.value(1e200)
    assert v == PEN.value(1e150)


@pytest.fixture(scope="module", params=sorted(KERNEL_FIXTURES))
def kernel_case(request):
    name = request.param
    prob = build_problem2d(*KERNEL_FIXTURES[name])
    fx = load(name)
    st = oracle.PbmState(**state_dict(fx))
    ops = ElementOps2D(prob.fine)
    bounds = DensityBounds.for_problem(prob.m, prob.volume, 0.0)
    ev = oracle.eval_lagrangian(st, ops, prob.f, bounds, PEN)
    return name, prob, fx, st, ops, bounds, ev


def test_phi_pass_matches_reference(kernel_case):
    _, prob, fx, st, ops, bounds, ev = kernel_case
    assert ev.value == pytest.approx(float(fx["value"]), rel=1e-12)
    assert ev.tau_res == pytest.approx(float(fx["tau_res"]), rel=1e-12)
    assert ev.res_alpha == pytest.approx(float(fx["res_alpha"]), rel=1e-12, abs=1e-12 * prob.volume)
    for key in ("res_u", "res_lo", "res_up", "q", "mu_hat_lo", "mu_hat_up"):
        close(getattr(ev, key), fx[key])
    for key in ("w", "a", "b_lo", "b_up", "rho_hat"):
        close(getattr(ev.blocks, key), fx[key])


def test_schur_system_and_apply_match_reference(kernel_case):
    _, prob, fx, st, ops, bounds, ev = kernel_case
    mat, rhs = oracle.schur_system(ev, ops)
    close(rhs, fx["rhs"])
    close(mat.border, fx["border"])
    assert mat.corner == pytest.approx(float(fx["corner"]), rel=1e-13)
    close(mat.matvec(fx["x"]), fx["Sx"])


def test_reconstruct_and_trial_value_match_reference(kernel_case):
    _, prob, fx, st, ops, bounds, ev = kernel_case
    dnu_lo, dnu_up = oracle.reconstruct_nu(ev, ops, fx["du"], float(fx["dalpha"]))
    close(dnu_lo, fx["dnu_lo"])
    close(dnu_up, fx["dnu_up"])
    k = float(fx["kappa"])
    trial = oracle.al_value(st.u + k * fx["du"], st.alpha + k * float(fx["dalpha"]),
                            st.nu_lo + k * dnu_lo, st.nu_up + k * dnu_up, st, ops, prob.f, bounds, PEN)
    assert trial == pytest.approx(float(fx["trial_value"]), rel=1e-12)


def test_multigrid_chain_and_vcycle_match_reference(kernel_case):
    _, prob, fx, st, ops, bounds, ev = kernel_case
    mat, rhs = oracle.schur_system(ev, ops)
    mg = oracle.MgPreconditioner(mat, prob.transfers)
    assert mg.shifted == bool(fx["shifted"])
    for k, lev in enumerate(mg.mats):
        close(lev.matvec(fx[f"level{k}_probe"]), fx[f"level{k}_apply"])
    close(mg.apply(fx["vcycle_in"]), fx["vcycle_out"])
    close(mg.apply(rhs), fx["vcycle_rhs_out"])


def test_minres_history_matches_reference(kernel_case):
    _, prob, fx, st, ops, bounds, ev = kernel_case
    mat, rhs = oracle.schur_system(ev, ops)
    mg = oracle.MgPreconditioner(mat, prob.transfers)
    hist = []
    res = oracle.minres_solve(mat, rhs, oracle.MinresConfig(tol=1e-14, max_iters=20), mg.apply,
                              history=hist)
    cnt = min(len(hist), fx["minres_hist"].size)  # the solve may stop before 20 iterations
    ref = fx["minres_hist"][:cnt]
    h = np.array(hist[:cnt])
    # rounding-level deviations are absolute near the floor
    assert np.all(np.abs(h - ref) <= 1e-8 * ref + 1e-13)
    if int(fx["minres_iters"][-1]) == 20:
        close(res.x, fx["minres20_x"], 1e-8)
    res6 = oracle.minres_solve(mat, rhs, oracle.MinresConfig(tol=1e-6, max_iters=1000), mg.apply)
    assert res6.iterations == int(fx["minres_tol6_iters"])
    close(res6.x, fx["minres_tol6_x"], 1e-9)


def test_schur_coefficients_positive(kernel_case):
    _, prob, fx, st, ops, bounds, ev = kernel_case
    chat, _ = schur_coefficients(ev)
    assert np.all(chat > 0.0)


@pytest.mark.parametrize("name,args", [
    ("pbm_c1", ("cantilever", 16, 8, 3, 0.5)),
    ("pbm_mbb32", ("mbb", 4, 2, 4, 0.4)),
])
def test_full_pbm_matches_reference(name, args):
    fx = load(name)
    rep = oracle.solve_pbm(build_problem2d(*args))
    assert rep.converged == bool(fx["converged"])
    assert rep.outer_iterations == int(fx["outer"])
    np.testing.assert_array_equal(np.array(rep.extras["minres_per_newton"]), fx["minres_per_newton"])
    assert rep.objective == pytest.approx(float(fx["objective"]), rel=1e-10)
    close(rep.rho, fx["rho"], 1e-7)
    close(rep.extras["u"], fx["u"], 1e-7)


@pytest.mark.slow
def test_full_pbm_c2_matches_reference():
    fx = load("pbm_c2")
    rep = oracle.solve_pbm(oracle.build_config("C2"))
    assert rep.outer_iterations == int(fx["outer"])
    np.testing.assert_array_equal(np.array(rep.extras["minres_per_newton"]), fx["minres_per_newton"])
    assert rep.objective == pytest.approx(float(fx["objective"]), rel=1e-10)
    close(rep.rho[fx["rho_sample_idx"]], fx["rho_sample"], 1e-7)
