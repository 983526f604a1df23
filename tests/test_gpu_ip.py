"""Interior-point path on the device operators against the reference's own ip.py.

Fixtures (`tests/golden/make_golden_ip.py`) come from the unmodified
`vtsopt.ip` on the 2D glue: every block of one Newton step at a seeded
interior state of C1, and a full `solve_ip` run on C1.  Tolerances are the
PBM path's: element values, applies and the V-cycle at
rtol 1e-12 (atol 1e-12 max|ref|); the full solve's objective and density
field within 1e-6 with the outer-iteration count within +-1.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU containers
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1904_06556_b200 as vts  # noqa: E402
from paper_1904_06556_b200 import ip  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def close(a, b, rtol=1e-12):
    a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    scale = max(float(np.abs(b).max()), 1e-300)
    np.testing.assert_allclose(a, b, rtol=rtol, atol=rtol * scale)


def dev(x):
    return torch.as_tensor(np.asarray(x, dtype=np.float64), device="cuda").contiguous()


@pytest.fixture(scope="module")
def step():
    fx = np.load(os.path.join(GOLD, "ip_c1_state.npz"))
    prob = vts.build_config("C1")
    ops = vts.ElementOps(prob.fine)
    bounds = vts.DensityBounds.for_problem(prob.m, prob.volume, 1e-7)
    st = ip.IpState(u=dev(fx["u"]), alpha=float(fx["alpha"]), rho=dev(fx["rho"]), nu_lo=dev(fx["nu_lo"]),
                    nu_up=dev(fx["nu_up"]), r=float(fx["r"]), s=float(fx["s"]))
    res = ip.kkt_residual(st, ops, prob.f, bounds)
    return fx, prob, ops, bounds, st, res


def test_kkt_residual_matches_reference(step):
    fx, _, _, _, _, res = step
    for k in ("res_u", "res_c", "res_lo", "res_up", "q"):
        close(getattr(res, k), fx[k])
    assert res.res_alpha == pytest.approx(float(fx["res_alpha"]), rel=1e-12)
    assert res.tau_res == pytest.approx(float(fx["tau_res"]), rel=1e-12)
    assert res.comp_max == pytest.approx(float(fx["comp_max"]), rel=1e-15)


def test_condensed_system_apply_and_vcycle_match_reference(step):
    fx, prob, ops, bounds, st, res = step
    mat, rhs, dcoef, g = ip.schur_system(st, res, ops, bounds)
    close(rhs, fx["rhs"])
    close(dcoef, fx["dcoef"])
    close(g, fx["g"])
    assert mat.corner == pytest.approx(float(fx["corner"]), rel=1e-12)
    close(mat.matvec(dev(fx["x"])), fx["Sx"])  # S+ x, border sign +1 (ip.py:154)
    mg = vts.MgPreconditioner(mat, prob.transfers)
    close(mg.apply(dev(fx["x"])), fx["Mx"])
    sol = vts.minres_solve(mat, rhs, vts.MinresConfig(tol=1e-8, max_iters=1000), mg.apply)
    assert sol.iterations == int(fx["minres_iters"])
    close(sol.x, fx["minres_x"], rtol=1e-6)


def test_reconstruct_and_step_lengths_match_reference(step):
    fx, prob, ops, bounds, st, res = step
    _, _, dcoef, g = ip.schur_system(st, res, ops, bounds)
    x = fx["minres_x"]
    drho, dnu_up, dnu_lo = ip.reconstruct(st, res, ops, bounds, dev(x[:-1]), float(x[-1]), dcoef, g)
    close(drho, fx["drho"])
    close(dnu_up, fx["dnu_up"])
    close(dnu_lo, fx["dnu_lo"])
    kap = ip.step_lengths(st, drho, dnu_lo, dnu_up, bounds, 0.9, ops)
    np.testing.assert_allclose(kap, fx["kappa"], rtol=1e-12)


def test_full_ip_solve_matches_reference_run():
    run = np.load(os.path.join(GOLD, "ip_c1_run.npz"))
    rep = ip.solve_ip(vts.build_config("C1"))
    assert rep.converged and bool(run["converged"])
    assert abs(rep.outer_iterations - run["rows"].shape[0]) <= 1
    assert rep.objective == pytest.approx(float(run["objective"]), rel=1e-6)
    rho, ref = rep.rho.cpu().numpy(), run["rho"]
    assert np.linalg.norm(rho - ref) <= 1e-6 * np.linalg.norm(ref)
    assert rep.volume == pytest.approx(float(run["volume"]), rel=1e-6)
    # the first iterations take the same MINRES counts (the tolerance policy and
    # the operators are the reference's)
    got = [r[1] for r in rep.rows[:5]]
    assert got == [int(v) for v in run["rows"][:5, 1]]
