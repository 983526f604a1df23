"""GPU parity of the 3D hexahedral path against the UNMODIFIED reference.

The reference's own discretisation is 3D, so these fixtures
(`tests/golden/make_golden_3d.py`) are the reference run with nothing
replaced -- no 2D glue.  Tolerances as for the 2D path (BASELINE.json's
north_star): per-element g / phi outputs, the Schur blocks, S x and every
Galerkin level at rtol 1e-12 (atol 1e-12 max|ref|); the V-cycle at 1e-11
(the coarse Galerkin entries' rounding, see tests/test_gpu_target.py); MINRES
histories |dh| <= 1e-8 h + 1e-13; full solves to the same counts and the
objective at 1e-9.  The CANT-2-2-2-3 solve at tol 1e-6 is the reference
README's run record (pkg/README.md:70-71: 14 outer / 6460 MINRES,
objective 6.4023097317).
"""

from __future__ import annotations

import numpy as np
import pytest

from golden_io import STATE_KEYS, load

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU containers
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1904_06556_b200 as vts  # noqa: E402

CASES = {"cant2223": "CANT-2-2-2-3", "bridge2223": "BRIDGE-2-2-2-3"}


def close(a, b, rtol=1e-12):
    a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    scale = max(float(np.abs(b).max()), 1e-300)
    np.testing.assert_allclose(a, b, rtol=rtol, atol=rtol * scale)


def dev(x):
    return torch.as_tensor(np.asarray(x, dtype=np.float64), device="cuda").contiguous()


class Hex:
    def __init__(self, tag):
        self.fx = load(f"hex_{tag}_kernels")
        self.prob = vts.build_problem(CASES[tag])
        self.ops = vts.ElementOps(self.prob.fine)
        assert self.ops.dim == 3 and self.ops.dofs_per_elem == 24
        st = {k: self.fx["st_" + k] for k in STATE_KEYS}
        self.state = vts.PbmState(**{k: (float(v) if k == "alpha" else dev(v)) for k, v in st.items()})
        self.bounds = vts.DensityBounds.for_problem(self.prob.m, self.prob.volume, 0.0)
        self.pen = vts.PenaltyBarrier()
        self.ev = vts.eval_lagrangian(self.state, self.ops, self.prob.f, self.bounds, self.pen, keep_w=True)


@pytest.fixture(scope="module", params=sorted(CASES))
def case(request):
    return Hex(request.param)


def test_hex_mesh_and_stiffness():
    prob = vts.build_problem("CANT-2-2-2-3")
    assert (prob.n, prob.m, len(prob.levels)) == (1944, 512, 3)
    assert prob.fine.shape == (8, 8, 8) and prob.fine.edge == 0.25
    from paper_1904_06556_b200.mesh3d import hex_stiffness

    ke = hex_stiffness(1.0, 0.3, 1.0)
    ev = np.linalg.eigvalsh(ke)
    assert np.all(np.abs(ev[:6]) < 1e-12) and ev[6] > 1e-3  # six rigid-body modes
    np.testing.assert_allclose(hex_stiffness(1.0, 0.3, 0.5), 0.5 * ke, rtol=1e-15)


def test_hex_phi_pass(case):
    ev, fx = case.ev, case.fx
    assert ev.value == pytest.approx(float(fx["value"]), rel=1e-12)
    assert ev.tau_res == pytest.approx(float(fx["tau_res"]), rel=1e-12)
    assert ev.res_alpha == pytest.approx(float(fx["res_alpha"]), rel=1e-12, abs=1e-12 * case.prob.volume)
    for key in ("res_u", "res_lo", "res_up", "q", "mu_hat_lo", "mu_hat_up"):
        close(getattr(ev, key), fx[key])
    for key in ("a", "b_lo", "b_up", "rho_hat", "w"):
        close(getattr(ev.blocks, key), fx[key])


def test_hex_schur_apply_reconstruct(case):
    fx = case.fx
    mat, rhs = vts.schur_system(case.ev, case.ops)
    close(rhs, fx["rhs"])
    close(mat.border, fx["border"])
    assert mat.corner == pytest.approx(float(fx["corner"]), rel=1e-13)
    close(mat.matvec(dev(fx["x"])), fx["Sx"])
    dnu_lo, dnu_up = vts.reconstruct_nu(case.ev, case.ops, dev(fx["du"]), float(fx["dalpha"]))
    close(dnu_lo, fx["dnu_lo"])
    close(dnu_up, fx["dnu_up"])
    k = float(fx["kappa"])
    st = case.state
    du = dev(fx["du"])
    trial = vts.al_value(st.u + k * du, st.alpha + k * float(fx["dalpha"]), st.nu_lo + k * dnu_lo,
                         st.nu_up + k * dnu_up, st, case.ops, case.prob.f, case.bounds, case.pen)
    assert trial == pytest.approx(float(fx["trial_value"]), rel=1e-12)


def test_hex_levels_vcycle_minres(case):
    fx = case.fx
    mat, rhs = vts.schur_system(case.ev, case.ops)
    mg = vts.MgPreconditioner(mat, case.prob.transfers)
    assert mg.shifted == bool(fx["shifted"])
    for k, lev in enumerate(mg.mats):
        close(lev.matvec(dev(fx[f"level{k}_probe"])), fx[f"level{k}_apply"])
    close(mg.apply(dev(fx["x"])), fx["vcycle_x"], 1e-11)
    close(mg.apply(rhs), fx["vcycle_rhs"], 1e-11)
    hist = []
    vts.minres_solve(mat, rhs, vts.MinresConfig(tol=1e-14, max_iters=20), mg.apply, history=hist)
    ref = fx["minres_hist"]
    cnt = min(len(hist), ref.size)
    h = np.array(hist[:cnt])
    assert cnt >= 10
    assert np.all(np.abs(h - ref[:cnt]) <= 1e-8 * ref[:cnt] + 1e-13 + 0.25 * ref.min()), (h, ref)
    res = vts.minres_solve(mat, rhs, vts.MinresConfig(tol=1e-6, max_iters=1000), mg.apply)
    assert res.iterations == int(fx["minres_tol6_iters"])
    close(res.x, fx["minres_tol6_x"], 1e-9)


def test_hex_pbm_reproduces_reference_readme_record():
    """CANT-2-2-2-3, tol 1e-6: the reference README's 14 / 6460 / 6.4023097317."""
    fx = load("hex_pbm_cant2223")
    rep = vts.solve_pbm(vts.build_problem("CANT-2-2-2-3"), vts.PbmConfig(tol=1e-6))
    assert rep.converged and rep.outer_iterations == int(fx["outer"]) == 14
    counts = np.array(rep.extras["minres_per_newton"])
    ref = fx["minres_per_newton"]
    assert counts.size == ref.size == 37
    assert abs(int(counts.sum()) - int(ref.sum())) <= 0.01 * ref.sum()  # ~175 MINRES per late step
    assert rep.objective == pytest.approx(float(fx["objective"]), rel=1e-9)
    assert f"{rep.objective:.10f}".startswith("6.4023097317")
    close(rep.rho, fx["rho"], 1e-6)


def test_hex_bridge_pbm_and_cantilever_doc():
    fx = load("hex_pbm_bridge2223")
    rep = vts.solve_pbm(vts.build_problem("BRIDGE-2-2-2-3"))
    assert rep.converged and rep.outer_iterations == int(fx["outer"])
    np.testing.assert_array_equal(np.array(rep.extras["minres_per_newton"]), fx["minres_per_newton"])
    assert rep.objective == pytest.approx(float(fx["objective"]), rel=1e-9)
    close(rep.rho, fx["rho"], 1e-6)
    fx = load("hex_doc_cant2223")
    rep = vts.solve_doc(vts.build_problem("CANT-2-2-2-3"))
    rows, ref = np.array(rep.rows, dtype=float), fx["rows"]
    assert rep.converged == bool(fx["converged"]) and rows.shape == ref.shape
    np.testing.assert_array_equal(rows[:, 1], ref[:, 1])
    assert rep.objective == pytest.approx(float(fx["objective"]), rel=1e-9)
    close(rep.rho, fx["rho"], 1e-6)
