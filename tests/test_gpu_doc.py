"""GPU parity of the DOC path and of minres_solve's general contract.

Fixtures come from the unmodified reference (`tests/golden/make_golden_doc.py`:
`vtsopt.doc`, `vtsopt.model`, the reference's `assemble_stiffness` /
`element_products` on the validated 2D glue).  Tolerances as for the PBM
path: operator applies / V-cycle / element products at rtol 1e-12
(atol 1e-12 max|ref|); MINRES histories |dh| <= 1e-8 h + 1e-13; the full C1
`solve_doc` to the same iteration and MINRES counts, compliance at 1e-9.

Also here: `minres_solve` with a warm start `x0` on the bound system
(linalg.py:144-154), with a user operator (dense / sparse tensor or callable)
and a foreign preconditioner (linalg.py:118-125), and the reference's
MinresError paths (indefinite preconditioner, breakdown; test_linalg_multigrid.py:140-153).
"""

from __future__ import annotations

import numpy as np
import pytest

from golden_io import load

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU containers
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1904_06556_b200 as vts  # noqa: E402
from paper_1904_06556_b200 import doc as vdoc  # noqa: E402


def close(a, b, rtol=1e-12):
    a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    scale = max(float(np.abs(b).max()), 1e-300)
    np.testing.assert_allclose(a, b, rtol=rtol, atol=rtol * scale)


def dev(x):
    return torch.as_tensor(np.asarray(x, dtype=np.float64), device="cuda").contiguous()


@pytest.fixture(scope="module")
def blocks():
    fx = load("doc_c1_blocks")
    prob = vts.build_config("C1")
    ops = vts.ElementOps(prob.fine)
    cfg = vdoc.DocConfig()
    bounds = vts.DensityBounds.for_problem(prob.m, prob.volume, cfg.rho_lower)
    k_mat = ops.assemble_stiffness(dev(fx["rho"]))
    chain = vts.MgPreconditioner(k_mat, prob.transfers)
    return dict(fx=fx, prob=prob, ops=ops, cfg=cfg, bounds=bounds, k=k_mat, chain=chain)


def test_stiffness_apply_levels_and_vcycle(blocks):
    fx, k, chain = blocks["fx"], blocks["k"], blocks["chain"]
    assert k.shape == (blocks["prob"].n, blocks["prob"].n) and k.border is None
    close(k.matvec(dev(fx["x"])), fx["Kx"])
    assert chain.shifted == bool(fx["shifted"])
    for j, lev in enumerate(chain.mats):
        assert lev.dim == lev.core_dim
        close(lev.matvec(dev(fx[f"level{j}_probe"])), fx[f"level{j}_apply"])
    close(chain.apply(dev(fx["x"])), fx["vcycle_x"])
    close(chain.apply(blocks["prob"].f), fx["vcycle_f"])


def test_warm_started_minres_matches_reference(blocks):
    fx, k, chain, f = blocks["fx"], blocks["k"], blocks["chain"], blocks["prob"].f
    x0 = dev(fx["x0"])
    hist = []
    vts.minres_solve(k, f, vts.MinresConfig(tol=1e-14, max_iters=15), chain.apply, x0=x0, history=hist)
    ref = fx["warm_hist"]
    h = np.array(hist)
    cnt = min(h.size, ref.size)
    assert cnt >= 8
    assert np.all(np.abs(h[:cnt] - ref[:cnt]) <= 1e-8 * ref[:cnt] + 1e-13), (h, ref)
    res = vts.minres_solve(k, f, vts.MinresConfig(tol=1e-4, max_iters=1000), chain.apply, x0=x0)
    assert res.iterations == int(fx["warm_iters"]) and res.converged
    close(res.x, fx["warm_x"], 1e-9)
    # the warm start already meets a loose floor: x0 back, no iteration (linalg.py:153-154)
    res = vts.minres_solve(k, f, vts.MinresConfig(tol=1e-4, max_iters=1000, floor=1e-1), chain.apply, x0=x0)
    assert res.iterations == int(fx["floor_iters"]) == 0
    assert res.relres == pytest.approx(float(fx["floor_relres"]), rel=1e-9)
    assert torch.equal(res.x, x0)


def test_element_products_update_bisection_and_gap(blocks):
    fx, ops, bounds, cfg = blocks["fx"], blocks["ops"], blocks["bounds"], blocks["cfg"]
    u = dev(fx["u"])
    w, q = ops.element_products(u)
    close(w, fx["w"])
    close(q, fx["q"])
    rho = dev(fx["rho"])
    z = 2.0 * dev(fx["q"])
    close(vdoc.doc_update(rho, z, float(fx["update_alpha"]), cfg.exponent, bounds, ops), fx["update"])
    alpha, rho_new = vdoc.bisect_volume(rho, z, bounds, cfg, ops)
    assert alpha == pytest.approx(float(fx["bisect_alpha"]), rel=1e-12)
    close(rho_new, fx["bisect_rho"])
    meas = (__import__("ctypes").c_double * 5)()
    from paper_1904_06556_b200 import _lib
    from paper_1904_06556_b200.fem import ptr

    rc = _lib.load().vts_doc_measure(ops.handle, ptr(rho_new), ptr(rho), ptr(dev(fx["q"])), ptr(u),
                                     ptr(blocks["prob"].f), ptr(bounds.lower), ptr(bounds.upper),
                                     float(bounds.volume), meas)
    _lib.check(rc, "vts_doc_measure")
    assert meas[0] == pytest.approx(float(fx["step_inf"]), rel=1e-12)
    assert meas[1] == pytest.approx(float(fx["fu"]), rel=1e-12)
    assert meas[2] == pytest.approx(float(fx["gap"]), rel=1e-9, abs=1e-12 * abs(float(fx["fu"])))
    assert meas[3] == float(fx["gap_alpha"])
    with pytest.raises(ValueError, match="bracket invalid"):
        vdoc.bisect_volume(rho, 1e12 * z, bounds, vdoc.DocConfig(alpha_hi=1e-6), ops)


def test_full_doc_c1_matches_reference():
    fx = load("doc_c1_run")
    rep = vts.solve_doc(vts.build_config("C1"))
    ref_rows = fx["rows"]
    assert rep.converged == bool(fx["converged"])
    assert rep.outer_iterations == ref_rows.shape[0]
    rows = np.array(rep.rows, dtype=float)
    np.testing.assert_array_equal(rows[:, 1], ref_rows[:, 1])  # MINRES per state solve
    np.testing.assert_allclose(rows[:, 4], ref_rows[:, 4], rtol=1e-9)  # compliance per iteration
    np.testing.assert_allclose(rows[:, 2], ref_rows[:, 2], rtol=1e-6, atol=1e-9)  # step sizes
    assert rep.objective == pytest.approx(float(fx["objective"]), rel=1e-9)
    assert rep.volume == pytest.approx(float(fx["volume"]), rel=1e-9)
    close(rep.rho, fx["rho"], 1e-6)


# --- minres_solve's general contract (linalg.py:118-158) ------------------------------

def _spd(n, seed):
    g = torch.Generator().manual_seed(seed)
    a = torch.randn(n, n, generator=g, dtype=torch.float64)
    return (a @ a.T + n * torch.eye(n, dtype=torch.float64)).cuda()


def test_generic_operator_dense_sparse_callable_and_x0():
    n = 120
    a = _spd(n, 1)
    b = torch.randn(n, dtype=torch.float64, generator=torch.Generator().manual_seed(2)).cuda()
    dinv = 1.0 / torch.diagonal(a)
    cfg = vts.MinresConfig(tol=1e-10, max_iters=500)
    r_dense = vts.minres_solve(a, b, cfg, lambda v: dinv * v)
    r_sparse = vts.minres_solve(a.to_sparse_csr(), b, cfg, lambda v: dinv * v)
    r_call = vts.minres_solve(lambda v: a @ v, b, cfg, lambda v: dinv * v)
    for r in (r_dense, r_sparse, r_call):
        assert r.converged and r.relres <= 1e-10
        assert float(torch.linalg.norm(b - a @ r.x) / torch.linalg.norm(b)) <= 1e-10
    assert r_dense.iterations == r_call.iterations
    warm = vts.minres_solve(a, b, cfg, lambda v: dinv * v, x0=r_dense.x)
    assert warm.iterations <= 2
    exact = vts.minres_solve(a, b, vts.MinresConfig(tol=1e-10, floor=1e-6), None, x0=r_dense.x)
    assert exact.iterations == 0 and torch.equal(exact.x, r_dense.x)
    zero = vts.minres_solve(a, torch.zeros(n, dtype=torch.float64, device="cuda"), cfg)
    assert zero.iterations == 0 and zero.converged and float(zero.x.abs().max()) == 0.0


def test_generic_error_paths_match_reference_messages():
    n = 40
    a = _spd(n, 3)
    b = torch.ones(n, dtype=torch.float64, device="cuda")
    cfg = vts.MinresConfig(tol=1e-12, max_iters=100)
    # indefinite preconditioner: <M r, r> < 0 (linalg.py:166-169; test_linalg_multigrid.py:140-146)
    with pytest.raises(vts.MinresError, match="indefinite") as ei:
        vts.minres_solve(a, b, cfg, lambda v: -v)
    assert ei.value.x is not None and float(ei.value.x.abs().max()) == 0.0
    # breakdown: a singular operator whose Krylov recurrence produces gamma = 0
    # (linalg.py:214-217; test_linalg_multigrid.py:147-153)
    z = torch.zeros(n, n, dtype=torch.float64, device="cuda")
    with pytest.raises(vts.MinresError, match="broke down"):
        vts.minres_solve(z, b, cfg)
    # a callback error propagates unchanged
    def bad(v):
        raise KeyError("user operator failed")
    with pytest.raises(KeyError):
        vts.minres_solve(bad, b, cfg)


def test_nonfinite_operator_raises():
    a = torch.full((4, 4), float("nan"), dtype=torch.float64, device="cuda")
    with pytest.raises(vts.MinresError):  # test_linalg_multigrid.py:156-159
        vts.minres_solve(a, torch.ones(4, dtype=torch.float64, device="cuda"), vts.MinresConfig(tol=1e-8))


def test_device_indefinite_preconditioner_on_the_bound_stiffness(blocks):
    # test_linalg_multigrid.py:140-145: the bound K(rho) with an indefinite preconditioner
    with pytest.raises(vts.MinresError, match="indefinite"):
        vts.minres_solve(blocks["k"], blocks["prob"].f, vts.MinresConfig(tol=1e-8), precond=lambda v: -v)


def test_coarse_shift_fallback_and_hard_failure(caplog):
    """multigrid.py:92-103 on the device.

    * mu_lo = 0 makes every b_lo and hence every rank-one coefficient c_hat
      exactly 0 (pbm.py:211-212): the coarsest bordered matrix has an exactly
      zero border row and corner, the first factorization fails and the
      trace-scaled shift succeeds, with the reference's warning;
    * K(-rho) is negative definite: the shifted retry fails too and the
      reference's LinAlgError propagates (and assembling it warns).
    """
    import logging

    fx = load("c1_random_state")
    prob = vts.build_config("C1")
    ops = vts.ElementOps(prob.fine)
    st = {k: fx["st_" + k] for k in ("u", "alpha", "nu_lo", "nu_up", "rho", "mu_lo", "mu_up", "p", "q_lo", "q_up")}
    st["mu_lo"] = np.zeros_like(st["mu_lo"])
    state = vts.PbmState(**{k: (float(v) if k == "alpha" else dev(v)) for k, v in st.items()})
    ev = vts.eval_lagrangian(state, ops, prob.f, vts.DensityBounds.for_problem(prob.m, prob.volume, 0.0),
                             vts.PenaltyBarrier())
    mat, _ = vts.schur_system(ev, ops)
    assert mat.corner == 0.0 and float(mat.border.abs().max()) == 0.0
    with caplog.at_level(logging.WARNING, logger="paper_1904_06556_b200.multigrid"):
        pre = vts.MgPreconditioner(mat, prob.transfers)
    assert pre.shifted
    assert any("not positive definite" in rec.message for rec in caplog.records)
    with pytest.warns(RuntimeWarning, match="negative densities"):
        k_neg = ops.assemble_stiffness(-dev(fx["st_rho"]))
    with pytest.raises(np.linalg.LinAlgError):
        vts.MgPreconditioner(k_neg, prob.transfers)
