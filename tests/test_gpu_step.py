"""The device-resident Newton step (vts_newton_step, csrc/step.inc.cu) against the
call-by-call host path of newton_inner (pbm.py:244-338).

Both run the same kernels, so full solves must agree bit for bit: outer rows,
per-Newton MINRES counts, accepted Armijo steps and slopes, compliance and the
thickness field.  The reference itself is pinned against the host path in
test_gpu_parity.py / test_gpu_fullsize.py.
"""

import ctypes

import pytest
import torch

import paper_1904_06556_b200 as vts
from paper_1904_06556_b200 import _lib

pytestmark = pytest.mark.gpu


_EXTRA = {"MBB32": ("mbb", 4, 2, 4, 0.4), "BRIDGE32": ("bridge", 4, 2, 4, 0.3)}


def _solve(key, monkeypatch, host: bool):
    monkeypatch.setenv("VTS_HOST_NEWTON", "1" if host else "0")
    trace: dict = {}
    prob = vts.build_problem(*_EXTRA[key]) if key in _EXTRA else vts.build_config(key)
    rep = vts.solve_pbm(prob, trace=trace)
    torch.cuda.synchronize()
    return rep, trace


@pytest.mark.parametrize("key", ["C1", "MBB32", "BRIDGE32"])
def test_device_step_solve_is_bitwise_the_host_path(key, monkeypatch):
    dev, tdev = _solve(key, monkeypatch, host=False)
    host, thost = _solve(key, monkeypatch, host=True)
    assert dev.rows == host.rows
    assert dev.extras["minres_per_newton"] == host.extras["minres_per_newton"]
    assert tdev["kappa"] == thost["kappa"] and tdev["slope"] == thost["slope"]
    assert dev.objective == host.objective
    assert torch.equal(dev.rho, host.rho)
    assert torch.equal(dev.extras["u"], host.extras["u"])
    assert dev.extras["alpha"] == host.extras["alpha"]


def test_device_step_c2_counts_and_compliance(monkeypatch):
    dev, _ = _solve("C2", monkeypatch, host=False)
    host, _ = _solve("C2", monkeypatch, host=True)
    assert dev.rows == host.rows
    assert dev.objective == host.objective
    assert torch.equal(dev.rho, host.rho)


def test_device_step_syncs_and_graph_replays():
    """One host synchronisation per step (after the MINRES loop); from the second step
    on both phases replay their CUDA graphs."""
    prob = vts.build_config("C1")
    ops = vts.ElementOps(prob.fine)
    cfg = vts.PbmConfig()
    bounds = vts.DensityBounds.for_problem(prob.m, prob.volume, cfg.rho_lower)
    pen = vts.PenaltyBarrier(cfg.branch)
    state = vts.PbmState.initial(prob.n, prob.m, prob.volume)
    from paper_1904_06556_b200 import pbm

    seen = []
    real = _lib.load().vts_newton_step

    class Spy:
        def __call__(self, h, a, r):
            rc = real(h, a, r)
            res = ctypes.cast(r, ctypes.POINTER(_lib.NewtonStepResult)).contents
            seen.append((rc, res.host_syncs, res.graphs, res.trials))
            return rc

    lib = _lib.load()
    orig = lib.vts_newton_step
    lib.vts_newton_step = Spy()
    try:
        mtol = vts.StagnationTolerance(tol=0.5)
        out = pbm.newton_inner(state, ops, prob.f, bounds, pen, prob.transfers, 1e-3, mtol, cfg)
    finally:
        lib.vts_newton_step = orig
    assert out.steps >= 2 and len(seen) >= 2
    assert all(rc == 0 for rc, *_ in seen)
    assert all(s == 1 for _, s, _, t in seen if t <= 2)
    assert all(g == 2 for _, _, g, _ in seen)


def test_blocks_w_is_available_without_keep_w():
    """HessianBlocks.w (pbm.py:101-116) exists whether or not the evaluation wrote it:
    formed on first access from the evaluation's u, bit for bit the keep_w product."""
    prob = vts.build_config("C1")
    ops = vts.ElementOps(prob.fine)
    bounds = vts.DensityBounds.for_problem(prob.m, prob.volume, 0.0)
    gen = torch.Generator(device="cuda").manual_seed(3)
    state = vts.PbmState.initial(prob.n, prob.m, prob.volume)
    state.u = torch.randn(prob.n, dtype=torch.float64, device="cuda", generator=gen) * 1e-2
    lazy = vts.eval_lagrangian(state, ops, prob.f, bounds, vts.PenaltyBarrier())
    full = vts.eval_lagrangian(state, ops, prob.f, bounds, vts.PenaltyBarrier(), keep_w=True)
    assert lazy.blocks._w is None
    assert torch.equal(lazy.blocks.w, full.blocks.w)
    assert lazy.blocks.w.shape == (prob.m, 8)


def test_fused_evaluation_matches_the_two_kernel_pass(monkeypatch):
    """k_phi_tile (one launch) against k_phi_elem + k_phi_node + k_phi_finish: every
    vector bit for bit, the scalars to their reductions' rounding."""
    import subprocess
    import sys

    code = ("import sys; sys.path.insert(0, '.'); import numpy as np, torch, paper_1904_06556_b200 as vts;"
            "p = vts.build_config('C2'); o = vts.ElementOps(p.fine);"
            "b = vts.DensityBounds.for_problem(p.m, p.volume, 0.0); g = np.random.default_rng(2);"
            "s = vts.PbmState.initial(p.n, p.m, p.volume);"
            "s.u = torch.as_tensor(g.normal(0, 1e-2, p.n), device='cuda');"
            "s.nu_lo = torch.as_tensor(g.uniform(0, 1e-2, p.m), device='cuda');"
            "s.p = torch.full((p.m,), 1e-2, dtype=torch.float64, device='cuda');"
            "e = vts.eval_lagrangian(s, o, p.f, b, vts.PenaltyBarrier());"
            "np.savez(sys.argv[1], res_u=e.res_u.cpu(), res_lo=e.res_lo.cpu(), q=e.q.cpu(), a=e.blocks.a.cpu(),"
            " rho_hat=e.blocks.rho_hat.cpu(), scal=np.array([e.value, e.res_alpha, e.tau_res]))")
    import numpy as np
    import os
    import tempfile

    out = {}
    with tempfile.TemporaryDirectory() as tmp:
        for mode in ("0", "1"):
            path = os.path.join(tmp, f"e{mode}.npz")
            env = dict(os.environ, VTS_PHI_SPLIT=mode)
            subprocess.run([sys.executable, "-c", code, path], check=True, env=env,
                           cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
            with np.load(path) as z:
                out[mode] = {k: z[k] for k in z.files}
    for k in ("res_u", "res_lo", "q", "a", "rho_hat"):
        assert np.array_equal(out["0"][k], out["1"][k]), k
    np.testing.assert_allclose(out["0"]["scal"], out["1"]["scal"], rtol=1e-14)


def _step_args(prob, ops, state, ev, W, cfg, bounds, pen):
    from paper_1904_06556_b200 import pbm
    from paper_1904_06556_b200.fem import ptr

    a = _lib.NewtonStepArgs()
    a.u, a.nu_lo, a.nu_up = ptr(W.u), ptr(W.nu_lo), ptr(W.nu_up)
    for k in ("rho", "p", "mu_lo", "mu_up", "q_lo", "q_up"):
        setattr(a, k, ptr(getattr(state, k)))
    a.f, a.lower, a.upper = ptr(prob.f), ptr(bounds.lower), ptr(bounds.upper)
    a.volume, a.norm_f, a.norm_bounds, a.branch = float(bounds.volume), ops.norm_f, bounds.norm, pen.branch
    for k in pbm._StepWork._EV:
        setattr(a, k, ptr(W.ev[k]))
    a.chat, a.rhs, a.border, a.du, a.dnu_lo, a.dnu_up = (ptr(t) for t in (W.chat, W.rhs, W.border, W.du, W.dnu_lo,
                                                                          W.dnu_up))
    a.minres_floor, a.minres_cap, a.minres_tol = cfg.minres_floor, cfg.minres_cap, 0.5
    a.armijo_c1, a.armijo_shrink, a.armijo_max_halvings = cfg.armijo_c1, cfg.armijo_shrink, cfg.armijo_max_halvings
    a.shift_scale = 1e-12
    a.alpha, a.value, a.res_alpha = float(state.alpha), ev.value, ev.res_alpha
    return a


def _c1_step_setup():
    from paper_1904_06556_b200 import pbm

    prob = vts.build_config("C1")
    ops = vts.ElementOps(prob.fine)
    cfg = vts.PbmConfig()
    bounds = vts.DensityBounds.for_problem(prob.m, prob.volume, cfg.rho_lower)
    pen = vts.PenaltyBarrier(cfg.branch)
    state = vts.PbmState.initial(prob.n, prob.m, prob.volume)
    ev = vts.eval_lagrangian(state, ops, prob.f, bounds, pen)
    W = pbm._StepWork(ops)
    W.u.copy_(state.u)
    W.nu_lo.copy_(state.nu_lo)
    W.nu_up.copy_(state.nu_up)
    for k in pbm._StepWork._EV:
        W.ev[k].copy_(getattr(ev, k) if hasattr(ev, k) else getattr(ev.blocks, k))
    return prob, ops, cfg, bounds, pen, state, ev, W


def test_device_step_exhausted_line_search_leaves_the_state():
    """An unreachable decrease target (value = -1e300): every one of the 41 trials is
    rejected (pbm.py:299-318), the step reports the exhausted search after 21 host
    passes of two trials, and neither the state nor the evaluation moves."""
    prob, ops, cfg, bounds, pen, state, ev, W = _c1_step_setup()
    a = _step_args(prob, ops, state, ev, W, cfg, bounds, pen)
    a.value = -1e300
    u0, nu0, res0 = W.u.clone(), W.nu_lo.clone(), W.ev["res_u"].clone()
    r = _lib.NewtonStepResult()
    assert _lib.load().vts_newton_step(ops.handle, ctypes.byref(a), ctypes.byref(r)) == 0
    assert r.status == 2
    assert r.trials == cfg.armijo_max_halvings + 1
    assert r.host_syncs == (cfg.armijo_max_halvings + 2) // 2
    assert r.slope < 0.0
    assert torch.equal(W.u, u0) and torch.equal(W.nu_lo, nu0) and torch.equal(W.ev["res_u"], res0)
    assert r.alpha == float(state.alpha)


def test_device_step_minres_error_carries_the_sound_iterate():
    """A negative density makes the bound Schur matrix indefinite; with a preconditioner
    built from it MINRES raises (linalg.py:166-169 / 205-206) -- through the device step
    with the same code as the call-by-call path."""
    prob, ops, cfg, bounds, pen, state, ev, W = _c1_step_setup()
    state.rho[: prob.m // 2] = -1.0
    ev = vts.eval_lagrangian(state, ops, prob.f, bounds, pen)
    from paper_1904_06556_b200 import pbm

    for k in pbm._StepWork._EV:
        W.ev[k].copy_(getattr(ev, k) if hasattr(ev, k) else getattr(ev.blocks, k))
    a = _step_args(prob, ops, state, ev, W, cfg, bounds, pen)
    r = _lib.NewtonStepResult()
    rc_dev = _lib.load().vts_newton_step(ops.handle, ctypes.byref(a), ctypes.byref(r))
    mat, rhs = vts.schur_system(ev, ops)
    try:
        mg = vts.MgPreconditioner(mat, prob.transfers)
        vts.minres_solve(mat, rhs, vts.MinresConfig(tol=0.5, max_iters=cfg.minres_cap), mg.apply)
        rc_host = 0
    except vts.MinresError as exc:
        rc_host = {"preconditioner is indefinite: <M r, r> < 0": 1, "MINRES recurrence broke down": 2}.get(str(exc), 3)
    except Exception:  # the coarse factor failed even with the shift (multigrid.py:102)
        rc_host = 6
    assert rc_dev == rc_host
    assert rc_dev != 0
