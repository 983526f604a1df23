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
