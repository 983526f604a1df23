"""Run-to-run determinism of the CUDA path (bit for bit).

Every reduction is a fixed tree, the wavefront has a fixed schedule and no
atomics touch values, so repeated solves must agree exactly.  This also
guards the wavefront's reliance on finite slot data at out-of-range
positions: a stale-shared-memory NaN there shows up as a run-to-run
difference or a MINRES breakdown (it did once).
"""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU containers
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1904_06556_b200 as vts  # noqa: E402


def _system(key: str, seed: int = 0):
    prob = vts.build_config(key)
    n, m = prob.n, prob.m
    rng = np.random.default_rng(seed)
    host = dict(u=rng.normal(0.0, 1e-2, n), alpha=1e-3, nu_lo=rng.uniform(0, 1e-2, m),
                nu_up=rng.uniform(0, 1e-2, m), rho=rng.uniform(0.5, 2.0, m), mu_lo=np.ones(m), mu_up=np.ones(m),
                p=np.full(m, 1e-2), q_lo=np.ones(m), q_up=np.ones(m))
    st = vts.PbmState(**{k: (v if k == "alpha" else torch.as_tensor(v, device="cuda")) for k, v in host.items()})
    ops = vts.ElementOps(prob.fine)
    ev = vts.eval_lagrangian(st, ops, prob.f, vts.DensityBounds.for_problem(m, prob.volume, 0.0),
                             vts.PenaltyBarrier())
    mat, rhs = vts.schur_system(ev, ops)
    return prob, mat, rhs


@pytest.mark.parametrize("key", ["C1", "C2"])
def test_vcycle_and_minres_bitwise_repeatable(key):
    prob, mat, rhs = _system(key)
    mg = vts.MgPreconditioner(mat, prob.transfers)
    z0 = mg.apply(rhs).cpu().numpy()
    for _ in range(100):
        assert np.array_equal(mg.apply(rhs).cpu().numpy(), z0)
    cfg = vts.MinresConfig(tol=1e-10, max_iters=500)
    ref = vts.minres_solve(mat, rhs, cfg, mg.apply)
    for _ in range(10):
        res = vts.minres_solve(mat, rhs, cfg, mg.apply)
        assert res.iterations == ref.iterations
        assert np.array_equal(res.x.cpu().numpy(), ref.x.cpu().numpy())


def test_full_pbm_bitwise_repeatable():
    runs = [vts.solve_pbm(vts.build_config("C1")) for _ in range(4)]
    for r in runs[1:]:
        assert r.outer_iterations == runs[0].outer_iterations
        assert list(r.extras["minres_per_newton"]) == list(runs[0].extras["minres_per_newton"])
        assert r.objective == runs[0].objective
        assert np.array_equal(r.rho.cpu().numpy(), runs[0].rho.cpu().numpy())


def _run_ab(tmp_path, name, env_extra, key="C2"):
    import os
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = tmp_path / f"{name}.npy"
    env = dict(os.environ, **env_extra)
    subprocess.run([sys.executable, os.path.join(repo, "tools", "checks", "ab_vcycle.py"), str(out), key],
                   cwd=repo, env=env, check=True, capture_output=True, timeout=600)
    return np.load(out)


@pytest.mark.parametrize("switch,key", [("VTS_NO_PAIR", "C2"), ("VTS_UNFUSED_BOTTOM", "C2"),
                                        ("VTS_UNFUSED_BOTTOM", "C1"), ("VTS_CHOL_LEFT", "C1"),
                                        ("VTS_CHOL_LEFT", "C2")])
def test_fast_paths_are_bitwise_identical_to_the_plain_path(tmp_path, switch, key):
    """The pipelined sweep pairs and the fused V-cycle bottom compute exactly what
    the one-sweep-per-launch path computes (V-cycle output and a MINRES solution).
    C1's coarsest system (290 unknowns) takes the fused bottom's blocked substitution,
    against k_coarse_solve's column-by-column one.  VTS_CHOL_LEFT: the blocked
    right-looking coarse factor against k_cholesky's left-looking column loop."""
    fast = _run_ab(tmp_path, "fast", {}, key)
    plain = _run_ab(tmp_path, "plain", {switch: "1"}, key)
    assert np.array_equal(fast, plain)


@pytest.mark.parametrize("env_extra", [{"VTS_PAIR_CS_ASC": "4,4,4,4", "VTS_PAIR_CS_DESC": "6,5,3,3"},
                                       {"VTS_PAIR_INTERLEAVE": "1", "VTS_PAIR_CS_ASC": "3"},
                                       {"VTS_ARENA_PAD": "3"},
                                       {"VTS_DOVL_BLOCKS": "7,3,2,2", "VTS_OVL_BLOCKS": "5,2,1,1"}])
def test_scheduling_switches_do_not_change_a_bit(tmp_path, env_extra):
    """Cluster sizes of the pairs (more bands handed over through global memory), the order of
    the two sweeps' clusters in the grid, the placement of the level arrays and the number of
    blocks that draw residual / restriction / prolongation items by ticket only change when
    and where work runs: the V-cycle output and a MINRES solution on C3 (nine levels, five
    of them overlapped) keep every bit."""
    ref = _run_ab(tmp_path, "default", {}, "C3")
    alt = _run_ab(tmp_path, "switched", env_extra, "C3")
    assert np.array_equal(ref, alt)
