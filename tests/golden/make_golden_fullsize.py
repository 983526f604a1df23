"""Golden fixtures at the north_star target size (1024x512, 9 levels), from the reference.

Run HERE (the build container, where /root/reference is mounted):

    NUMBA_CACHE_DIR=/tmp/numba_vtsopt python tests/golden/make_golden_fullsize.py [c3] [c4]

Like `make_golden.py` (whose glue it imports), every line that computes runs
the *unmodified* reference solver modules; the only new code on that side is
the 2D Q1 discretisation glue validated by `tests/test_glue_invariants.py`.

* `c3_ref_samples.npz` -- the C3 microbench state of BASELINE.json configs[2]
  (the seed-0 state and RHS `bench.py` uses, plus a both-branch variant with
  nu_lo, nu_up ~ U(0, 1e-2)).  Full 1M-length vectors would be ~150 MB, so the
  fixture keeps every output at 8192 seeded sample positions plus its 2-norm
  and sum: phi-pass outputs (pbm.py:150-199), Schur rhs / border / corner
  (pbm.py:202-218), S x (linalg.py:56-62), every level's Galerkin apply
  (multigrid.py:88-90), the V-cycle of x and of rhs (multigrid.py:109-143),
  the first 20 MINRES relative residuals (the reference's own max_iters=k
  replays, linalg.py:128-242), the tol-1e-6 iteration count, and the
  reconstruction / Armijo trial value (pbm.py:135-147, 221-232).
* `pbm_c4.npz` -- the full C4 solve (pbm.py:341-465): objective, counts, rows,
  per-Newton MINRES counts and the final thickness field rho (float64).
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as mg_  # noqa: E402  (imports the reference + installs the 2D glue)

rpbm, rlinalg, rmg, rfem = mg_.rpbm, mg_.rlinalg, mg_.rmg, mg_.rfem
PEN = mg_.PEN
N_SAMPLE = 8192


def sample_idx(length: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    idx = np.unique(np.concatenate([rng.choice(length, size=min(N_SAMPLE, length), replace=False),
                                    [0, length - 1]]))
    return idx.astype(np.int64)


def put(out: dict, name: str, vec, seed: int) -> None:
    """Store a long vector as (sample positions, values at them, 2-norm, sum)."""
    v = np.asarray(vec, dtype=float)
    if v.size <= 2 * N_SAMPLE:
        out[name] = v
        return
    idx = sample_idx(v.size, seed)
    out[f"{name}__idx"] = idx
    out[f"{name}__val"] = v[idx]
    out[f"{name}__norm"] = float(np.linalg.norm(v))
    out[f"{name}__sum"] = float(v.sum())
    out[f"{name}__max"] = float(np.abs(v).max())


def c3_state(prob, seed: int, both_branches: bool):
    """bench.py microbench_inputs (configs[2]); both_branches adds nu ~ U(0, 1e-2)."""
    rng = np.random.default_rng(seed)
    n, m = prob.n, prob.m
    u = rng.normal(0.0, 1e-2, n)
    rho = rng.uniform(0.5, 2.0, m)
    rhs = rng.standard_normal(n + 1)
    one = np.ones(m)
    nu_lo, nu_up = one.copy(), one.copy()
    if both_branches:
        nu_lo = rng.uniform(0.0, 1e-2, m)
        nu_up = rng.uniform(0.0, 1e-2, m)
    st = rpbm.PbmState(u=u, alpha=1e-3, nu_lo=nu_lo, nu_up=nu_up, rho=rho, mu_lo=one.copy(), mu_up=one.copy(),
                       p=np.full(m, 1e-2), q_lo=one.copy(), q_up=one.copy())
    return st, rhs


def c3_fixture(prob, seed: int, both_branches: bool, tag: str) -> dict:
    st, rhs_bench = c3_state(prob, seed, both_branches)
    ops = mg_.ElementOps2DGlue(prob.fine)
    bounds = rfem.DensityBounds.for_problem(prob.m, prob.volume, 0.0)
    t0 = time.perf_counter()
    ev = rpbm.eval_lagrangian(st, ops, prob.f, bounds, PEN)
    s_mat, rhs = rpbm.schur_system(ev, ops)
    out = {"seed": seed, "both_branches": both_branches, "value": ev.value, "res_alpha": ev.res_alpha,
           "tau_res": ev.tau_res, "corner": s_mat.corner}
    for name, vec in (("q", ev.q), ("rho_hat", ev.blocks.rho_hat), ("a", ev.blocks.a), ("b_lo", ev.blocks.b_lo),
                      ("b_up", ev.blocks.b_up), ("mu_hat_lo", ev.mu_hat_lo), ("mu_hat_up", ev.mu_hat_up),
                      ("res_lo", ev.res_lo), ("res_up", ev.res_up), ("res_u", ev.res_u), ("w", ev.blocks.w.ravel()),
                      ("rhs", rhs), ("border", s_mat.border)):
        put(out, name, vec, 11)
    rng = np.random.default_rng(1000 + seed)
    x = rng.standard_normal(prob.n + 1)
    put(out, "Sx", s_mat.matvec(x), 12)
    mg = rmg.MgPreconditioner(s_mat, prob.transfers)
    out["shifted"] = mg.shifted
    put(out, "vcycle_x", mg.apply(x), 13)
    put(out, "vcycle_rhs", mg.apply(rhs), 14)
    put(out, "vcycle_bench_rhs", mg.apply(rhs_bench), 15)
    for k, mat in enumerate(mg.mats):
        v = np.random.default_rng(2000 + k).standard_normal(mat.core_dim + 1)
        put(out, f"level{k}_apply", mat.matvec(v), 20 + k)
    du = 1e-2 * rng.standard_normal(prob.n)
    dalpha = float(1e-3 * rng.standard_normal())
    dnu_lo, dnu_up = rpbm.reconstruct_nu(ev, ops, du, dalpha)
    put(out, "dnu_lo", dnu_lo, 16)
    put(out, "dnu_up", dnu_up, 17)
    kappa = 0.5
    out["trial_value"] = rpbm._al_value(st.u + kappa * du, st.alpha + kappa * dalpha, st.nu_lo + kappa * dnu_lo,
                                        st.nu_up + kappa * dnu_up, st, ops, prob.f, bounds, PEN)
    print(f"[{tag}] eval/schur/mg/recon {time.perf_counter() - t0:.1f} s", flush=True)
    for name, b in (("rhs", rhs), ("bench_rhs", rhs_bench)):
        t0 = time.perf_counter()
        hist = []
        for k in range(1, 21):
            res = rlinalg.minres_solve(s_mat, b, rlinalg.MinresConfig(tol=1e-14, max_iters=k), mg.apply)
            hist.append(res.relres)
            if k == 20:
                put(out, f"minres20_x_{name}", res.x, 30)
        out[f"minres_hist_{name}"] = np.array(hist)
        print(f"[{tag}] minres history ({name}) {time.perf_counter() - t0:.1f} s", flush=True)
    t0 = time.perf_counter()
    res = rlinalg.minres_solve(s_mat, rhs, rlinalg.MinresConfig(tol=1e-6, max_iters=1000), mg.apply)
    out["minres_tol6_iters"] = res.iterations
    out["minres_tol6_relres"] = res.relres
    put(out, "minres_tol6_x", res.x, 31)
    print(f"[{tag}] minres tol 1e-6: {res.iterations} its, {time.perf_counter() - t0:.1f} s", flush=True)
    return out


def main(argv):
    which = set(argv) or {"c3", "c4"}
    meta_path = os.path.join(HERE, "golden_meta_fullsize.json")
    meta = json.load(open(meta_path)) if os.path.exists(meta_path) else {}
    meta["generator"] = "tests/golden/make_golden_fullsize.py"
    if "c3" in which:
        prob = mg_.build_config("C3")
        out = {}
        for tag, both in (("ref", False), ("br", True)):
            for k, v in c3_fixture(prob, 0, both, tag).items():
                out[f"{tag}_{k}"] = v
        np.savez_compressed(os.path.join(HERE, "c3_ref_samples.npz"), **out)
        meta["c3"] = {"ref_minres_tol6_iters": int(out["ref_minres_tol6_iters"]),
                      "br_minres_tol6_iters": int(out["br_minres_tol6_iters"])}
    if "c4" in which:
        prob = mg_.build_config("C4")
        out, rep = mg_.pbm_fixture(prob, with_vectors=False)
        out.pop("rho_sample_idx", None)
        out.pop("rho_sample", None)
        out["rho"] = rep.rho
        np.savez_compressed(os.path.join(HERE, "pbm_c4.npz"), **out)
        meta["pbm_c4"] = {"objective": rep.objective, "outer": rep.outer_iterations, **rep.totals(),
                          "wall_clock_s": rep.wall_clock}
    with open(meta_path, "w") as fh:
        json.dump(meta, fh, indent=1, default=float)
    print(json.dumps(meta, indent=1, default=float))


if __name__ == "__main__":
    main(sys.argv[1:])
