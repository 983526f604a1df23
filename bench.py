"""Benchmark: MG-preconditioned MINRES on the 1024x512 VTS Newton system (BASELINE.json configs[2]).

A "step" is one preconditioned MINRES iteration (linalg.py:190-242) on the
bordered Schur system of the C3 microbench state: one matrix-free Newton apply,
one V(2,2) cycle with exact-order Gauss-Seidel on 9 levels, and the Lanczos /
Givens vector updates.  `value` = MINRES iterations/s with all inputs resident
in HBM; `e2e` = the same through the C-ABI call with the right-hand side
copied host->device and the solution device->host inside the timed region.
Inputs (the per-level stencils alone are 226 MB) exceed the 126 MB L2, so no
explicit flush is needed.  Extra keys report the other BASELINE.json figures
(phi pass, 100 applies, 100 V-cycles, full-PBM wall time of C4) and the
roofline of the dominant kernel.

`--impl reference` times the reference's CPU algorithm (the oracle port in
`oracle/`, test infrastructure) on the same workload; under torchrun only
rank 0 runs it.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "MG-MINRES iters/s + HBM GB/s (frac of 8 TB/s) on VTS Newton system; PBM wall s"
CONFIG_KEY = "C3"
N_ELEM_X, N_ELEM_Y = 1024, 512


def microbench_inputs(n: int, m: int, seed: int = 0):
    """BASELINE.json configs[2]: u ~ N(0, 1e-4) per free dof, alpha = 1e-3,
    rho ~ U(0.5, 2), p = 1e-2, other fields at the reference's initial values,
    RHS ~ N(0, 1) of length n + 1."""
    rng = np.random.default_rng(seed)
    u = rng.normal(0.0, 1e-2, n)
    rho = rng.uniform(0.5, 2.0, m)
    rhs = rng.standard_normal(n + 1)
    one = np.ones(m)
    state = dict(u=u, alpha=1e-3, nu_lo=one.copy(), nu_up=one.copy(), rho=rho, mu_lo=one.copy(),
                 mu_up=one.copy(), p=np.full(m, 1e-2), q_lo=one.copy(), q_up=one.copy())
    return state, rhs


def workload_config(n: int, m: int, world: int) -> dict:
    """The `config` both arms print (identical dicts, so the driver can pair them)."""
    return {"workload": "C3 microbench: preconditioned MINRES on the 1024x512 cantilever Newton system, "
                        "9 MG levels, V(2,2) exact-order GS", "n": n, "m": m, "seed": 0,
            "parallelism": "replicas only" if world > 1 else "single GPU",
            "l2": "inputs > 126 MB L2 (stencils 226 MB), no flush"}


def algorithmic_bytes(prob) -> dict:
    """SURVEY.md Appendix B byte model (fp64 words x 8)."""
    n, m = prob.n, prob.m
    lv = prob.levels
    A_phi = 8 * (4 * n + 16 * m)
    A_ap = 8 * (3 * n + 2 * m + 2)
    A_V = 0
    for k in range(1, len(lv)):  # every level but the coarsest
        nk, nkm1 = lv[k].n, lv[k - 1].n
        Bk = 8 * (nk + 2 * m) if k == len(lv) - 1 else 76 * nk
        A_V += 5 * (Bk + 32 * nk) + 24 * (nk + nkm1)
    A_MR = A_ap + A_V + 160 * (n + 1)
    # one forward GS sweep on the finest level: operator (matrix-free credit) + b, x, x', border
    A_gs = (8 * (n + 2 * m) + 32 * n)
    # one finest-level wavefront launch (k_gs_tri): per grid node the 20-double
    # half-stencil it solves with, the 2-double right-hand side P, the 2-double result
    fine = lv[-1]
    A_tri = fine.nx * fine.ny * 8 * (20 + 2 + 2)
    # one finest-level sweep pair (k_gs_pair), per node: sweep B reads the 20-double
    # solve half, 18 doubles of the other half, b, border and sweep A's result and
    # writes its own (46 doubles); descent sweep A (zero guess) reads the solve half,
    # b, border and writes its result (26); ascent sweep A builds its P like B (46)
    nodes = fine.nx * fine.ny
    B_side = 20 + 18 + 2 + 2 + 2 + 2
    A_pair = nodes * 8 * ((20 + 2 + 2 + 2) + B_side)
    A_pair_asc = nodes * 8 * (B_side + B_side)
    return dict(phi=A_phi, apply=A_ap, vcycle=A_V, minres_iter=A_MR, gs_fine_sweep=A_gs, gs_tri_fine=A_tri,
                gs_pair_fine=A_pair, gs_pair_asc_fine=A_pair_asc)


def ncu_traffic(kernel: str = "k_gs_tri"):
    """dram bytes per finest-level launch of `kernel` from the committed ncu --set full capture."""
    import csv

    for rnd in ("r02", "r01"):
        path = os.path.join(REPO, "profiles", f"{rnd}_ncu_full_{kernel}_fine_raw_subset.csv")
        if os.path.exists(path):
            break
    try:
        with open(path) as fh:
            rows = list(csv.reader(fh))
        head, units, vals = rows[0], rows[1], rows[2]
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot = 0.0
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = head.index(key)
            tot += float(vals[i].replace(",", "")) * scale[units[i]]
        return tot
    except (OSError, ValueError, KeyError, IndexError):
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) == 7:
                    self.rows.append(parts)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def aggregate_over_ranks(elapsed, units, world: int, device: str):
    """Replicas-only multi-GPU: every rank solves its own system;
    the job's time is the max over ranks and its work the sum over ranks."""
    if world <= 1:
        return float(elapsed), float(units)
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(elapsed)], dtype=torch.float64, device=device)
    u = torch.tensor([float(units)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(u, op=dist.ReduceOp.SUM)
    return float(t.item()), float(u.item())


def run_reference(args) -> None:
    """CPU reference arm: the oracle port of the reference algorithm, same workload."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle

    prob = oracle.build_config(CONFIG_KEY)
    st, rhs = microbench_inputs(prob.n, prob.m)
    ops = oracle.ElementOps2D(prob.fine)
    bounds = oracle.DensityBounds.for_problem(prob.m, prob.volume, 0.0)
    ev = oracle.eval_lagrangian(oracle.PbmState(**st), ops, prob.f, bounds, oracle.PenaltyBarrier())
    mat, _ = oracle.schur_system(ev, ops)
    mg = oracle.MgPreconditioner(mat, prob.transfers)
    oracle.minres_solve(mat, rhs, oracle.MinresConfig(tol=1e-14, max_iters=max(args.warmup, 1)), mg.apply)
    t0 = time.perf_counter()
    res = oracle.minres_solve(mat, rhs, oracle.MinresConfig(tol=1e-14, max_iters=args.steps), mg.apply)
    dt = time.perf_counter() - t0
    its = res.iterations
    value = its / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "MINRES iterations/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / its, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE configs[2])",
        "config": workload_config(prob.n, prob.m, world),
        "cpu_baseline": {"value": value, "unit": "MINRES iterations/s", "cores": 1, "kind": "port",
                         "sample": f"{its} preconditioned MINRES iterations on the C3 Newton system "
                                   "(oracle/ restatement: numpy/scipy CSR + sequential C Gauss-Seidel, "
                                   "single-threaded by construction)", **host_cores()},
        "e2e": {"value": value, "unit": "MINRES iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def host_cores() -> dict:
    """Host CPU resources of this box (cpu_count and affinity)."""
    aff = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None
    return {"os_cpu_count": os.cpu_count(), "sched_getaffinity": aff}


def cpu_baseline_sample() -> dict:
    """Bounded oracle sample on the host (rank 0, N=1), about 10 s of CPU work.

    The value is MINRES iterations/s (10 iterations on C3).  Beside it, the
    other north_star figures on the same inputs: the phi pass (with the BLAS
    pool at its default size and at one thread, the OPENBLAS_NUM_THREADS=1
    run SURVEY.md §8(d) asks for, via threadpoolctl), the Galerkin/Cholesky
    setup, one Newton-matrix apply (mean of 50) and one V-cycle (mean of 5).
    The Gauss-Seidel loops (C) and scipy's CSR kernels are single-threaded.
    """
    import oracle
    from threadpoolctl import threadpool_info, threadpool_limits

    prob = oracle.build_config(CONFIG_KEY)
    st, rhs = microbench_inputs(prob.n, prob.m)
    ops = oracle.ElementOps2D(prob.fine)
    bounds = oracle.DensityBounds.for_problem(prob.m, prob.volume, 0.0)

    def phi():
        return oracle.eval_lagrangian(oracle.PbmState(**st), ops, prob.f, bounds, oracle.PenaltyBarrier())

    phi()
    t0 = time.perf_counter()
    ev = phi()
    t_phi = time.perf_counter() - t0
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        phi()
        t_phi1 = time.perf_counter() - t0
    mat, _ = oracle.schur_system(ev, ops)
    t0 = time.perf_counter()
    mg = oracle.MgPreconditioner(mat, prob.transfers)
    t_setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    for _ in range(50):
        mat.matvec(rhs)
    t_apply = (time.perf_counter() - t0) / 50
    t0 = time.perf_counter()
    for _ in range(5):
        mg.apply(rhs)
    t_vc = (time.perf_counter() - t0) / 5
    its = 10
    t0 = time.perf_counter()
    res = oracle.minres_solve(mat, rhs, oracle.MinresConfig(tol=1e-14, max_iters=its), mg.apply)
    dt = time.perf_counter() - t0
    blas = [p.get("num_threads") for p in threadpool_info() if p.get("user_api") == "blas"]
    return {"value": res.iterations / dt, "unit": "MINRES iterations/s", "cores": 1, "kind": "port",
            "sample": f"{res.iterations} preconditioned MINRES iterations on the C3 Newton system "
                      f"({dt:.1f} s); oracle/ restatement, single thread (C Gauss-Seidel, scipy CSR)",
            **host_cores(), "blas_threads_default": blas[0] if blas else None,
            "phi_pass_ms": 1e3 * t_phi, "phi_pass_ms_blas1": 1e3 * t_phi1, "mg_setup_ms": 1e3 * t_setup,
            "apply_ms": 1e3 * t_apply, "vcycle_ms": 1e3 * t_vc,
            "pbm_c4_wall_s_recorded": recorded_c4_wall(),
            "note": "pbm_c4_wall_s_recorded: the unmodified reference (+2D glue) full C4 solve, timed when "
                    "tests/golden/make_golden_fullsize.py ran on the build container (not this box: ~4 min)"}


def recorded_c4_wall():
    try:
        with open(os.path.join(REPO, "tests", "golden", "golden_meta_fullsize.json")) as fh:
            return json.load(fh)["pbm_c4"]["wall_clock_s"]
    except (OSError, KeyError, ValueError):
        return None


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-pbm", action="store_true", help="skip the C4 full-PBM wall-time extra")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
        return

    import ctypes

    import torch
    import torch.distributed as dist

    import paper_1904_06556_b200 as vts
    from paper_1904_06556_b200 import _lib
    from paper_1904_06556_b200.fem import ptr

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl")
    lib = _lib.load()
    prob = vts.build_config(CONFIG_KEY)
    n, m = prob.n, prob.m
    st_h, rhs_h = microbench_inputs(n, m, seed=rank)
    st = vts.PbmState(**{k: (v if k == "alpha" else torch.as_tensor(v, device="cuda")) for k, v in st_h.items()})
    ops = vts.ElementOps(prob.fine)
    bounds = vts.DensityBounds.for_problem(m, prob.volume, 0.0)
    pen = vts.PenaltyBarrier()
    stream = torch.cuda.current_stream()

    # --- phi pass (K1) timed with events
    for _ in range(3):
        ev = vts.eval_lagrangian(st, ops, prob.f, bounds, pen)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    reps_phi = 10
    for _ in range(reps_phi):
        ev = vts.eval_lagrangian(st, ops, prob.f, bounds, pen)
    e1.record(stream)
    torch.cuda.synchronize()
    phi_ms = e0.elapsed_time(e1) / reps_phi
    mat, _ = vts.schur_system(ev, ops)
    t_setup0 = time.perf_counter()
    mg = vts.MgPreconditioner(mat, prob.transfers)
    setup_wall_ms = 1e3 * (time.perf_counter() - t_setup0)
    rhs = torch.as_tensor(rhs_h, device="cuda")
    x = torch.empty(n + 1, dtype=torch.float64, device="cuda")
    itv, rel, conv = ctypes.c_int32(), ctypes.c_double(), ctypes.c_int32()

    def minres_dev(k: int) -> int:
        rc = lib.vts_minres(ops.handle, ptr(rhs), ptr(x), 1e-14, k, 1e-9, 1, ctypes.byref(itv), ctypes.byref(rel),
                            ctypes.byref(conv), None)
        _lib.check(rc, "vts_minres")
        return itv.value

    # --- per-kernel device times (roofline) and the 100-apply / 100-V-cycle figures
    kms = (ctypes.c_double * 6)()
    _lib.check(lib.vts_time_kernels(ops.handle, 100, kms), "vts_time_kernels")
    apply_warm_ms, vcycle_ms, gs_fine_ms, gs_l2_ms, resid_warm_ms, setup_ms = list(kms)
    # the apply's and the residual's inputs (34 / 118 MB) fit in the 126 MB L2, so
    # back-to-back launches would read L2: time them cold (L2 overwritten before
    # each launch), as they run inside a MINRES iteration
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    cold = (ctypes.c_double * 2)()
    _lib.check(lib.vts_time_cold(ops.handle, 50, flush.data_ptr(), flush.numel(), cold), "vts_time_cold")
    apply_ms, resid_ms = list(cold)
    # the same cold launch after a read sweep (L2 clean, as ncu's cache flush leaves it), and
    # this harness's floor: a plain streaming kernel over the apply's bytes (VTS_TIME_FLOOR)
    apply_cold = {}
    for flush_kind in ("memset", "read"):
        os.environ["VTS_COLD_FLUSH"], os.environ["VTS_TIME_FLOOR"] = flush_kind, "1"
        _lib.check(lib.vts_time_cold(ops.handle, 50, flush.data_ptr(), flush.numel(), cold), "vts_time_cold")
        apply_cold[flush_kind] = (cold[0], cold[1])
    os.environ.pop("VTS_COLD_FLUSH")
    os.environ.pop("VTS_TIME_FLOOR")
    del flush

    # --- warm-up then the timed region: K MINRES iterations, device resident
    minres_dev(args.warmup)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ops.kernel_launches
    with ClockSampler(local) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        its = minres_dev(args.steps)
        t1.record(stream)
        torch.cuda.synchronize()
    launches = ops.kernel_launches - launches0
    dt_ms, total_its = aggregate_over_ranks(t0.elapsed_time(t1), its, world, "cuda")
    value = total_its / (dt_ms * 1e-3)

    # --- profiling pass (not the timed value): the same K iterations with every
    # wavefront launch bracketed by CUDA events on the context stream, giving the
    # dominant kernel's average launch time and its share of the step
    prof = (ctypes.c_double * 8)()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    _lib.check(lib.vts_profile_begin(ops.handle), "vts_profile_begin")
    p0.record(stream)
    minres_dev(args.steps)
    p1.record(stream)
    _lib.check(lib.vts_profile_end(ops.handle, prof), "vts_profile_end")
    prof_region_ms = p0.elapsed_time(p1)
    (gs_total_ms, gs_n, tri_fine_ms, tri_fine_n, pair_fine_ms, pair_fine_n, asc_fine_ms,
     asc_fine_n) = list(prof)

    # --- e2e through the C-ABI with host buffers (pinned), copies inside the timed region
    rhs_host = torch.as_tensor(rhs_h).pin_memory()
    x_host = torch.empty(n + 1, dtype=torch.float64).pin_memory()
    rhs_dev = torch.empty(n + 1, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    rhs_dev.copy_(rhs_host, non_blocking=True)
    rc = lib.vts_minres(ops.handle, ptr(rhs_dev), ptr(x), 1e-14, args.steps, 1e-9, 1, ctypes.byref(itv),
                        ctypes.byref(rel), ctypes.byref(conv), None)
    _lib.check(rc, "vts_minres")
    x_host.copy_(x, non_blocking=True)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - w0
    e2e_s, e2e_its = aggregate_over_ranks(e2e_s, itv.value, world, "cuda")
    e2e_value = e2e_its / e2e_s

    bytes_ = algorithmic_bytes(prob)
    peaks_path = os.path.join(REPO, "MEASURED_PEAKS.json")
    peak, peak_src = 6526.8, "MEASURED_PEAKS.json hbm_gbs"
    if os.path.exists(peaks_path):
        with open(peaks_path) as fh:
            peak = float(json.load(fh).get("hbm_gbs", peak))
    else:
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"

    def gbs(nbytes, ms):
        return nbytes / (ms * 1e-3) / 1e9

    # dominant kernel of the MINRES iteration: the wavefront Gauss-Seidel kernel,
    # k_gs_pair (both sweeps of a smoothing step) when the pipelined pairs ran,
    # else k_gs_tri; roofline unit = one finest-level launch (for the pair: the
    # descent pair, the launch the committed ncu capture is of; the ascent pair's
    # time and bytes are reported beside it)
    # roofline credit = SURVEY.md §8(d)'s matrix-free algorithmic bytes: a finest
    # sweep pair is two finest sweeps (2 x [8(n+2m) + 32n]), a single sweep one;
    # the implementation's own reads (assembled half-stencils) are reported beside it
    if pair_fine_n > 0:
        dom, dom_ms, dom_n = "k_gs_pair", pair_fine_ms, pair_fine_n
        dom_bytes, impl_bytes = 2 * bytes_["gs_fine_sweep"], bytes_["gs_pair_fine"]
    else:
        dom, dom_ms, dom_n = "k_gs_tri", tri_fine_ms, tri_fine_n
        dom_bytes, impl_bytes = bytes_["gs_fine_sweep"], bytes_["gs_tri_fine"]
    dom_avg_ms = dom_ms / max(dom_n, 1.0)
    achieved = gbs(dom_bytes, dom_avg_ms)
    traffic = ncu_traffic(dom)
    pbm = None
    if not args.no_pbm and rank == 0:
        # the microbenchmark's context goes first: its device arena returns to the
        # library's pool and the solve's context reuses it (as a solver creating one
        # context per problem does from its second problem on)
        del mat, mg, ev, ops
        import gc

        gc.collect()
        torch.cuda.synchronize()
        def timed_solves(reps):
            walls, last = [], None
            for _ in range(reps):
                torch.cuda.synchronize()
                t_p = time.perf_counter()
                last = vts.solve_pbm(vts.build_config("C4"))
                torch.cuda.synchronize()
                walls.append(time.perf_counter() - t_p)
            return walls, last

        # three solves per mode (each: mesh build, context creation, solve): the first one of a
        # process also pays one-time costs (graph instantiation, pool growth) that vary by 0.1 s
        walls, rep = timed_solves(3)
        pbm = {"config": "C4 full PBM 1024x512 cantilever", "wall_s": sorted(walls)[1], "wall_s_runs": walls,
               "note": "median of three solve_pbm calls, each with its mesh build and context creation (device "
                       "arena recycled from the microbenchmark context); each Newton step one vts_newton_step "
                       "(device-resident, CUDA graphs, one host synchronisation per step); wall_s_runs[0] is "
                       "the process's first solve",
               "outer": rep.outer_iterations, **rep.totals(), "compliance": rep.objective,
               "converged": rep.converged}
        os.environ["VTS_HOST_NEWTON"] = "1"  # the call-by-call host orchestration, same kernels (same bits)
        walls_h, rep_h = timed_solves(3)
        pbm["host_orchestrated_wall_s"] = sorted(walls_h)[1]
        pbm["host_orchestrated_wall_s_runs"] = walls_h
        pbm["host_orchestrated_same_result"] = bool(rep_h.objective == rep.objective and rep_h.rows == rep.rows)
        os.environ.pop("VTS_HOST_NEWTON")
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_sample()
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": value, "unit": "MINRES iterations/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt_ms / its, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE configs[2] state and RHS)",
        "config": workload_config(n, m, world),
        "e2e": {"value": e2e_value, "unit": "MINRES iterations/s", "h2d_bytes_per_step": 8 * (n + 1) / args.steps,
                "d2h_bytes_per_step": 8 * (n + 1) / args.steps,
                "note": "one C-ABI vts_minres call of K iterations; RHS H2D and solution D2H once per call"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "limited_by": "latency: the exact-order Gauss-Seidel wavefront is a chain "
                                                   "of nx + 2 ny dependent block solves (DESIGN.md §4)",
                     "kernel": f"{dom}, finest level (1025x513 wavefront"
                               f"{' sweep pair' if dom == 'k_gs_pair' else ' sweep'})",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "frac_of_8TBs": achieved / 8000.0, "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": dom_bytes,
                     "algorithmic_bytes_rule": "SURVEY.md §8(d) / Appendix B matrix-free sweep bytes "
                                               "8(n+2m)+32n per finest sweep, x2 for a pair",
                     "implementation_bytes_per_launch": impl_bytes,
                     "implementation_GBs": gbs(impl_bytes, dom_avg_ms),
                     "launch_ms": dom_avg_ms,
                     "launches_in_profiled_region": int(gs_n), "finest_launches": int(dom_n),
                     "share_of_step": gs_total_ms / prof_region_ms,
                     "ascent_pair": ({"launch_ms": asc_fine_ms / asc_fine_n,
                                      "algorithmic_bytes_per_launch": 2 * bytes_["gs_fine_sweep"],
                                      "achieved": gbs(2 * bytes_["gs_fine_sweep"], asc_fine_ms / asc_fine_n),
                                      "implementation_bytes_per_launch": bytes_["gs_pair_asc_fine"]}
                                     if asc_fine_n > 0 else None),
                     "apply_frac": gbs(bytes_["apply"], apply_ms) / peak,
                     "apply_note": "k_newton_apply, A_ap = 8(3n+2m+2) per launch, timed cold (L2 overwritten "
                                   "by a memset: every miss also writes a dirty line back)",
                     "apply_frac_clean_l2": gbs(bytes_["apply"], apply_cold["read"][0]) / peak,
                     "apply_harness_floor": {
                         "note": "a plain grid-stride kernel reading and writing the apply's bytes, timed the same "
                                 "way: what a launch + cold-L2 measurement of this size can reach",
                         "floor_ms_dirty_l2": apply_cold["memset"][1], "floor_ms_clean_l2": apply_cold["read"][1],
                         "apply_ms_clean_l2": apply_cold["read"][0],
                         "apply_over_floor_dirty": apply_ms / apply_cold["memset"][1],
                         "apply_over_floor_clean": apply_cold["read"][0] / apply_cold["read"][1]},
                     "vcycle_frac": gbs(bytes_["vcycle"], vcycle_ms) / peak,
                     "vcycle_note": "one V(2,2), A_V of SURVEY.md Appendix B, mean of 100 back-to-back",
                     "phi_frac": gbs(bytes_["phi"], phi_ms) / peak,
                     "minres_iter_frac": gbs(bytes_["minres_iter"], dt_ms / its) / peak,
                     "note": "traffic = dram bytes per launch from the committed ncu --set full capture "
                             "(profiles/)"},
        "kernels": {
            "phi_pass_ms": phi_ms, "phi_pass_GBs": gbs(bytes_["phi"], phi_ms),
            "apply_ms": apply_ms, "apply_GBs": gbs(bytes_["apply"], apply_ms), "applies_per_s": 1e3 / apply_ms,
            "apply_frac": gbs(bytes_["apply"], apply_ms) / peak,
            "apply_l2_warm_ms": apply_warm_ms, "residual_l2_warm_ms": resid_warm_ms,
            "note": "apply and residual timed cold (256 MB written between launches); phi pass: 10 back-to-back "
                    "vts_eval_lagrangian calls, each one k_phi_tile launch plus its scalar read-back and host "
                    "synchronisation (100 MB of inputs, partly L2-resident)",
            "vcycle_ms": vcycle_ms, "vcycles_per_s": 1e3 / vcycle_ms,
            "gs_fine_sweep_ms": gs_fine_ms, "gs_fine_sweep_GBs": gbs(bytes_["gs_fine_sweep"], gs_fine_ms),
            "gs_level8_sweep_ms": gs_l2_ms, "residual_fine_ms": resid_ms, "mg_setup_ms": setup_ms,
            "mg_setup_wall_ms": setup_wall_ms,
            "minres_iter_GBs": gbs(bytes_["minres_iter"], dt_ms / its),
            "minres_iter_frac_of_8TBs": gbs(bytes_["minres_iter"], dt_ms / its) / 8000.0,
            "algorithmic_bytes": bytes_,
        },
        "clocks": clk.summary(),
    }
    if pbm:
        line["pbm"] = pbm
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
