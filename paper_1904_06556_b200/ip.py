"""Primal-dual interior-point method on the device operators (the reference's ip.py).

Same classes, signatures, control flow and report as `vtsopt.ip` (ip.py:1-372):
one Newton step per outer iteration on the perturbed KKT residual, condensed to
the bordered (n+1) system S+ = K(rho) + sum_i (1/D_i) v_i v_i^T,
v_i = [K_i u; +1], solved by multigrid-preconditioned MINRES, then a stable
back-substitution and distinct fraction-to-boundary step lengths, with the
reference's one-iteration shift of the barrier parameters.

Every array operation runs in the library (`vts_ip_*` in include/vts_b200.h):
the KKT residual, the condensed system bound as the matrix-free operator the
PBM path uses (S+ differs from the PBM Newton matrix only by the sign of its
border; the context holds E S+ E, E = diag(I, -1), and flips border entries
at the API edge), the Galerkin V-cycle and MINRES unchanged, and the
reconstruction and step bounds.  The host keeps the scalars the reference
keeps in Python floats.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field, replace

import torch

from . import _lib
from .fem import DensityBounds, ElementOps, ptr
from .linalg import ComplementarityTolerance, MinresConfig, NewtonMatrix, minres_solve
from .multigrid import MgPreconditioner
from .pbm import SolveReport, _step

__all__ = ["IpConfig", "IpState", "IpResidual", "kkt_residual", "schur_system", "reconstruct", "step_lengths",
           "solve_ip"]


@dataclass
class IpConfig:
    """Interior-point parameters (ip.py:46-70)."""

    tol: float = 1e-5
    rho_lower: float = 1e-7
    sigma_r: float = 0.2
    sigma_s: float = 0.2
    barrier0: float = 1e-2
    boundary_frac: float = 0.9
    max_iters: int = 500
    stall_window: int = 15
    minres_tol0: float = 1e-2
    minres_floor: float = 1e-9
    minres_scale: float = 100.0
    minres_cap: int = 1000

    @classmethod
    def conditioning(cls, **overrides) -> "IpConfig":
        return replace(cls(rho_lower=1e-3), **overrides)


@dataclass
class IpState:
    """Strictly interior primal-dual iterate with staged barrier values (ip.py:73-85)."""

    u: torch.Tensor
    alpha: float
    rho: torch.Tensor
    nu_lo: torch.Tensor
    nu_up: torch.Tensor
    r: float
    s: float
    r_next: float = field(default=0.0)
    s_next: float = field(default=0.0)


@dataclass
class IpResidual:
    """The five KKT residual blocks (ip.py:100-111); `w` is recomputed on the device
    from `u` wherever the reference reuses it.  The extra scalars come from the same
    pass: f.u, sum rho, the barrier staging dots, comp_max, min_slack, min nu."""

    res_u: torch.Tensor
    res_alpha: float
    res_c: torch.Tensor
    res_lo: torch.Tensor
    res_up: torch.Tensor
    q: torch.Tensor
    u: torch.Tensor
    tau_res: float
    fu: float = 0.0
    rho_sum: float = 0.0
    lo_dot: float = 0.0
    up_dot: float = 0.0
    comp_max: float = 0.0
    min_slack: float = 0.0
    nu_min: float = 0.0


def _require_interior(res: IpResidual, state: IpState) -> None:
    """ip.py:88-97 from the residual pass's minima."""
    if not (res.min_slack > 0.0 and res.nu_min > 0.0):
        raise ValueError("iterate lost strict interiority")
    if not (state.r > 0.0 and state.s > 0.0):
        raise ValueError("barrier parameters must stay positive")


def kkt_residual(state: IpState, ops: ElementOps, f, bounds: DensityBounds) -> IpResidual:
    """Perturbed KKT residual at a strictly interior state (ip.py:114-134)."""
    m, n = ops.m, ops.n
    u = ops.check_vec(state.u, n, "u")
    q, res_c, res_lo, res_up = (ops.vec(m) for _ in range(4))
    res_u = ops.vec(n)
    sc = (ctypes.c_double * 9)()
    rc = _lib.load().vts_ip_residual(ops.handle, ptr(u), float(state.alpha), ptr(state.rho), ptr(state.nu_lo),
                                     ptr(state.nu_up), float(state.r), float(state.s), ptr(bounds.lower),
                                     ptr(bounds.upper), float(bounds.volume), ptr(f), ops.norm_f, ptr(q),
                                     ptr(res_c), ptr(res_lo), ptr(res_up), ptr(res_u), sc)
    _lib.check(rc, "vts_ip_residual")
    res = IpResidual(res_u, sc[0], res_c, res_lo, res_up, q, u, sc[1], fu=sc[2], rho_sum=sc[3], lo_dot=sc[4],
                     up_dot=sc[5], comp_max=sc[6], min_slack=sc[7], nu_min=sc[8])
    _require_interior(res, state)
    return res


def schur_system(state: IpState, res: IpResidual, ops: ElementOps, bounds: DensityBounds):
    """Doubly condensed (n+1) system (ip.py:137-158): (S+, rhs, D, g)."""
    _require_interior(res, state)
    m, n = ops.m, ops.n
    dcoef, g = ops.vec(m), ops.vec(m)
    rhs = ops.vec(n + 1)
    corner = ctypes.c_double(0.0)
    rc = _lib.load().vts_ip_schur_system(ops.handle, ptr(res.u), ptr(state.rho), ptr(state.nu_lo),
                                         ptr(state.nu_up), ptr(bounds.lower), ptr(bounds.upper), ptr(res.res_c),
                                         ptr(res.res_lo), ptr(res.res_up), ptr(res.res_u), float(res.res_alpha),
                                         ptr(dcoef), ptr(g), ptr(rhs), ctypes.byref(corner))
    _lib.check(rc, "vts_ip_schur_system")
    ops._system_version = getattr(ops, "_system_version", 0) + 1
    mat = NewtonMatrix(ops, None, corner.value, ops._system_version)
    mat.border_sign = 1.0
    return mat, rhs, dcoef, g


def reconstruct(state: IpState, res: IpResidual, ops: ElementOps, bounds: DensityBounds, du, dalpha: float,
                dcoef, g):
    """Back-substitute (d_rho, d_nu_up, d_nu_lo) (ip.py:161-186)."""
    m = ops.m
    du = ops.check_vec(du, ops.n, "du")
    drho, dnu_up, dnu_lo = ops.vec(m), ops.vec(m), ops.vec(m)
    rc = _lib.load().vts_ip_reconstruct(ops.handle, ptr(res.u), ptr(du), float(dalpha), ptr(dcoef), ptr(g),
                                        ptr(res.res_c), ptr(res.res_lo), ptr(res.res_up), ptr(state.rho),
                                        ptr(state.nu_lo), ptr(state.nu_up), ptr(bounds.lower), ptr(bounds.upper),
                                        ptr(drho), ptr(dnu_up), ptr(dnu_lo))
    _lib.check(rc, "vts_ip_reconstruct")
    return drho, dnu_up, dnu_lo


def step_lengths(state: IpState, drho, dnu_lo, dnu_up, bounds: DensityBounds, frac: float = 0.9, ops=None):
    """(kappa_primal, kappa_nu_lo, kappa_nu_up), all in (0, 1] (ip.py:197-222)."""
    if ops is None:
        raise TypeError("step_lengths needs the ElementOps context of the state")
    mins = (ctypes.c_double * 4)()
    rc = _lib.load().vts_ip_step_bounds(ops.handle, ptr(state.rho), ptr(drho), ptr(state.nu_lo), ptr(dnu_lo),
                                        ptr(state.nu_up), ptr(dnu_up), ptr(bounds.lower), ptr(bounds.upper), mins)
    _lib.check(rc, "vts_ip_step_bounds")
    up, dn, lo_nu, up_nu = mins
    kappa = 1.0
    if math.isfinite(up):
        kappa = min(kappa, frac * up)
    if math.isfinite(dn):
        kappa = min(kappa, frac * dn)
    # _boundary_step (ip.py:189-194)
    k_lo = min(1.0, frac * lo_nu) if math.isfinite(lo_nu) else 1.0
    k_up = min(1.0, frac * up_nu) if math.isfinite(up_nu) else 1.0
    return kappa, k_lo, k_up


def _gap(ops, state: IpState, res: IpResidual, f, bounds: DensityBounds):
    """duality_gap(-alpha, q, f.u, bounds) (model.py:69-79) and f.u, in one device pass."""
    d_val, gap, fu, rho_sum = (ctypes.c_double() for _ in range(4))
    rc = _lib.load().vts_gap(ops.handle, ptr(state.u), -float(state.alpha), ptr(res.q), ptr(f), ptr(state.nu_lo),
                             ptr(state.nu_up), ptr(bounds.lower), ptr(bounds.upper), float(bounds.volume),
                             ptr(state.rho), ctypes.byref(d_val), ctypes.byref(gap), ctypes.byref(fu),
                             ctypes.byref(rho_sum))
    _lib.check(rc, "vts_gap")
    return gap.value, fu.value, rho_sum.value


def solve_ip(problem, cfg: IpConfig | None = None, ops: ElementOps | None = None) -> SolveReport:
    """Run the interior-point method on a problem instance (ip.py:225-372)."""
    cfg = cfg or IpConfig()
    t0 = time.perf_counter()
    ops = ops or ElementOps(problem.fine)
    bounds = DensityBounds.for_problem(problem.m, problem.volume, cfg.rho_lower)
    f = problem.f
    m, n = problem.m, problem.n
    dev = dict(dtype=torch.float64, device="cuda")
    state = IpState(u=torch.zeros(n, **dev), alpha=1.0, rho=torch.full((m,), problem.volume / m, **dev),
                    nu_lo=torch.ones(m, **dev), nu_up=torch.ones(m, **dev), r=cfg.barrier0, s=cfg.barrier0)
    mtol = ComplementarityTolerance(tol=cfg.minres_tol0, floor=cfg.minres_floor, scale=cfg.minres_scale)
    res = kkt_residual(state, ops, f, bounds)
    # stage the first shifted update from the initial iterate (ip.py:244-246)
    state.r_next = cfg.sigma_r * res.lo_dot / m
    state.s_next = cfg.sigma_s * res.up_dot / m

    columns = ("iter", "minres", "gap_scaled", "tau_res", "r", "s", "min_slack")
    rows: list = []
    notes: list = []
    converged = False
    gap_scaled = math.inf
    best_gap = math.inf
    since_best = 0
    fu = 0.0
    for it in range(1, cfg.max_iters + 1):
        mtol.observe(res.comp_max)  # ip.py:270-274, from the current state's residual pass
        s_mat, rhs, dcoef, g = schur_system(state, res, ops, bounds)
        chain = MgPreconditioner(s_mat, problem.transfers)
        sol = minres_solve(s_mat, rhs, MinresConfig(tol=mtol.current(), max_iters=cfg.minres_cap,
                                                    floor=cfg.minres_floor), chain.apply)
        du, dalpha = sol.x[:-1].contiguous(), float(sol.x[-1])
        drho, dnu_up, dnu_lo = reconstruct(state, res, ops, bounds, du, dalpha, dcoef, g)
        # shifted barrier update (ip.py:290-292)
        state.r, state.s = state.r_next, state.s_next
        kappa_p, kappa_lo, kappa_up = step_lengths(state, drho, dnu_lo, dnu_up, bounds, cfg.boundary_frac, ops)
        state.u = _step(state.u, kappa_p, du, ops)
        state.alpha = state.alpha + dalpha
        state.rho = _step(state.rho, kappa_p, drho, ops)
        state.nu_lo = _step(state.nu_lo, kappa_lo, dnu_lo, ops)
        state.nu_up = _step(state.nu_up, kappa_up, dnu_up, ops)

        res = kkt_residual(state, ops, f, bounds)
        delta, fu, _ = _gap(ops, state, res, f, bounds)
        objective = 0.5 * fu
        gap_scaled = delta / objective
        rows.append((it, sol.iterations, gap_scaled, res.tau_res, state.r, state.s, res.min_slack))
        if cfg.tol > gap_scaled > -0.1 * cfg.tol and res.tau_res < 10.0 * cfg.tol:
            converged = True
            break
        state.r_next = cfg.sigma_r * res.lo_dot / m
        state.s_next = cfg.sigma_s * res.up_dot / m
        if abs(gap_scaled) < best_gap:
            best_gap = abs(gap_scaled)
            since_best = 0
        else:
            since_best += 1
            if since_best >= cfg.stall_window:
                notes.append(f"no convergence apparent: scaled gap did not improve for {cfg.stall_window} "
                             "iterations")
                break
    else:
        notes.append("iteration cap reached without meeting the stopping band")
    if cfg.rho_lower >= 1e-3:
        notes.append(f"conditioning profile rho_lower={cfg.rho_lower:g}: objective not comparable with "
                     "default-bound runs")
    certificate = None
    if converged:
        certificate = (f"duality gap / objective = {gap_scaled:.6e} within ({-0.1 * cfg.tol:.1e}, {cfg.tol:.1e}); "
                       f"feasibility {res.tau_res:.6e} < {10.0 * cfg.tol:.1e}")
    return SolveReport(
        method="ip", problem=problem.name, tol=cfg.tol, converged=converged, columns=columns, rows=rows,
        count_columns=("minres",), objective=0.5 * fu, dual_objective=math.nan, gap_scaled=gap_scaled,
        tau_res=res.tau_res, volume=res.rho_sum, rho=state.rho.clone(), wall_clock=time.perf_counter() - t0,
        notes="; ".join(notes), certificate=certificate,
        extras={"u": state.u, "alpha": state.alpha, "nu_lo": state.nu_lo, "nu_up": state.nu_up,
                "minres_tol_final": mtol.current()})
