"""Penalty-barrier multiplier method: the inner Newton step on B200.

Mirrors the reference's `pbm.py` call for call (same names, arguments,
return types and stopping logic), with every array a CUDA fp64 tensor and
every array operation a fused kernel behind the C ABI:

* `eval_lagrangian`  (pbm.py:150-199) -> vts_eval_lagrangian (one element
  pass + one node pass + a deterministic reduction)
* `schur_system`     (pbm.py:202-218) -> vts_schur_system; the Newton matrix
  stays matrix-free in the context (`NewtonMatrix`)
* `reconstruct_nu`   (pbm.py:221-232) -> vts_reconstruct_nu (+ the slope)
* `_al_value`        (pbm.py:135-147) -> vts_al_value, fused with x + kappa dx
* `newton_inner`     (pbm.py:244-338), `solve_pbm` (pbm.py:341-465) — host
  control flow identical to the reference; only scalars cross to the host.
  On a 2D context each Newton step is one vts_newton_step call (device-resident:
  Schur system, multigrid setup, MINRES, reconstruction, Armijo search, update
  and the new evaluation with one host synchronisation; two CUDA graphs);
  VTS_HOST_NEWTON=1 runs the call-by-call path above instead (same bits).
"""

from __future__ import annotations

import ctypes
import logging
import os
import time
from dataclasses import dataclass, field, replace
from math import sqrt

import torch

from . import _lib
from .fem import DensityBounds, ElementOps, ptr
from .linalg import _ERRORS, MinresConfig, MinresError, NewtonMatrix, StagnationTolerance, minres_solve
from .multigrid import MgPreconditioner
from .penalty import PenaltyBarrier, warn_saturated

__all__ = [
    "PbmConfig",
    "PbmState",
    "HessianBlocks",
    "LagrangianEval",
    "eval_lagrangian",
    "schur_system",
    "reconstruct_nu",
    "al_value",
    "newton_inner",
    "solve_pbm",
    "SolveReport",
]


@dataclass
class PbmConfig:
    """Parameters of the multiplier method (pbm.py:56-82, same defaults)."""

    tol: float = 1e-5
    rho_lower: float = 0.0
    beta: float = 0.3
    gamma: float = 0.3
    penalty_floor: float = 1e-8
    tol_newton0: float = 1.0
    tol_newton_min: float = 1e-3
    armijo_c1: float = 1e-4
    armijo_shrink: float = 0.5
    armijo_max_halvings: int = 40
    max_outer: int = 60
    max_newton: int = 150
    stall_steps: int = 3
    minres_tol_scale: float = 1e-4
    minres_floor: float = 1e-9
    minres_cap: int = 1000
    branch: float = -0.5

    @classmethod
    def large(cls, **overrides) -> "PbmConfig":
        cfg = cls(beta=0.5, gamma=0.5, minres_tol_scale=1e-5)
        return replace(cfg, **overrides)


@dataclass
class PbmState:
    """Dual iterate, multipliers and penalties (pbm.py:85-98), CUDA tensors."""

    u: torch.Tensor
    alpha: float
    nu_lo: torch.Tensor
    nu_up: torch.Tensor
    rho: torch.Tensor
    mu_lo: torch.Tensor
    mu_up: torch.Tensor
    p: torch.Tensor
    q_lo: torch.Tensor
    q_up: torch.Tensor

    @classmethod
    def initial(cls, n: int, m: int, volume: float) -> "PbmState":
        """Starting point of solve_pbm (pbm.py:352-363)."""
        dev = dict(dtype=torch.float64, device="cuda")
        one = lambda: torch.ones(m, **dev)  # noqa: E731
        return cls(torch.zeros(n, **dev), 1.0, one(), one(), torch.full((m,), volume / m, **dev), one(), one(),
                   one(), one(), one())


class HessianBlocks:
    """Per-element Hessian blocks (pbm.py:101-116).  `w` (m x dofs, the element
    products u_e K_e) is always available like the reference's: written by the
    evaluation when asked for (keep_w), else formed on first access from the u the
    evaluation belongs to (vts_element_products) -- the Newton step itself never
    needs it materialised (the apply recomputes K_e u_e)."""

    def __init__(self, w, a, b_lo, b_up, rho_hat, ops=None, u=None):
        self._w, self.a, self.b_lo, self.b_up, self.rho_hat = w, a, b_lo, b_up, rho_hat
        self._ops, self._u = ops, u

    @property
    def w(self) -> torch.Tensor | None:
        if self._w is None and self._ops is not None:
            self._w, _ = self._ops.element_products(self._u)
        return self._w

    def __repr__(self) -> str:
        return f"HessianBlocks(m={self.a.numel()}, w={'materialised' if self._w is not None else 'lazy'})"


@dataclass
class LagrangianEval:
    value: float
    res_u: torch.Tensor
    res_alpha: float
    res_lo: torch.Tensor
    res_up: torch.Tensor
    tau_res: float
    q: torch.Tensor
    mu_hat_lo: torch.Tensor
    mu_hat_up: torch.Tensor
    blocks: HessianBlocks
    u: torch.Tensor = field(default=None, repr=False)  # the state's u the data belongs to


def eval_lagrangian(state: PbmState, ops: ElementOps, f, bounds: DensityBounds, pen: PenaltyBarrier,
                    keep_w: bool = False) -> LagrangianEval:
    n, m = ops.n, ops.m
    u = ops.check_vec(state.u, n, "u")
    out = {k: ops.vec(m) for k in ("res_lo", "res_up", "q", "mu_hat_lo", "mu_hat_up", "a", "b_lo", "b_up",
                                  "rho_hat")}
    res_u = ops.vec(n)
    w = torch.empty((m, ops.dofs_per_elem), dtype=torch.float64, device="cuda") if keep_w else None
    sc = (ctypes.c_double * 8)()
    flags = ctypes.c_uint32(0)
    rc = _lib.load().vts_eval_lagrangian(
        ops.handle, ptr(u), float(state.alpha), ptr(state.nu_lo), ptr(state.nu_up), ptr(state.rho),
        ptr(state.mu_lo), ptr(state.mu_up), ptr(state.p), ptr(state.q_lo), ptr(state.q_up), ptr(f),
        ptr(bounds.lower), ptr(bounds.upper), float(bounds.volume), ops.norm_f, bounds.norm, pen.branch,
        ptr(res_u), ptr(out["res_lo"]), ptr(out["res_up"]), ptr(out["q"]), ptr(out["mu_hat_lo"]),
        ptr(out["mu_hat_up"]), ptr(out["a"]), ptr(out["b_lo"]), ptr(out["b_up"]), ptr(out["rho_hat"]), ptr(w),
        sc, ctypes.byref(flags))
    _lib.check(rc, "vts_eval_lagrangian")
    warn_saturated(flags.value)
    blocks = HessianBlocks(w, out["a"], out["b_lo"], out["b_up"], out["rho_hat"], ops, u)
    return LagrangianEval(sc[0], res_u, sc[1], out["res_lo"], out["res_up"], sc[2], out["q"], out["mu_hat_lo"],
                          out["mu_hat_up"], blocks, u)


def schur_system(ev: LagrangianEval, ops: ElementOps):
    """Reduced (n+1) Newton system (pbm.py:202-218): (NewtonMatrix, rhs)."""
    blk = ev.blocks
    chat = ops.vec(ops.m)
    rhs = ops.vec(ops.n + 1)
    border = ops.vec(ops.n)
    corner = ctypes.c_double(0.0)
    rc = _lib.load().vts_schur_system(ops.handle, ptr(ev.u), ptr(ev.res_u), float(ev.res_alpha), ptr(ev.res_lo),
                                      ptr(ev.res_up), ptr(blk.a), ptr(blk.b_lo), ptr(blk.b_up), ptr(blk.rho_hat),
                                      ptr(chat), ptr(rhs), ptr(border), ctypes.byref(corner))
    _lib.check(rc, "vts_schur_system")
    ops._system_version = getattr(ops, "_system_version", 0) + 1
    mat = NewtonMatrix(ops, border, corner.value, ops._system_version)
    mat.chat = chat
    return mat, rhs


def _reconstruct(ev: LagrangianEval, ops: ElementOps, du, dalpha: float, want_slope: bool):
    blk = ev.blocks
    du = ops.check_vec(du, ops.n, "du")
    dnu_lo, dnu_up = ops.vec(ops.m), ops.vec(ops.m)
    slope = ctypes.c_double(0.0)
    rc = _lib.load().vts_reconstruct_nu(ops.handle, ptr(ev.u), ptr(du), float(dalpha), ptr(ev.res_u),
                                        float(ev.res_alpha), ptr(ev.res_lo), ptr(ev.res_up), ptr(blk.a),
                                        ptr(blk.b_lo), ptr(blk.b_up), ptr(dnu_lo), ptr(dnu_up),
                                        ctypes.byref(slope) if want_slope else None)
    _lib.check(rc, "vts_reconstruct_nu")
    return dnu_lo, dnu_up, slope.value


def reconstruct_nu(ev: LagrangianEval, ops: ElementOps, du, dalpha: float):
    """Bound-multiplier increments (pbm.py:221-232)."""
    dnu_lo, dnu_up, _ = _reconstruct(ev, ops, du, dalpha, False)
    return dnu_lo, dnu_up


def _trial_value(state: PbmState, ops, f, bounds, pen, du, dalpha, dnu_lo, dnu_up, kappa: float) -> float:
    value = ctypes.c_double(0.0)
    flags = ctypes.c_uint32(0)
    rc = _lib.load().vts_al_value(ops.handle, ptr(state.u), float(state.alpha), ptr(state.nu_lo),
                                  ptr(state.nu_up), ptr(du), float(dalpha), ptr(dnu_lo), ptr(dnu_up), float(kappa),
                                  ptr(state.rho), ptr(state.p), ptr(state.mu_lo), ptr(state.mu_up),
                                  ptr(state.q_lo), ptr(state.q_up), ptr(f), ptr(bounds.lower), ptr(bounds.upper),
                                  float(bounds.volume), pen.branch, ctypes.byref(value), ctypes.byref(flags))
    _lib.check(rc, "vts_al_value")
    warn_saturated(flags.value)
    return value.value


def al_value(u, alpha, nu_lo, nu_up, state: PbmState, ops, f, bounds, pen) -> float:
    """Augmented Lagrangian at a trial point, multipliers fixed (pbm.py:135-147)."""
    trial = replace(state, u=ops.check_vec(u, ops.n, "u"), alpha=float(alpha), nu_lo=nu_lo, nu_up=nu_up)
    return _trial_value(trial, ops, f, bounds, pen, trial.u, 0.0, nu_lo, nu_up, 0.0)


def _step(x: torch.Tensor, kappa: float, dx: torch.Tensor, ops) -> torch.Tensor:
    """x + kappa dx as a new tensor (pbm.py:320-323 rebinds, never mutates)."""
    out = x.clone()
    _lib.check(_lib.load().vts_axpy(ops.handle, out.numel(), float(kappa), ptr(dx), ptr(out)), "vts_axpy")
    return out


_mg_log = logging.getLogger("paper_1904_06556_b200.multigrid")


class _StepWork:
    """Buffers of the device-resident Newton step, owned by one ElementOps: the
    working copies of u, nu_lo, nu_up, the evaluation the step updates in place,
    and the Newton system / direction.  Kept across newton_inner calls so that
    vts_newton_step replays its CUDA graphs (their launches bake the pointers)."""

    _EV = ("res_u", "res_lo", "res_up", "q", "mu_hat_lo", "mu_hat_up", "a", "b_lo", "b_up", "rho_hat")

    def __init__(self, ops):
        n, m = ops.n, ops.m
        self.u, self.nu_lo, self.nu_up = ops.vec(n), ops.vec(m), ops.vec(m)
        self.ev = {k: ops.vec(n if k == "res_u" else m) for k in self._EV}
        self.chat, self.rhs, self.border = ops.vec(m), ops.vec(n + 1), ops.vec(n)
        self.du, self.dnu_lo, self.dnu_up = ops.vec(n + 1), ops.vec(m), ops.vec(m)


def _device_step_ok(ops) -> bool:
    return getattr(ops, "dim", 2) == 2 and os.environ.get("VTS_HOST_NEWTON", "0") != "1"


def _newton_inner_device(state: PbmState, ops: ElementOps, f, bounds: DensityBounds, pen: PenaltyBarrier,
                         tol_newton: float, mtol: StagnationTolerance, cfg: PbmConfig, trace: dict | None
                         ) -> "NewtonOutcome":
    """newton_inner (pbm.py:244-338) with each step one vts_newton_step call: the
    same loop control on the host, everything between two residual checks on the
    device.  The state is rebound to new tensors on return, as the reference rebinds."""
    mtol.reset()
    ev = eval_lagrangian(state, ops, f, bounds, pen)
    W = getattr(ops, "_step_work", None)
    if W is None:
        W = ops._step_work = _StepWork(ops)
    W.u.copy_(state.u)
    W.nu_lo.copy_(state.nu_lo)
    W.nu_up.copy_(state.nu_up)
    for k in _StepWork._EV:
        W.ev[k].copy_(getattr(ev, k) if hasattr(ev, k) else getattr(ev.blocks, k))
    alpha, value, res_alpha, tau = float(state.alpha), ev.value, ev.res_alpha, ev.tau_res
    steps = 0
    counts: list[int] = []
    best_tau = float("inf")
    no_improve = 0
    lib = _lib.load()
    a = _lib.NewtonStepArgs()
    a.u, a.nu_lo, a.nu_up = ptr(W.u), ptr(W.nu_lo), ptr(W.nu_up)
    for k in ("rho", "p", "mu_lo", "mu_up", "q_lo", "q_up"):
        setattr(a, k, ptr(getattr(state, k)))
    a.f, a.lower, a.upper = ptr(f), ptr(bounds.lower), ptr(bounds.upper)
    a.volume, a.norm_f, a.norm_bounds, a.branch = float(bounds.volume), ops.norm_f, bounds.norm, pen.branch
    for k in _StepWork._EV:
        setattr(a, k, ptr(W.ev[k]))
    a.chat, a.rhs, a.border, a.du, a.dnu_lo, a.dnu_up = (ptr(t) for t in (W.chat, W.rhs, W.border, W.du, W.dnu_lo,
                                                                          W.dnu_up))
    a.minres_floor, a.minres_cap = cfg.minres_floor, cfg.minres_cap
    a.armijo_c1, a.armijo_shrink, a.armijo_max_halvings = cfg.armijo_c1, cfg.armijo_shrink, cfg.armijo_max_halvings
    a.shift_scale = 1e-12  # MgPreconditioner's default shift_scale (multigrid.py:82)
    r = _lib.NewtonStepResult()
    stalled, note = False, ""
    while tau >= tol_newton:
        if steps >= cfg.max_newton:
            stalled, note = True, "newton iteration cap reached"
            break
        a.alpha, a.value, a.res_alpha = alpha, value, res_alpha
        a.minres_tol = min(mtol.current(), 0.99)
        rc = lib.vts_newton_step(ops.handle, ctypes.byref(a), ctypes.byref(r))
        ops._system_version = getattr(ops, "_system_version", 0) + 1
        if rc in _ERRORS:
            if steps:  # the accepted steps stay, as the reference has rebound the state by then
                state.u, state.nu_lo, state.nu_up = W.u.clone(), W.nu_lo.clone(), W.nu_up.clone()
                state.alpha = alpha
            raise MinresError(_ERRORS[rc], W.du.clone())
        _lib.check(rc, "vts_newton_step")
        if r.warnings & _lib.VTS_W_SHIFTED:
            _mg_log.warning("coarse matrix is not positive definite; retrying Cholesky with a trace-scaled shift")
        warn_saturated(r.warnings)
        counts.append(r.minres_iterations)
        if r.status == 1:
            stalled, note = True, "non-descent Newton direction"
            break
        if r.status == 2:
            stalled, note = True, "line search exhausted"
            break
        if trace is not None:
            trace.setdefault("kappa", []).append(r.kappa)
            trace.setdefault("slope", []).append(r.slope)
        alpha = r.alpha
        value, res_alpha, tau = r.scalars[0], r.scalars[1], r.scalars[2]
        steps += 1
        mtol.observe(tau)
        if tau < best_tau:
            best_tau = tau
            no_improve = 0
        else:
            no_improve += 1
            if no_improve >= cfg.stall_steps:
                stalled, note = True, "no residual improvement over consecutive steps"
                break
    if steps:
        state.u, state.nu_lo, state.nu_up = W.u.clone(), W.nu_lo.clone(), W.nu_up.clone()
        state.alpha = alpha
        out = {k: W.ev[k].clone() for k in _StepWork._EV}
        blocks = HessianBlocks(None, out["a"], out["b_lo"], out["b_up"], out["rho_hat"], ops, state.u)
        ev = LagrangianEval(value, out["res_u"], res_alpha, out["res_lo"], out["res_up"], tau, out["q"],
                            out["mu_hat_lo"], out["mu_hat_up"], blocks, state.u)
    return NewtonOutcome(steps, counts, stalled, note, ev)


@dataclass
class NewtonOutcome:
    steps: int
    minres_per_step: list
    stalled: bool
    note: str
    ev: LagrangianEval


def newton_inner(state: PbmState, ops: ElementOps, f, bounds: DensityBounds, pen: PenaltyBarrier, transfers,
                 tol_newton: float, mtol: StagnationTolerance, cfg: PbmConfig, trace: dict | None = None
                 ) -> NewtonOutcome:
    """Damped Newton minimisation of the augmented Lagrangian (pbm.py:244-338)."""
    if _device_step_ok(ops):
        return _newton_inner_device(state, ops, f, bounds, pen, tol_newton, mtol, cfg, trace)
    mtol.reset()
    ev = eval_lagrangian(state, ops, f, bounds, pen)
    steps = 0
    counts: list[int] = []
    best_tau = float("inf")
    no_improve = 0
    while ev.tau_res >= tol_newton:
        if steps >= cfg.max_newton:
            return NewtonOutcome(steps, counts, True, "newton iteration cap reached", ev)
        s_mat, rhs = schur_system(ev, ops)
        chain = MgPreconditioner(s_mat, transfers)
        mr_cfg = MinresConfig(tol=min(mtol.current(), 0.99), max_iters=cfg.minres_cap, floor=cfg.minres_floor)
        sol = minres_solve(s_mat, rhs, mr_cfg, chain.apply)
        counts.append(sol.iterations)
        du = sol.x[:-1]
        dalpha = float(sol.x[-1])
        dnu_lo, dnu_up, slope = _reconstruct(ev, ops, du, dalpha, True)
        if slope >= 0.0:
            return NewtonOutcome(steps, counts, True, "non-descent Newton direction", ev)
        kappa = 1.0
        accepted = False
        for _ in range(cfg.armijo_max_halvings + 1):
            trial = _trial_value(state, ops, f, bounds, pen, du, dalpha, dnu_lo, dnu_up, kappa)
            if trial <= ev.value + cfg.armijo_c1 * kappa * slope:
                accepted = True
                break
            kappa *= cfg.armijo_shrink
        if not accepted:
            return NewtonOutcome(steps, counts, True, "line search exhausted", ev)
        if trace is not None:
            trace.setdefault("kappa", []).append(kappa)
            trace.setdefault("slope", []).append(slope)
        state.u = _step(state.u, kappa, du.contiguous(), ops)
        state.alpha = state.alpha + kappa * dalpha
        state.nu_lo = _step(state.nu_lo, kappa, dnu_lo, ops)
        state.nu_up = _step(state.nu_up, kappa, dnu_up, ops)
        steps += 1
        ev = eval_lagrangian(state, ops, f, bounds, pen)
        mtol.observe(ev.tau_res)
        if ev.tau_res < best_tau:
            best_tau = ev.tau_res
            no_improve = 0
        else:
            no_improve += 1
            if no_improve >= cfg.stall_steps:
                return NewtonOutcome(steps, counts, True, "no residual improvement over consecutive steps", ev)
    return NewtonOutcome(steps, counts, False, "", ev)


@dataclass
class SolveReport:
    """Solve summary (report.py:22-52); arrays stay on the device."""

    method: str
    problem: str
    tol: float
    converged: bool
    columns: tuple
    rows: list
    count_columns: tuple
    objective: float
    dual_objective: float | None
    gap_scaled: float
    tau_res: float
    volume: float
    rho: torch.Tensor
    wall_clock: float
    notes: str = ""
    certificate: str | None = None
    extras: dict = field(default_factory=dict)

    def totals(self) -> dict:
        return {c: int(sum(r[self.columns.index(c)] for r in self.rows)) for c in self.count_columns}

    @property
    def outer_iterations(self) -> int:
        return len(self.rows)


def _measure(ops, state, ev, f, bounds):
    """dual objective, gap (model.py:50-79), f.u and sum(rho) in one device pass."""
    d_val, gap, fu, rho_sum = (ctypes.c_double() for _ in range(4))
    rc = _lib.load().vts_gap(ops.handle, ptr(state.u), float(state.alpha), ptr(ev.q), ptr(f), ptr(state.nu_lo),
                             ptr(state.nu_up), ptr(bounds.lower), ptr(bounds.upper), float(bounds.volume),
                             ptr(state.rho), ctypes.byref(d_val), ctypes.byref(gap), ctypes.byref(fu),
                             ctypes.byref(rho_sum))
    _lib.check(rc, "vts_gap")
    return d_val.value, gap.value, fu.value, rho_sum.value


def _safeguard(ops, cfg, state, ev, multipliers: bool, penalties: bool) -> None:
    rc = _lib.load().vts_outer_update(
        ops.handle, cfg.beta, cfg.gamma, cfg.penalty_floor, ptr(ev.blocks.rho_hat),
        ptr(ev.mu_hat_lo) if multipliers else None, ptr(ev.mu_hat_up) if multipliers else None,
        ptr(state.rho), ptr(state.mu_lo), ptr(state.mu_up), ptr(state.p), ptr(state.q_lo), ptr(state.q_up),
        1 if penalties else 0)
    _lib.check(rc, "vts_outer_update")


def solve_pbm(problem, cfg: PbmConfig | None = None, trace: dict | None = None, ops: ElementOps | None = None
              ) -> SolveReport:
    """Run the multiplier method on a problem instance (pbm.py:341-465)."""
    cfg = cfg or PbmConfig()
    t0 = time.perf_counter()
    ops = ops or ElementOps(problem.fine)
    bounds = DensityBounds.for_problem(problem.m, problem.volume, cfg.rho_lower)
    f = problem.f
    m, n = problem.m, problem.n
    pen = PenaltyBarrier(cfg.branch)
    state = PbmState.initial(n, m, problem.volume)
    mtol = StagnationTolerance(tol=min(cfg.minres_tol_scale * sqrt(n), 0.5), floor=cfg.minres_floor)
    tol_newton = cfg.tol_newton0
    columns = ("outer", "newton", "minres", "gap_scaled", "tau_res", "volume")
    rows: list[tuple] = []
    minres_per_newton: list[int] = []
    notes: list[str] = []
    converged = False
    gap_scaled = float("inf")
    d_val = float("nan")
    ev = None
    fu = 0.0
    pre_gap = gap_scaled
    for outer in range(1, cfg.max_outer + 1):
        out = newton_inner(state, ops, f, bounds, pen, problem.transfers, tol_newton, mtol, cfg, trace)
        minres_per_newton.extend(out.minres_per_step)
        ev = out.ev
        d_val, delta, fu, rho_sum = _measure(ops, state, ev, f, bounds)
        gap_scaled = delta / max(abs(d_val), 1e-300)
        rows.append((outer, out.steps, sum(out.minres_per_step), gap_scaled, ev.tau_res, rho_sum))
        if out.stalled:
            notes.append(f"inner stall at outer {outer}: {out.note}")
        if abs(gap_scaled) < cfg.tol:
            converged = True
            break
        _safeguard(ops, cfg, state, ev, multipliers=True, penalties=True)
        tol_newton = max(min(100.0 * abs(gap_scaled), tol_newton), cfg.tol_newton_min)
    else:
        notes.append("outer iteration cap reached without meeting the gap tolerance")

    if converged:
        pre_gap = gap_scaled
        out = newton_inner(state, ops, f, bounds, pen, problem.transfers, 10.0 * cfg.tol, mtol, cfg, trace)
        minres_per_newton.extend(out.minres_per_step)
        ev = out.ev
        _safeguard(ops, cfg, state, ev, multipliers=False, penalties=False)
        d_val, delta, fu, rho_sum = _measure(ops, state, ev, f, bounds)
        gap_scaled = delta / max(abs(d_val), 1e-300)
        rows.append((len(rows) + 1, out.steps, sum(out.minres_per_step), gap_scaled, ev.tau_res, rho_sum))
        notes.append(f"final pass: scaled gap {pre_gap:.3e} -> {gap_scaled:.3e}")
        if out.stalled:
            notes.append(f"final-pass stall accepted near optimum: {out.note}")

    volume = rows[-1][5] if rows else float("nan")
    if not converged and ev is not None:
        # the cap path ends with a safeguarded update after the last row: the
        # report's volume is sum(rho) after it, like the reference (pbm.py:451)
        volume = _measure(ops, state, ev, f, bounds)[3]
    torch.cuda.current_stream().synchronize()
    certificate = None
    if converged:
        certificate = f"|duality gap|/|dual objective| = {abs(pre_gap):.6e} < tol = {cfg.tol:.1e}"
    return SolveReport(
        method="pbm", problem=problem.name, tol=cfg.tol, converged=converged, columns=columns, rows=rows,
        count_columns=("newton", "minres"), objective=0.5 * fu, dual_objective=d_val, gap_scaled=gap_scaled,
        tau_res=ev.tau_res if ev is not None else float("inf"), volume=volume,
        rho=state.rho.clone(), wall_clock=time.perf_counter() - t0, notes="; ".join(notes),
        certificate=certificate,
        extras={"u": state.u, "alpha": state.alpha, "nu_lo": state.nu_lo, "nu_up": state.nu_up,
                "mu_lo": state.mu_lo, "mu_up": state.mu_up, "p": state.p, "q_lo": state.q_lo, "q_up": state.q_up,
                "minres_per_newton": minres_per_newton, "minres_tol_final": mtol.current(),
                "kernel_launches": ops.kernel_launches},
    )
