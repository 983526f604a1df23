/*
 * vts_b200.h — C ABI of the B200-native PBM inner Newton step.
 *
 * The reference (`vtsopt`, /root/reference/pkg/src/vtsopt) is pure Python and
 * has no FFI; the path sits behind Python call signatures.
 * Each entry point below replaces one of those call sites; the file:line of
 * the reference interface it stands in for is given with it.  A ctypes
 * binding (the reference-side stub a maintainer would add) is shown in
 * INTEGRATION.md; the package `paper_1904_06556_b200` is that binding.
 *
 * Conventions
 *  - Every pointer argument is a raw CUDA device pointer to contiguous fp64
 *    (or int) data owned by the caller, unless documented as host memory.
 *    The library borrows it for the duration of the call only.
 *  - "free" vectors use the reference's free-dof numbering (node-major,
 *    x then y, Dirichlet dofs skipped; mesh.py:266-267): length n, or n+1
 *    when bordered (volume-multiplier unknown last).  Element arrays have
 *    length m in the reference's element order (mesh.py:253-259).
 *  - `stream` is a cudaStream_t passed as an integer (0 = legacy default).
 *    All work is stream-ordered; calls that return host scalars synchronise
 *    that stream.
 *  - Return codes: VTS_OK or one of the VTS_E* codes; vts_last_error()
 *    returns a message for the calling thread's last failure.
 *  - A context is not thread safe; one context per problem instance.
 */
#ifndef VTS_B200_H
#define VTS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VTS_OK 0
#define VTS_E_INDEFINITE 1   /* MinresError("preconditioner is indefinite ...") linalg.py:168,205 */
#define VTS_E_BREAKDOWN 2    /* MinresError("MINRES recurrence broke down") linalg.py:216 */
#define VTS_E_NONFINITE 3    /* MinresError("NaN/inf encountered ...") linalg.py:227 */
#define VTS_E_ARGUMENT 4     /* ValueError */
#define VTS_E_CUDA 5         /* CUDA runtime failure */
#define VTS_E_CHOLESKY 6     /* coarse Cholesky failed even after the shift (multigrid.py:102) */

/* warning bits returned through `warn_flags` */
#define VTS_W_SATURATED 1u   /* penalty input saturated (penalty.py:85-95 RuntimeWarning) */
#define VTS_W_SHIFTED 2u     /* coarse Cholesky needed the shift (multigrid.py:95-103 log.warning) */

typedef struct vts_ctx vts_ctx;

const char* vts_last_error(void);
int vts_version(void);

/*
 * Context over one mesh hierarchy.  Replaces the data the reference builds in
 * `build_problem` / `MeshLevel` (mesh.py:216-287) and `ElementOps.__init__`
 * (fem.py:150-162): `ex[k]`, `ey[k]` are the element counts of level k
 * (coarsest first, each level doubling the previous one), `dof_maps[k]` is a
 * HOST int64 array (n_nodes_k x 2) holding the free-dof index of each node
 * component or -1 for a Dirichlet dof (MeshLevel.dof), `ke` a HOST row-major
 * 8x8 element stiffness (fem.hex_stiffness analogue).
 */
int vts_ctx_create(vts_ctx** out, int32_t levels, const int32_t* ex, const int32_t* ey,
                   const int64_t* const* dof_maps, const double* ke, int64_t stream);
/*
 * Context over one HEXAHEDRAL hierarchy -- the reference's own 3D
 * discretisation (mesh.py:216-287: trilinear 8-node cubes, three dofs per
 * node, whole nodes fixed; fem.py:150-162).  `ez[k]` adds the third axis,
 * `dof_maps[k]` is a HOST int64 array (n_nodes_k x 3), `ke` a HOST row-major
 * 24x24 element stiffness of the finest level (fem.hex_stiffness with the
 * finest edge).  Every other entry point below works on either kind of
 * context with the same conventions (element products w are m x 24 here);
 * the benchmark probes and the interior-point blocks are 2D only.
 */
int vts_ctx_create3(vts_ctx** out, int32_t levels, const int32_t* ex, const int32_t* ey, const int32_t* ez,
                    const int64_t* const* dof_maps, const double* ke, int64_t stream);
/* 2 or 3: the context's discretisation */
int vts_ctx_dim(const vts_ctx* ctx);
int vts_ctx_destroy(vts_ctx* ctx);
/* n (free dofs of the finest level) and m (elements); HOST outputs */
int vts_ctx_sizes(const vts_ctx* ctx, int64_t* n, int64_t* m);

/*
 * Augmented Lagrangian value, gradient blocks and curvatures:
 * `eval_lagrangian` (pbm.py:150-199).  State arrays (length m) and u, f
 * (length n) are inputs; every output array is written in full.  `w_out`
 * (m x 8, element-local K_e u_e) may be NULL.  `scalars` (HOST, 8 doubles) =
 * {value, res_alpha, tau_res, f.u, sum rho_hat, ||res_u||, ||res_lo||, 0}.
 */
int vts_eval_lagrangian(vts_ctx* ctx, const double* u, double alpha, const double* nu_lo,
                        const double* nu_up, const double* rho, const double* mu_lo,
                        const double* mu_up, const double* p, const double* q_lo,
                        const double* q_up, const double* f, const double* lower,
                        const double* upper, double volume, double norm_f, double norm_bounds,
                        double branch, double* res_u, double* res_lo, double* res_up, double* q,
                        double* mu_hat_lo, double* mu_hat_up, double* a, double* b_lo,
                        double* b_up, double* rho_hat, double* w_out, double* scalars,
                        uint32_t* warn_flags);

/*
 * Reduced (n+1) Newton system: `schur_system` (pbm.py:202-218) with the
 * assembly `ElementOps.assemble(..., border_sign=-1)` (fem.py:188-209)
 * replaced by a matrix-free operator bound into the context.  Inputs are the
 * eval outputs; writes chat (m), rhs (n+1, free, bordered) and border (n,
 * may be NULL); `corner` (HOST) = sum chat.  After this call the context
 * holds the Newton matrix used by vts_newton_apply / vts_mg_setup /
 * vts_minres.
 */
int vts_schur_system(vts_ctx* ctx, const double* u, const double* res_u, double res_alpha,
                     const double* res_lo, const double* res_up, const double* a,
                     const double* b_lo, const double* b_up, const double* rho_hat, double* chat,
                     double* rhs, double* border, double* corner);

/* y = S x for the bound Newton matrix: BorderedMatrix.matvec (linalg.py:56-62). */
int vts_newton_apply(vts_ctx* ctx, const double* x, double* y);

/*
 * Galerkin hierarchy + coarsest Cholesky of the bound Newton matrix:
 * MgPreconditioner.__init__ (multigrid.py:82-103).  HOST `shifted` = 1 when
 * the coarse factorisation needed the trace-scaled shift.
 */
int vts_mg_setup(vts_ctx* ctx, double shift_scale, int32_t* shifted);

/* One V(2,2) cycle from a zero guess: MgPreconditioner.apply (multigrid.py:109-143). */
int vts_vcycle(vts_ctx* ctx, const double* b, double* z);

/*
 * Level operator probe for parity tests: y = A_k x on level k (0 = coarsest),
 * bordered free vectors of that level (MgPreconditioner.mats[k].matvec).
 */
int vts_level_apply(vts_ctx* ctx, int32_t level, const double* x, double* y);
/* free-dof count of level k (HOST output) */
int vts_level_size(const vts_ctx* ctx, int32_t level, int64_t* n);

/*
 * Preconditioned MINRES on the bound Newton matrix with the V-cycle
 * preconditioner: minres_solve(S, b, MinresConfig(tol, max_iters, floor),
 * mg.apply) (linalg.py:128-242), zero initial guess.  `x` (n+1) receives the
 * iterate (the last sound one on error).  HOST outputs: iterations, relres,
 * converged.  `history` (HOST, may be NULL, length >= max_iters) receives the
 * true relative residual after every iteration (costs one extra apply each).
 */
int vts_minres(vts_ctx* ctx, const double* b, double* x, double tol, int32_t max_iters,
               double floor_tol, int32_t precondition, int32_t* iterations, double* relres,
               int32_t* converged, double* history);

/*
 * Diagnostic probe (no reference counterpart): one smoothing step of level
 * `level` as the V-cycle runs it -- two lexicographic Gauss-Seidel sweeps
 * (forward or backward, multigrid.py:35-64 via _smooth :145-154) on
 * A_k x = b - border x_alpha, x_alpha = x[last]; `zero_first` takes the
 * first forward sweep from x = 0 (the pre-smoothing start).  b, x: level-k
 * bordered free vectors (x in/out).
 */
int vts_debug_smooth(vts_ctx* ctx, int32_t level, int32_t forward, int32_t zero_first, const double* b, double* x);

/*
 * vts_minres with a warm start: `x0` (device, n+1 entries, or n for a bound
 * stiffness, may be NULL) is the initial iterate of minres_solve(..., x0=...)
 * (linalg.py:144-154): r = b - A x0, and when ||r||/||b|| <= floor_tol x0 is
 * returned with 0 iterations.  On errors x holds the last sound iterate (x0
 * when none was taken).
 */
int vts_minres_warm(vts_ctx* ctx, const double* b, double* x, const double* x0, double tol, int32_t max_iters,
                    double floor_tol, int32_t precondition, int32_t* iterations, double* relres,
                    int32_t* converged, double* history);

/*
 * minres_solve for an arbitrary operator (linalg.py:118-242 with `a` a CSR
 * matrix, ndarray or callable and `precond` any callable, _as_matvec
 * linalg.py:118-125).  `op(user, in, out)` and `precond(user, in, out)` apply
 * the operator / preconditioner to device vectors of `len` entries and return
 * 0 (nonzero aborts with that code); `precond` may be NULL.  The callbacks are
 * called with the context stream drained and must leave `out` complete.  The
 * Lanczos / Givens recurrences are the device kernels of vts_minres.
 */
typedef int (*vts_apply_fn)(void* user, const double* in, double* out);
int vts_minres_generic(vts_ctx* ctx, int64_t len, const double* b, double* x, const double* x0, double tol,
                       int32_t max_iters, double floor_tol, vts_apply_fn op, vts_apply_fn precond, void* user,
                       int32_t* iterations, double* relres, int32_t* converged, double* history);

/*
 * Bound-multiplier back-substitution + directional derivative:
 * reconstruct_nu (pbm.py:221-232) and the slope (pbm.py:290-295).
 * HOST `slope` (may be NULL).
 */
int vts_reconstruct_nu(vts_ctx* ctx, const double* u, const double* du, double dalpha,
                       const double* res_u, double res_alpha, const double* res_lo,
                       const double* res_up, const double* a, const double* b_lo,
                       const double* b_up, double* dnu_lo, double* dnu_up, double* slope);

/*
 * Augmented Lagrangian at the trial point x + kappa dx with multipliers
 * fixed: _al_value (pbm.py:135-147) fused with the axpys of pbm.py:300-305.
 * HOST output `value`.
 */
int vts_al_value(vts_ctx* ctx, const double* u, double alpha, const double* nu_lo,
                 const double* nu_up, const double* du, double dalpha, const double* dnu_lo,
                 const double* dnu_up, double kappa, const double* rho, const double* p,
                 const double* mu_lo, const double* mu_up, const double* q_lo,
                 const double* q_up, const double* f, const double* lower, const double* upper,
                 double volume, double branch, double* value, uint32_t* warn_flags);

/* x += kappa dx for the accepted Newton step (pbm.py:320-323), n and m parts. */
int vts_axpy(vts_ctx* ctx, int64_t len, double kappa, const double* dx, double* x);

/*
 * Safeguarded multiplier / penalty update of the outer loop (pbm.py:397-402):
 * rho <- clip(rho_hat, beta rho, rho/beta) (same for mu_lo, mu_up),
 * p, q_lo, q_up <- max(gamma x, floor).  Pass rho_hat = NULL to skip the
 * multiplier part, update_penalties = 0 to skip the penalty part.
 */
int vts_outer_update(vts_ctx* ctx, double beta, double gamma, double floor_p, const double* rho_hat,
                     const double* mu_hat_lo, const double* mu_hat_up, double* rho, double* mu_lo,
                     double* mu_up, double* p, double* q_lo, double* q_up, int32_t update_penalties);

/*
 * Dual objective and scaled duality gap at (u, alpha): dual_objective and
 * duality_gap (model.py:50-79).  HOST outputs: d_val, gap (unscaled), f.u,
 * sum(rho).
 */
int vts_gap(vts_ctx* ctx, const double* u, double alpha, const double* q, const double* f,
            const double* nu_lo, const double* nu_up, const double* lower, const double* upper,
            double volume, const double* rho, double* d_val, double* gap, double* fu,
            double* rho_sum);

/*
 * phi, phi', phi'' of a device vector tau (length n): PenaltyBarrier.value /
 * deriv / deriv2 (penalty.py:49-82) with the saturation rule of
 * penalty.py:85-95 (VTS_W_SATURATED).  Output pointers may be NULL.
 */
int vts_penalty_eval(vts_ctx* ctx, int64_t n, const double* tau, double branch, double* value, double* d1,
                     double* d2, uint32_t* warn_flags);

/*
 * Interior-point Newton step (ip.py:114-222) on the same operators.  All
 * arrays are DEVICE pointers (u, du, res_u: n free dofs; element arrays: m).
 *
 * vts_ip_residual: `kkt_residual` (ip.py:114-134): writes q, res_c, res_lo,
 * res_up (m) and res_u = K(rho) u - f (n); HOST `scalars` (9) = {res_alpha,
 * tau_res, f.u, sum rho, nu_lo.(rho-lower), nu_up.(upper-rho), comp_max
 * (ip.py:285-288), min_slack (ip.py:311-313), min(nu_lo, nu_up)}.
 */
int vts_ip_residual(vts_ctx* ctx, const double* u, double alpha, const double* rho, const double* nu_lo,
                    const double* nu_up, double r, double s, const double* lower, const double* upper, double volume,
                    const double* f, double norm_f, double* q, double* res_c, double* res_lo, double* res_up,
                    double* res_u, double* scalars);

/*
 * vts_ip_schur_system: `schur_system` (ip.py:137-158) bound into the context.
 * The reference's S+ has border +sum (1/D) w (`assemble(..., border_sign=+1)`,
 * fem.py:188-209); with E = diag(I, -1) the context holds S- = E S+ E (the
 * PBM operator's sign) and flips the border entry of every bordered vector at
 * the API edge, so vts_newton_apply / vts_vcycle / vts_minres act as S+ and
 * its preconditioner on vectors in the reference's convention.  Writes D
 * (`dcoef`), g (m) and `rhs` (n+1, ip.py:155-157); HOST `corner` = sum 1/D.
 */
int vts_ip_schur_system(vts_ctx* ctx, const double* u, const double* rho, const double* nu_lo, const double* nu_up,
                        const double* lower, const double* upper, const double* res_c, const double* res_lo,
                        const double* res_up, const double* res_u, double res_alpha, double* dcoef, double* g,
                        double* rhs, double* corner);

/* vts_ip_reconstruct: `reconstruct` (ip.py:161-186); dalpha in the reference's sign. */
int vts_ip_reconstruct(vts_ctx* ctx, const double* u, const double* du, double dalpha, const double* dcoef,
                       const double* g, const double* res_c, const double* res_lo, const double* res_up,
                       const double* rho, const double* nu_lo, const double* nu_up, const double* lower,
                       const double* upper, double* drho, double* dnu_up, double* dnu_lo);

/*
 * vts_ip_step_bounds: the minima behind `step_lengths` (ip.py:189-222), HOST
 * `mins` (4) = {min (upper-rho)/drho over drho > 0, min (lower-rho)/drho over
 * drho < 0, min -nu_lo/dnu_lo over dnu_lo < 0, min -nu_up/dnu_up over
 * dnu_up < 0}, +inf for an empty set.
 */
int vts_ip_step_bounds(vts_ctx* ctx, const double* rho, const double* drho, const double* nu_lo,
                       const double* dnu_lo, const double* nu_up, const double* dnu_up, const double* lower,
                       const double* upper, double* mins);

/*
 * DOC reuse (doc.py:111-208).
 *
 * vts_bind_stiffness: bind K(rho) = sum_e rho_e K_e (fem.py:211-219,
 * `ElementOps.assemble_stiffness`) as the context's system.  vts_newton_apply,
 * vts_mg_setup / vts_vcycle / vts_level_apply (multigrid.py:82-154 on an
 * unbordered matrix) and vts_minres_warm then act on it with n-entry vectors.
 * HOST `warn_flags` bit 1: some rho < 0 (the reference's RuntimeWarning).
 */
int vts_bind_stiffness(vts_ctx* ctx, const double* rho, uint32_t* warn_flags);
/*
 * ElementOps.element_products (fem.py:175-180) for a free-dof u: w (m x 8,
 * element-local u_e K_e; may be NULL) and q_e = u_e . w_e / 2 (m).
 */
int vts_element_products(vts_ctx* ctx, const double* u, double* w, double* q);
/*
 * doc_update (doc.py:63-75): rho_new = clip(rho * z^exponent / alpha, lower,
 * upper) with z = z_scale * z_in (z_scale 1 for the reference's z, 2 when
 * `z` holds the energies q and z = 2 q, doc.py:149; both exact).
 */
int vts_doc_update(vts_ctx* ctx, const double* rho, const double* z, double z_scale, double alpha, double exponent,
                   const double* lower, const double* upper, double* rho_new);
/*
 * bisect_volume (doc.py:78-108) over that update: one cooperative launch for
 * the whole bisection; `rho_new` = the update at the last multiplier tried,
 * HOST `alpha` its value, HOST `status` 0 ok, 1 the bracket is invalid
 * (ValueError, doc.py:92-97), 2 not closed in `cap` steps (doc.py:107-108).
 */
int vts_doc_bisect(vts_ctx* ctx, const double* rho, const double* z, double z_scale, const double* lower,
                   const double* upper, double volume, double exponent, double alpha_hi, double tol, int32_t cap,
                   double* rho_new, double* alpha, int32_t* status);
/*
 * The per-iteration measures of solve_doc (doc.py:148-155): HOST out[5] =
 * {max |rho_new - rho|, f.u, best_alpha_gap's gap, its alpha (model.py:69-98),
 * sum(rho_new)}.
 */
int vts_doc_measure(vts_ctx* ctx, const double* rho_new, const double* rho, const double* q, const double* u,
                    const double* f, const double* lower, const double* upper, double volume, double* out);

/*
 * Benchmark helper (no reference counterpart): average device time in ms of
 * {Newton apply, one V-cycle, finest forward GS sweep, second-finest forward
 * GS sweep, finest residual, mg_setup} over `reps` back-to-back launches,
 * CUDA events on the context stream; HOST `ms` (6 doubles).  Needs a bound
 * Newton matrix and a set-up multigrid; overwrites context scratch vectors.
 */
int vts_time_kernels(vts_ctx* ctx, int32_t reps, double* ms);

/*
 * Benchmark helper (no reference counterpart): cold-L2 device time in ms of
 * {Newton apply, finest residual}, averaged over `reps` launches; before each
 * launch the DEVICE buffer `flush` (flush_bytes, larger than the 126 MB L2) is
 * overwritten on the context stream, and each launch has its own event pair.
 * HOST `ms` (2 doubles).  Same preconditions as vts_time_kernels.
 */
int vts_time_cold(vts_ctx* ctx, int32_t reps, void* flush, int64_t flush_bytes, double* ms);

/*
 * One damped Newton step of newton_inner (pbm.py:273-325) resident on the
 * device: schur_system (pbm.py:202-218), MgPreconditioner (multigrid.py:82-103,
 * the shifted retry of the coarse factor decided on the device), minres_solve
 * (linalg.py:128-242: its start-up checks on the device, the iteration loop
 * polled without stalling the stream), the direction's bound-multiplier part
 * and slope (pbm.py:221-232, 290-295), the Armijo search (pbm.py:296-318: the
 * trial steps, the sufficient-decrease test and the halving on the device), the
 * update of u, alpha, nu (pbm.py:320-323, in place) and eval_lagrangian at the
 * new point (pbm.py:324) -- with one host synchronisation after the MINRES loop
 * in the common case (a second when the search needs more than two trials).
 * The Newton-system setup and the search/update/evaluation phase are replayed
 * as CUDA graphs when the buffers are the ones of the previous step.
 * Every pointer is a DEVICE pointer; `args` and `result` are HOST structs.
 * Returns VTS_OK (result->status: 0 step taken, 1 non-descent direction,
 * 2 line search exhausted -- newton_inner's stall outcomes; the state and the
 * evaluation are then unchanged), a MINRES error code (the solve's last sound
 * iterate is in `du`), or VTS_E_CHOLESKY.
 */
typedef struct {
  /* state: u (n), nu_lo, nu_up (m) updated in place; alpha in/out through result */
  double* u;
  double* nu_lo;
  double* nu_up;
  double alpha;
  const double *rho, *p, *mu_lo, *mu_up, *q_lo, *q_up;
  /* problem data (f free order, bounds per element) */
  const double *f, *lower, *upper;
  double volume, norm_f, norm_bounds, branch;
  /* evaluation at the current point (eval_lagrangian's outputs), overwritten with the one at the new point */
  double *res_u, *res_lo, *res_up, *q, *mu_hat_lo, *mu_hat_up, *a, *b_lo, *b_up, *rho_hat;
  double value, res_alpha;
  /* workspace owned by the caller: chat (m), rhs (n+1), border (n), du (n+1), dnu_lo, dnu_up (m) */
  double *chat, *rhs, *border, *du, *dnu_lo, *dnu_up;
  /* controls (PbmConfig / MinresConfig) */
  double minres_tol, minres_floor;
  int32_t minres_cap;
  double armijo_c1, armijo_shrink;
  int32_t armijo_max_halvings;
  double shift_scale;
} vts_newton_step_args;

typedef struct {
  int32_t status;          /* 0 step taken; 1 non-descent direction; 2 line search exhausted */
  int32_t minres_iterations, minres_converged;
  double minres_relres;
  double kappa, slope, dalpha;
  double alpha;            /* alpha after the step */
  double scalars[8];       /* eval_lagrangian's scalars at the new point (value, res_alpha, tau_res, ...) */
  uint32_t warnings;       /* VTS_W_SATURATED / VTS_W_SHIFTED raised during the step */
  int32_t trials;          /* Armijo trial values evaluated */
  int32_t host_syncs;      /* host synchronisations the step made (MINRES status polls excluded) */
  int32_t graphs;          /* CUDA graph launches of the step */
} vts_newton_step_result;

int vts_newton_step(vts_ctx* ctx, const vts_newton_step_args* args, vts_newton_step_result* result);

/* Number of kernels this context launched since creation (evidence counter). */
int64_t vts_kernel_launches(const vts_ctx* ctx);

/*
 * Profiling helper (no reference counterpart): between vts_profile_begin and
 * vts_profile_end every launch of a wavefront Gauss-Seidel kernel (a single
 * sweep, or a pipelined pair of sweeps) is bracketed by a CUDA event pair on
 * the context stream.  vts_profile_end synchronises the stream and writes
 * HOST out[8] = {total ms of those launches, number of launches, then ms and
 * count of the finest-level single-sweep launches, descent pairs (zero guess
 * + forward) and ascent pairs (backward + backward)}.  Used by bench.py for the dominant kernel's share of a
 * MINRES iteration; costs two event records per launch while enabled.
 */
int vts_profile_begin(vts_ctx* ctx);
int vts_profile_end(vts_ctx* ctx, double* out);

#ifdef __cplusplus
}
#endif

#endif /* VTS_B200_H */
