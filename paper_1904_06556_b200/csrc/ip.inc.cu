// Interior-point Newton step on the same operators (unity-built into vts_b200.cu).
//
// ip.py's step (ip.py:114-222): the perturbed KKT residual, the doubly
// condensed (n+1) system S+ = [[K(rho) + sum (1/D) w w^T, +sum (1/D) w],
// [., sum 1/D]] with its right-hand side, the back-substitution of
// (d rho, d nu_up, d nu_lo) and the fraction-to-boundary bounds.  S+ differs
// from the PBM Newton matrix only by the sign of its border, so with
// E = diag(I, -1) the context binds S- = E S+ E (element weights rho, rank-one
// weights 1/D) and the matrix-free apply, the Galerkin hierarchy, the V-cycle
// and MINRES run unchanged; vectors cross the API in the reference's
// convention and their border entry flips at the free/grid conversion
// (exact: negations), so MINRES sees E b and returns E x.

namespace vts {

// kkt_residual element pass (ip.py:114-134): q, res_c, res_lo, res_up and the
// element sums of tau_res, the barrier staging dots (ip.py:275-276) and, as
// exact min / max, comp_max (ip.py:285-288) and min_slack (ip.py:311-313)
__global__ void __launch_bounds__(kThreads) k_ip_elem(int m, int ex, int nx, const double* __restrict__ ug,
                                                    double alpha, const double* __restrict__ rho,
                                                    const double* __restrict__ nu_lo,
                                                    const double* __restrict__ nu_up,
                                                    const double* __restrict__ lower,
                                                    const double* __restrict__ upper, double r, double s,
                                                    double* q_out, double* res_c, double* res_lo, double* res_up,
                                                    double* partials, double* mm_partials) {
  __shared__ double scratch[8 * kThreads / 32];
  __shared__ double mm[4][kThreads / 32];
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  double comp_max = 0.0, slack_lo = INFINITY, slack_up = INFINITY, nu_min = INFINITY;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    int nd[4];
    elem_nodes(e, ex, nx, nd);
    double ue[8], w[8];
    gather8(ug, nd, ue);
    ke_times(ue, w);
    double qq = w[0] * ue[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) qq = fma(w[i], ue[i], qq);
    qq = 0.5 * qq;
    const double rh = rho[e], nlo = nu_lo[e], nup = nu_up[e], lo = lower[e], up = upper[e];
    const double plo = __dsub_rn(rh, lo), pup = __dsub_rn(up, rh);
    const double clo = __dmul_rn(plo, nlo), cup = __dmul_rn(pup, nup);
    const double rc = __dsub_rn(__dadd_rn(__dadd_rn(qq, alpha), nlo), nup);
    const double rl = __dsub_rn(clo, r), ru = __dsub_rn(cup, s);
    q_out[e] = qq;
    res_c[e] = rc;
    res_lo[e] = rl;
    res_up[e] = ru;
    acc[0] += rh;
    acc[1] = fma(rc, rc, acc[1]);
    acc[2] = fma(nlo, nlo, acc[2]);
    acc[3] = fma(nup, nup, acc[3]);
    acc[4] += rl;
    acc[5] += ru;
    acc[6] = fma(nlo, plo, acc[6]);
    acc[7] = fma(nup, pup, acc[7]);
    comp_max = fmax(comp_max, fmax(fabs(clo), fabs(cup)));
    slack_lo = fmin(slack_lo, plo);
    slack_up = fmin(slack_up, pup);
    nu_min = fmin(nu_min, fmin(nlo, nup));
  }
  block_partials<8>(acc, scratch, partials);
  // exact reductions (order-free): max over the warp, then over the block
  for (int o = 16; o > 0; o >>= 1) {
    comp_max = fmax(comp_max, __shfl_xor_sync(0xffffffffu, comp_max, o));
    slack_lo = fmin(slack_lo, __shfl_xor_sync(0xffffffffu, slack_lo, o));
    slack_up = fmin(slack_up, __shfl_xor_sync(0xffffffffu, slack_up, o));
    nu_min = fmin(nu_min, __shfl_xor_sync(0xffffffffu, nu_min, o));
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    mm[0][warp] = comp_max;
    mm[1][warp] = slack_lo;
    mm[2][warp] = slack_up;
    mm[3][warp] = nu_min;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      comp_max = fmax(comp_max, mm[0][k]);
      slack_lo = fmin(slack_lo, mm[1][k]);
      slack_up = fmin(slack_up, mm[2][k]);
      nu_min = fmin(nu_min, mm[3][k]);
    }
    mm_partials[4 * blockIdx.x] = comp_max;
    mm_partials[4 * blockIdx.x + 1] = slack_lo;
    mm_partials[4 * blockIdx.x + 2] = slack_up;
    mm_partials[4 * blockIdx.x + 3] = nu_min;
  }
}

// scalars of kkt_residual: out = {res_alpha, tau_res, f.u, sum rho, nu_lo.(rho - lower),
// nu_up.(upper - rho), comp_max, min_slack, min(nu_lo, nu_up)}
__global__ void k_ip_finish(int nb_e, const double* __restrict__ pe, const double* __restrict__ pm, int nb_n,
                            const double* __restrict__ pn, int m, double volume, double norm_f, double* out) {
  __shared__ double scratch[10 * kThreads / 32];
  __shared__ double mm[4][kThreads / 32];
  double t[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  double cmax = 0.0, slo = INFINITY, sup = INFINITY, nmin = INFINITY;
  for (int b = threadIdx.x; b < nb_e; b += blockDim.x) {
    for (int i = 0; i < 8; ++i) t[i] += pe[b * 8 + i];
    cmax = fmax(cmax, pm[4 * b]);
    slo = fmin(slo, pm[4 * b + 1]);
    sup = fmin(sup, pm[4 * b + 2]);
    nmin = fmin(nmin, pm[4 * b + 3]);
  }
  for (int b = threadIdx.x; b < nb_n; b += blockDim.x)
    for (int i = 0; i < 2; ++i) t[8 + i] += pn[b * 2 + i];
  block_sum<10>(t, scratch);
  for (int o = 16; o > 0; o >>= 1) {
    cmax = fmax(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
    slo = fmin(slo, __shfl_xor_sync(0xffffffffu, slo, o));
    sup = fmin(sup, __shfl_xor_sync(0xffffffffu, sup, o));
    nmin = fmin(nmin, __shfl_xor_sync(0xffffffffu, nmin, o));
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    mm[0][warp] = cmax;
    mm[1][warp] = slo;
    mm[2][warp] = sup;
    mm[3][warp] = nmin;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      cmax = fmax(cmax, mm[0][k]);
      slo = fmin(slo, mm[1][k]);
      sup = fmin(sup, mm[2][k]);
      nmin = fmin(nmin, mm[3][k]);
    }
    const double res_alpha = t[0] - volume;  // ip.py:125
    // ip.py:130-136, the reference's left-to-right order
    const double tau = (((sqrt(t[8]) / norm_f + fabs(res_alpha) / volume) + sqrt(t[1]) / (sqrt(t[2]) + sqrt(t[3]))) +
                        fabs(t[4]) / m) +
                       fabs(t[5]) / m;
    out[0] = res_alpha;
    out[1] = tau;
    out[2] = t[9];
    out[3] = t[0];
    out[4] = t[6];
    out[5] = t[7];
    out[6] = cmax;
    out[7] = fmin(slo, sup);
    out[8] = nmin;
  }
}

// schur_system coefficients (ip.py:148-158): D, g, the bound weights (rho, 1/D)
// and t = -g/D, so k_schur_node / k_schur_finish form E rhs
__global__ void __launch_bounds__(kThreads) k_ip_schur_elem(int m, const double* __restrict__ rho,
                                                          const double* __restrict__ nu_lo,
                                                          const double* __restrict__ nu_up,
                                                          const double* __restrict__ lower,
                                                          const double* __restrict__ upper,
                                                          const double* __restrict__ res_c,
                                                          const double* __restrict__ res_lo,
                                                          const double* __restrict__ res_up, double* dcoef_out,
                                                          double* g_out, double* chat_ctx, double* rho_hat_ctx,
                                                          double* t_out, double* partials) {
  __shared__ double scratch[2 * kThreads / 32];
  double acc[2] = {0, 0};
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    const double rh = rho[e];
    const double plo = __dsub_rn(rh, lower[e]), pup = __dsub_rn(upper[e], rh);
    const double dc = __dadd_rn(nu_lo[e] / plo, nu_up[e] / pup);
    const double g = __dadd_rn(__dsub_rn(res_c[e], res_lo[e] / plo), res_up[e] / pup);
    const double ch = 1.0 / dc;
    const double tt = -(g / dc);
    dcoef_out[e] = dc;
    g_out[e] = g;
    chat_ctx[e] = ch;
    rho_hat_ctx[e] = rh;
    t_out[e] = tt;
    acc[0] += tt;
    acc[1] += ch;
  }
  block_partials<2>(acc, scratch, partials);
}

// reconstruct (ip.py:171-186): btdu = w.du_e, then d rho, d nu_up, d nu_lo
__global__ void __launch_bounds__(kThreads) k_ip_recon_elem(int m, int ex, int nx, const double* __restrict__ ug,
                                                          const double* __restrict__ dug, double dalpha,
                                                          const double* __restrict__ dcoef,
                                                          const double* __restrict__ g,
                                                          const double* __restrict__ res_c,
                                                          const double* __restrict__ res_lo,
                                                          const double* __restrict__ res_up,
                                                          const double* __restrict__ rho,
                                                          const double* __restrict__ nu_lo,
                                                          const double* __restrict__ nu_up,
                                                          const double* __restrict__ lower,
                                                          const double* __restrict__ upper, double* drho_out,
                                                          double* dnu_up_out, double* dnu_lo_out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    int nd[4];
    elem_nodes(e, ex, nx, nd);
    double ue[8], w[8], de[8];
    gather8(ug, nd, ue);
    gather8(dug, nd, de);
    ke_times(ue, w);
    double bt = w[0] * de[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) bt = fma(w[i], de[i], bt);
    const double lo = lower[e], up = upper[e];
    const double plo = __dsub_rn(rho[e], lo);
    const double bta = __dadd_rn(bt, dalpha);
    const double drho = __dadd_rn(bta, g[e]) / dcoef[e];
    const double rc = res_c[e];
    const double num = __dsub_rn(__dsub_rn(__dmul_rn(plo, bta), __dmul_rn(__dsub_rn(nu_lo[e], nu_up[e]), drho)),
                                 __dsub_rn(__dadd_rn(res_lo[e], res_up[e]), __dmul_rn(plo, rc)));
    const double dnup = num / __dsub_rn(up, lo);
    const double dnlo = __dsub_rn(__dsub_rn(__dsub_rn(dnup, bt), dalpha), rc);
    drho_out[e] = drho;
    dnu_up_out[e] = dnup;
    dnu_lo_out[e] = dnlo;
  }
}

// fraction-to-boundary minima (ip.py:189-222): {min (upper-rho)/drho over drho > 0,
// min (lower-rho)/drho over drho < 0, min -nu_lo/dnu_lo over dnu_lo < 0, min -nu_up/dnu_up
// over dnu_up < 0}; +inf where the set is empty.  Exact (min is order-free).
__global__ void __launch_bounds__(kThreads) k_ip_steps(int m, const double* __restrict__ rho,
                                                     const double* __restrict__ drho,
                                                     const double* __restrict__ nu_lo,
                                                     const double* __restrict__ dnu_lo,
                                                     const double* __restrict__ nu_up,
                                                     const double* __restrict__ dnu_up,
                                                     const double* __restrict__ lower,
                                                     const double* __restrict__ upper, double* mins) {
  __shared__ double sm[4][kThreads / 32];
  double v[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    const double d = drho[e], rh = rho[e];
    if (d > 0.0) v[0] = fmin(v[0], __dsub_rn(upper[e], rh) / d);
    if (d < 0.0) v[1] = fmin(v[1], __dsub_rn(lower[e], rh) / d);
    const double dl = dnu_lo[e], du = dnu_up[e];
    if (dl < 0.0) v[2] = fmin(v[2], -nu_lo[e] / dl);
    if (du < 0.0) v[3] = fmin(v[3], -nu_up[e] / du);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
    for (int o = 16; o > 0; o >>= 1) v[i] = fmin(v[i], __shfl_xor_sync(0xffffffffu, v[i], o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0)
    for (int i = 0; i < 4; ++i) sm[i][warp] = v[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
      for (int i = 0; i < 4; ++i) v[i] = fmin(v[i], sm[i][k]);
    for (int i = 0; i < 4; ++i) mins[4 * blockIdx.x + i] = v[i];
  }
}

__global__ void k_ip_steps_finish(int nb, const double* __restrict__ pm, double* out) {
  double v[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
  for (int b = 0; b < nb; ++b)
    for (int i = 0; i < 4; ++i) v[i] = fmin(v[i], pm[4 * b + i]);
  for (int i = 0; i < 4; ++i) out[i] = v[i];
}

// ---------------------------------------------------------------------------
// host wrappers
// ---------------------------------------------------------------------------
int ip_residual(Ctx* c, const double* u, double alpha, const double* rho, const double* nu_lo,
                const double* nu_up, double r, double s, const double* lower, const double* upper, double volume,
                const double* f, double norm_f, double* q, double* res_c, double* res_lo, double* res_up,
                double* res_u, double* scalars) {
  const int F = c->L - 1;
  const LevelDev& d = c->lv[F].d;
  double* ug = c->fvec[0];
  if (int rc = free_to_grid(c, F, u, ug, false)) return rc;
  const int ge = reduce_grid(c->m);
  double* pe = c->partials;                          // 8 per block
  double* pn = c->partials + kMaxBlocks * 8;         // 2 per block (k_phi_node)
  double* pm = c->partials + kMaxBlocks * 10;        // 3 per block
  k_ip_elem<<<ge, kThreads, 0, c->stream>>>(c->m, d.ex, d.nx, ug, alpha, rho, nu_lo, nu_up, lower, upper, r, s, q,
                                             res_c, res_lo, res_up, pe, pm);
  VTS_LAUNCHED(c);
  // res_u = scatter(rho w) - f (ip.py:123): the PBM node pass with rho as the weight
  const int gn = reduce_grid(d.nnodes);
  k_phi_node<<<gn, kThreads, 0, c->stream>>>(d.nnodes, d.nx, d.ex, d.ey, ug, rho, f, c->lv[F].grid2free, res_u,
                                              pn);
  VTS_LAUNCHED(c);
  k_ip_finish<<<1, kThreads, 0, c->stream>>>(ge, pe, pm, gn, pn, c->m, volume, norm_f, c->dscal);
  VTS_LAUNCHED(c);
  if (int rc = sync_scalars(c, 9)) return rc;
  for (int i = 0; i < 9; ++i) scalars[i] = c->hscal[i];
  return 0;
}

int ip_schur_system(Ctx* c, const double* u, const double* rho, const double* nu_lo, const double* nu_up,
                    const double* lower, const double* upper, const double* res_c, const double* res_lo,
                    const double* res_up, const double* res_u, double res_alpha, double* dcoef, double* g,
                    double* rhs, double* corner) {
  const int F = c->L - 1;
  const LevelDev& d = c->lv[F].d;
  if (int rc = free_to_grid(c, F, u, c->u_grid, false)) return rc;
  double* tcoef = c->fvec[1];  // m <= ngrid, scratch
  const int ge = reduce_grid(c->m);
  k_ip_schur_elem<<<ge, kThreads, 0, c->stream>>>(c->m, rho, nu_lo, nu_up, lower, upper, res_c, res_lo, res_up,
                                                   dcoef, g, c->chat, c->rho_hat, tcoef, c->partials);
  VTS_LAUNCHED(c);
  // rhs: core -res_u + scatter(t w) = -res_u - scatter((g/D) w) (ip.py:156), border
  // entry -(-(-res_alpha) - sum t) = -res_alpha - sum g/D (ip.py:157): the reference's
  // convention; the API edge flips it (border_flip) for the bound E S+ E
  k_schur_node<<<reduce_grid(d.nnodes), kThreads, 0, c->stream>>>(d.nnodes, d.nx, d.ex, d.ey, c->u_grid, tcoef,
                                                                   c->chat, res_u, c->lv[F].grid2free, rhs,
                                                                   nullptr, c->lv[F].d.border);
  VTS_LAUNCHED(c);
  k_schur_finish<<<1, kThreads, 0, c->stream>>>(ge, c->partials, -res_alpha, -1.0, c->n, rhs, c->d_corner,
                                                c->dscal);
  VTS_LAUNCHED(c);
  if (int rc = sync_scalars(c, 2)) return rc;
  c->corner = c->hscal[0];
  if (corner) *corner = c->corner;
  c->system_bound = true;
  c->border_flip = true;
  c->unbordered = false;
  c->mg_ready = false;
  return 0;
}

int ip_reconstruct(Ctx* c, const double* u, const double* du, double dalpha, const double* dcoef, const double* g,
                   const double* res_c, const double* res_lo, const double* res_up, const double* rho,
                   const double* nu_lo, const double* nu_up, const double* lower, const double* upper, double* drho,
                   double* dnu_up, double* dnu_lo) {
  const int F = c->L - 1;
  const LevelDev& d = c->lv[F].d;
  double* ug = c->fvec[0];
  double* dug = c->fvec[2];
  if (int rc = free_to_grid(c, F, u, ug, false)) return rc;
  if (int rc = free_to_grid(c, F, du, dug, false)) return rc;
  k_ip_recon_elem<<<reduce_grid(c->m), kThreads, 0, c->stream>>>(c->m, d.ex, d.nx, ug, dug, dalpha, dcoef, g, res_c,
                                                                  res_lo, res_up, rho, nu_lo, nu_up, lower, upper,
                                                                  drho, dnu_up, dnu_lo);
  VTS_LAUNCHED(c);
  VTS_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

int ip_step_bounds(Ctx* c, const double* rho, const double* drho, const double* nu_lo, const double* dnu_lo,
                   const double* nu_up, const double* dnu_up, const double* lower, const double* upper,
                   double* mins) {
  const int ge = reduce_grid(c->m);
  double* pm = c->partials;
  k_ip_steps<<<ge, kThreads, 0, c->stream>>>(c->m, rho, drho, nu_lo, dnu_lo, nu_up, dnu_up, lower, upper, pm);
  VTS_LAUNCHED(c);
  k_ip_steps_finish<<<1, 1, 0, c->stream>>>(ge, pm, c->dscal);
  VTS_LAUNCHED(c);
  if (int rc = sync_scalars(c, 4)) return rc;
  for (int i = 0; i < 4; ++i) mins[i] = c->hscal[i];
  return 0;
}

}  // namespace vts
