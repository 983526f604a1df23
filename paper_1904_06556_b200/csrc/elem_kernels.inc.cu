// Element and nodal passes of the PBM Newton step (unity-built into vts_b200.cu).
//
//  * k_phi_elem / k_phi_node      : eval_lagrangian          (pbm.py:150-199)
//  * k_schur_elem / k_schur_node  : schur_system coeffs/rhs  (pbm.py:202-218, fem.py:206-208)
//  * k_recon_elem                 : reconstruct_nu + slope   (pbm.py:221-232, 290-295)
//  * k_al_elem                    : _al_value at x + k dx    (pbm.py:135-147, 300-305)
//  * k_outer_update, k_gap_elem   : pbm.py:397-402, model.py:50-79
//
// All of these are HBM-bound single passes: one thread per element (or node),
// coalesced fp64 loads of the element arrays, the 8 nodal u values gathered
// from the node grid (16 B per node, L1/L2-shared between the 4 elements of a
// node), K_e from constant memory (uniform broadcast), and deterministic
// fixed-order block reductions finished by the last block to arrive.

namespace vts {

constexpr int kThreads = 256;
constexpr int kReduceGridCap = 148 * 8;  // grid-stride reductions: 8 CTAs per SM

// ---------------------------------------------------------------------------
// last-block deterministic reduction
// ---------------------------------------------------------------------------
// Every block contributes NV partial sums; the last block to finish sums them
// in block order (each thread a fixed strided subset, then the fixed block
// tree) and returns true with the totals in tot[] (valid in thread 0).
#ifndef VTS_REDUCE_SC
#define VTS_REDUCE_SC 0
#endif
// VTS_REDUCE_SC=1 (compile time) restores the sequentially consistent fence + atomic (A/B)
VTS_DEVICE_INLINE constexpr bool reduce_acq_rel() { return VTS_REDUCE_SC == 0; }

template <int NV>
__device__ bool last_block_reduce(double (&v)[NV], double* scratch, double* partials,
                                  unsigned* counter, double (&tot)[NV]) {
  __shared__ bool s_last;
  block_sum<NV>(v, scratch);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) partials[blockIdx.x * NV + i] = v[i];
    unsigned ticket;
    if (reduce_acq_rel()) {
      // release: this block's partials before its ticket; acquire: the last block
      // sees every partial released before the tickets it counted (the other
      // threads of the block are ordered behind thread 0 by the barrier below)
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(ticket) : "l"(counter) : "memory");
    } else {
      __threadfence();
      ticket = atomicAdd(counter, 1u);
    }
    s_last = (ticket == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return false;
  if (!reduce_acq_rel()) __threadfence();
#pragma unroll
  for (int i = 0; i < NV; ++i) tot[i] = 0.0;
  // thread t sums blocks t, t + blockDim, ... in that order; the loads of a
  // round of kU blocks are all issued before the first add (one L2 round
  // trip per round instead of one per block; absent blocks add +0.0)
  constexpr int kU = NV >= 4 ? 2 : 8;  // loads in flight per thread (registers: kU x NV)
  for (int b0 = threadIdx.x; b0 < (int)gridDim.x; b0 += kU * blockDim.x) {
    double v[kU][NV];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int b = b0 + u * blockDim.x;
#pragma unroll
      for (int i = 0; i < NV; ++i) v[u][i] = b < (int)gridDim.x ? __ldcg(partials + b * NV + i) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int i = 0; i < NV; ++i) tot[i] += v[u][i];
  }
  block_sum<NV>(tot, scratch);
  if (threadIdx.x == 0) *counter = 0u;
  return true;
}

VTS_DEVICE_INLINE void elem_nodes(int e, int ex, int nx, int (&nd)[4]) {
  const int exi = e % ex, eyi = e / ex;
  const int n0 = exi + nx * eyi;
  nd[0] = n0;
  nd[1] = n0 + 1;
  nd[2] = n0 + nx + 1;
  nd[3] = n0 + nx;
}

VTS_DEVICE_INLINE void gather8(const double* __restrict__ g, const int (&nd)[4], double (&ue)[8]) {
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const double2 v = *reinterpret_cast<const double2*>(g + 2 * nd[a]);
    ue[2 * a] = v.x;
    ue[2 * a + 1] = v.y;
  }
}

// w = u_e K_e  (fem.py:178 `ue @ ke`; K_e symmetric)
VTS_DEVICE_INLINE void ke_times(const double (&ue)[8], double (&w)[8]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    double s = ue[0] * c_ke[j];
#pragma unroll
    for (int i = 1; i < 8; ++i) s = fma(ue[i], c_ke[i * 8 + j], s);
    w[j] = s;
  }
}

// the two rows of u_e K_e belonging to local corner li
VTS_DEVICE_INLINE void ke_rows(const double (&ue)[8], int li, double& w0, double& w1) {
  double s0 = ue[0] * c_ke[2 * li], s1 = ue[0] * c_ke[2 * li + 1];
#pragma unroll
  for (int i = 1; i < 8; ++i) {
    s0 = fma(ue[i], c_ke[i * 8 + 2 * li], s0);
    s1 = fma(ue[i], c_ke[i * 8 + 2 * li + 1], s1);
  }
  w0 = s0;
  w1 = s1;
}

VTS_DEVICE_INLINE double dot8(const double (&a)[8], const double (&b)[8]) {
  double s = a[0] * b[0];
#pragma unroll
  for (int i = 1; i < 8; ++i) s = fma(a[i], b[i], s);
  return s;
}

// the four elements around node (ix, iy), in increasing element index (the
// accumulation order of the reference's bincount scatter, fem.py:170-173):
// (ix-1,iy-1) corner 2, (ix,iy-1) corner 3, (ix-1,iy) corner 1, (ix,iy) corner 0
struct NodeElems {
  int e[4];
  int li[4];
  int cnt;
};

VTS_DEVICE_INLINE NodeElems node_elems(int ix, int iy, int ex, int ey) {
  NodeElems r;
  r.cnt = 0;
  if (ix >= 1 && iy >= 1) { r.e[r.cnt] = (ix - 1) + ex * (iy - 1); r.li[r.cnt++] = 2; }
  if (ix < ex && iy >= 1) { r.e[r.cnt] = ix + ex * (iy - 1); r.li[r.cnt++] = 3; }
  if (ix >= 1 && iy < ey) { r.e[r.cnt] = (ix - 1) + ex * iy; r.li[r.cnt++] = 1; }
  if (ix < ex && iy < ey) { r.e[r.cnt] = ix + ex * iy; r.li[r.cnt++] = 0; }
  return r;
}

// ---------------------------------------------------------------------------
// layout conversions
// ---------------------------------------------------------------------------
__global__ void k_free_to_grid(int ngrid, int nfree, const int32_t* __restrict__ g2f,
                               const double* __restrict__ src, double* __restrict__ dst,
                               int bordered, const int* skip = nullptr) {
  if (skip && *skip) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < ngrid) {
    const int f = g2f[i];
    dst[i] = f >= 0 ? src[f] : 0.0;
  } else if (i == ngrid && bordered) {
    // -1: the bound system is E S+ E (ip.inc.cu); 2: unbordered K (no slot in src)
    dst[ngrid] = bordered == 2 ? 0.0 : (bordered < 0 ? -src[nfree] : src[nfree]);
  }
}

__global__ void k_grid_to_free(int nfree, int ngrid, const int32_t* __restrict__ f2g,
                               const double* __restrict__ src, double* __restrict__ dst,
                               int bordered) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nfree) dst[i] = src[f2g[i]];
  else if (i == nfree && bordered && bordered != 2) dst[nfree] = bordered < 0 ? -src[ngrid] : src[ngrid];
}

// trial displacement u + kappa du on the grid, with f . (u + kappa du)
// kappa_dev / skip (device-resident Newton step, step.inc.cu): the trial step from device
// memory, and the launch is a no-op once the line search has decided
__global__ void k_trial_grid(int ngrid, const int32_t* __restrict__ g2f, const double* __restrict__ u,
                             const double* __restrict__ du, double kappa,
                             const double* __restrict__ f, double* __restrict__ out,
                             double* partials, unsigned* counter, double* result,
                             const double* kappa_dev = nullptr, const int* skip = nullptr) {
  if (skip && *skip) return;
  if (kappa_dev) kappa = *kappa_dev;
  __shared__ double scratch[kThreads / 32];
  double acc[1] = {0.0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ngrid; i += gridDim.x * blockDim.x) {
    const int fi = g2f[i];
    double v = 0.0;
    if (fi >= 0) {
      v = __dadd_rn(u[fi], __dmul_rn(kappa, du[fi]));
      acc[0] = fma(f[fi], v, acc[0]);
    }
    out[i] = v;
  }
  double tot[1];
  if (last_block_reduce<1>(acc, scratch, partials, counter, tot) && threadIdx.x == 0) result[0] = tot[0];
}

// generic deterministic dot product of two length-len vectors
__global__ void k_dot(long long len, const double* __restrict__ a, const double* __restrict__ b,
                      double* partials, unsigned* counter, double* result, const int* skip) {
  if (skip && *skip) return;
  __shared__ double scratch[kThreads / 32];
  double acc[1] = {0.0};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < len;
       i += (long long)gridDim.x * blockDim.x)
    acc[0] = fma(a[i], b[i], acc[0]);
  double tot[1];
  if (last_block_reduce<1>(acc, scratch, partials, counter, tot) && threadIdx.x == 0) result[0] = tot[0];
}

__global__ void k_axpy(long long len, double kappa, const double* __restrict__ dx, double* x,
                       const double* kappa_dev = nullptr, const int* skip = nullptr) {
  if (skip && *skip) return;
  if (kappa_dev) kappa = *kappa_dev;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < len;
       i += (long long)gridDim.x * blockDim.x)
    x[i] = __dadd_rn(x[i], __dmul_rn(kappa, dx[i]));
}

// ---------------------------------------------------------------------------
// eval_lagrangian
// ---------------------------------------------------------------------------
struct PhiElemArgs {
  int m, ex, nx;
  const double* ug;
  double alpha, branch;
  const double *nu_lo, *nu_up, *rho, *mu_lo, *mu_up, *p, *q_lo, *q_up, *lower, *upper;
  double *q, *rho_hat, *mu_hat_lo, *mu_hat_up, *a, *b_lo, *b_up, *res_lo, *res_up, *w_out;
  const double* alpha_dev = nullptr;  // device-resident Newton step: alpha from device memory
  const int* skip = nullptr;          //   and the evaluation is skipped while *skip != 0
};

__global__ void __launch_bounds__(kThreads, 2) k_phi_elem(PhiElemArgs A, double* partials, unsigned* flags) {
  if (A.skip && *A.skip) return;
  __shared__ double scratch[7 * kThreads / 32];
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  unsigned sat = 0;
  const double alpha = A.alpha_dev ? *A.alpha_dev : A.alpha;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < A.m; e += gridDim.x * blockDim.x) {
    int nd[4];
    elem_nodes(e, A.ex, A.nx, nd);
    double ue[8], w[8];
    gather8(A.ug, nd, ue);
    ke_times(ue, w);
    double qq = w[0] * ue[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) qq = fma(w[i], ue[i], qq);
    qq = 0.5 * qq;
    const double nlo = A.nu_lo[e], nup = A.nu_up[e], pe = A.p[e], qlo = A.q_lo[e], qup = A.q_up[e];
    const double rh = A.rho[e], mlo = A.mu_lo[e], mup = A.mu_up[e];
    const double s = __dsub_rn(__dadd_rn(__dsub_rn(qq, alpha), nlo), nup);
    const PhiOut f1 = phi_eval(s / pe, A.branch, &sat);
    const PhiOut f2 = phi_eval(-nlo / qlo, A.branch, &sat);
    const PhiOut f3 = phi_eval(-nup / qup, A.branch, &sat);
    const double rho_hat = rh * f1.d1;
    const double mhl = mlo * f2.d1, mhu = mup * f3.d1;
    const double lo = A.lower[e], up = A.upper[e];
    const double rlo = __dsub_rn(__dadd_rn(-lo, rho_hat), mhl);
    const double rup = __dsub_rn(__dsub_rn(up, rho_hat), mhu);
    A.q[e] = qq;
    A.rho_hat[e] = rho_hat;
    A.mu_hat_lo[e] = mhl;
    A.mu_hat_up[e] = mhu;
    A.a[e] = (rh / pe) * f1.d2;
    A.b_lo[e] = (mlo / qlo) * f2.d2;
    A.b_up[e] = (mup / qup) * f3.d2;
    A.res_lo[e] = rlo;
    A.res_up[e] = rup;
    if (A.w_out) {
#pragma unroll
      for (int j = 0; j < 8; j += 2)
        *reinterpret_cast<double2*>(A.w_out + 8 * (size_t)e + j) = make_double2(w[j], w[j + 1]);
    }
    acc[0] += rh * __dmul_rn(pe, f1.v);
    acc[1] += mlo * __dmul_rn(qlo, f2.v);
    acc[2] += mup * __dmul_rn(qup, f3.v);
    acc[3] += rho_hat;
    acc[4] = fma(rlo, rlo, acc[4]);
    acc[5] = fma(lo, nlo, acc[5]);
    acc[6] = fma(up, nup, acc[6]);
  }
  if (sat) atomicOr(flags, 1u);
  block_partials<7>(acc, scratch, partials);
}

// res_u = scatter(rho_hat w) - f, written in free order; ||res_u||^2 and f.u partials
__global__ void __launch_bounds__(kThreads) k_phi_node(int nnodes, int nx, int ex, int ey,
                                                     const double* __restrict__ ug,
                                                     const double* __restrict__ rho_hat,
                                                     const double* __restrict__ f,
                                                     const int32_t* __restrict__ g2f,
                                                     double* __restrict__ res_u, double* partials,
                                                     const int* skip = nullptr) {
  if (skip && *skip) return;
  __shared__ double scratch[2 * kThreads / 32];
  double acc[2] = {0, 0};
  for (int nd = blockIdx.x * blockDim.x + threadIdx.x; nd < nnodes; nd += gridDim.x * blockDim.x) {
    const int ix = nd % nx, iy = nd / nx;
    const NodeElems ne = node_elems(ix, iy, ex, ey);
    double s0 = 0.0, s1 = 0.0;
    for (int k = 0; k < ne.cnt; ++k) {
      int n4[4];
      elem_nodes(ne.e[k], ex, nx, n4);
      double ue[8];
      gather8(ug, n4, ue);
      double w0, w1;
      ke_rows(ue, ne.li[k], w0, w1);
      const double rh = rho_hat[ne.e[k]];
      s0 = __dadd_rn(s0, __dmul_rn(rh, w0));
      s1 = __dadd_rn(s1, __dmul_rn(rh, w1));
    }
    const int f0 = g2f[2 * nd], f1 = g2f[2 * nd + 1];
    if (f0 >= 0) {
      const double r = __dsub_rn(s0, f[f0]);
      res_u[f0] = r;
      acc[0] = fma(r, r, acc[0]);
      acc[1] = fma(f[f0], ug[2 * nd], acc[1]);
    }
    if (f1 >= 0) {
      const double r = __dsub_rn(s1, f[f1]);
      res_u[f1] = r;
      acc[0] = fma(r, r, acc[0]);
      acc[1] = fma(f[f1], ug[2 * nd + 1], acc[1]);
    }
  }
  block_partials<2>(acc, scratch, partials);
}

// ---------------------------------------------------------------------------
// eval_lagrangian in one launch: k_phi_elem's element pass and k_phi_node's
// scatter fused per tile.  A CTA owns the elements [x0, x0 + 31) x [y0, y0 + 7)
// and the nodes [x0, x0 + 31) x [y0, y0 + 7); its 32 x 8 threads compute the
// elements [x0 - 1, x0 + 31) x [y0 - 1, y0 + 7) (one halo column and row, whose
// outputs the neighbouring tiles write), put rho_hat w_e in shared memory and
// every owned node sums its four contributions in the reference's scatter
// order (fem.py:170-173): the same arithmetic as the two-kernel pass, element
// products computed once per element instead of once per node and corner.  The
// nine partial sums end in a last-block reduction that forms the scalars
// (k_phi_finish's arithmetic).
// ---------------------------------------------------------------------------
constexpr int kPhiTX = 32, kPhiTY = 8;
#ifndef VTS_PHI_MINB
#define VTS_PHI_MINB 4  // 64 registers: 4 CTAs per SM (2: 74 us, 3: 59 us, 4: 55 us on C3)
#endif

struct PhiTileArgs {
  int nx, ny, ey, tiles_x, ntiles;  // ntiles: informational (the grid has one CTA per tile)
  const double* f;
  const int32_t* g2f;
  double* res_u;
  double volume, norm_f, norm_bounds;
  double* out;
};

__global__ void __launch_bounds__(kPhiTX * kPhiTY, VTS_PHI_MINB) k_phi_tile(PhiElemArgs A, PhiTileArgs T, double* partials,
                                                                  unsigned* counter, unsigned* flags) {
  if (A.skip && *A.skip) return;
  __shared__ double contrib[8][kPhiTX * kPhiTY];
  __shared__ double scratch[9 * kPhiTX * kPhiTY / 32];
  const int tid = threadIdx.x, lx = tid % kPhiTX, ly = tid / kPhiTX;
  const double alpha = A.alpha_dev ? *A.alpha_dev : A.alpha;
  double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  unsigned sat = 0;
  const int x0 = (blockIdx.x % T.tiles_x) * (kPhiTX - 1), y0 = (blockIdx.x / T.tiles_x) * (kPhiTY - 1);
  const int exi = x0 - 1 + lx, eyi = y0 - 1 + ly;
  const bool in_mesh = exi >= 0 && exi < A.ex && eyi >= 0 && eyi < T.ey;
  const bool owned = in_mesh && lx >= 1 && ly >= 1;
  double w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  double rho_hat = 0.0;
  if (in_mesh) {
    const int e = exi + A.ex * eyi;
    int nd[4];
    elem_nodes(e, A.ex, A.nx, nd);
    double ue[8];
    gather8(A.ug, nd, ue);
    ke_times(ue, w);
    double qq = w[0] * ue[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) qq = fma(w[i], ue[i], qq);
    qq = 0.5 * qq;
    const double nlo = A.nu_lo[e], nup = A.nu_up[e], pe = A.p[e], qlo = A.q_lo[e], qup = A.q_up[e];
    const double rh = A.rho[e], mlo = A.mu_lo[e], mup = A.mu_up[e];
    const double s = __dsub_rn(__dadd_rn(__dsub_rn(qq, alpha), nlo), nup);
    const PhiOut f1 = phi_eval(s / pe, A.branch, &sat);
    rho_hat = rh * f1.d1;
    if (owned) {
      const PhiOut f2 = phi_eval(-nlo / qlo, A.branch, &sat);
      const PhiOut f3 = phi_eval(-nup / qup, A.branch, &sat);
      const double mhl = mlo * f2.d1, mhu = mup * f3.d1;
      const double lo = A.lower[e], up = A.upper[e];
      const double rlo = __dsub_rn(__dadd_rn(-lo, rho_hat), mhl);
      const double rup = __dsub_rn(__dsub_rn(up, rho_hat), mhu);
      A.q[e] = qq;
      A.rho_hat[e] = rho_hat;
      A.mu_hat_lo[e] = mhl;
      A.mu_hat_up[e] = mhu;
      A.a[e] = (rh / pe) * f1.d2;
      A.b_lo[e] = (mlo / qlo) * f2.d2;
      A.b_up[e] = (mup / qup) * f3.d2;
      A.res_lo[e] = rlo;
      A.res_up[e] = rup;
      if (A.w_out) {
#pragma unroll
        for (int j = 0; j < 8; j += 2)
          *reinterpret_cast<double2*>(A.w_out + 8 * (size_t)e + j) = make_double2(w[j], w[j + 1]);
      }
      acc[0] += rh * __dmul_rn(pe, f1.v);
      acc[1] += mlo * __dmul_rn(qlo, f2.v);
      acc[2] += mup * __dmul_rn(qup, f3.v);
      acc[3] += rho_hat;
      acc[4] = fma(rlo, rlo, acc[4]);
      acc[5] = fma(lo, nlo, acc[5]);
      acc[6] = fma(up, nup, acc[6]);
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) contrib[j][tid] = __dmul_rn(rho_hat, w[j]);
  __syncthreads();
  // node (x0 + lx, y0 + ly): elements (ix-1, iy-1) corner 2, (ix, iy-1) corner 3,
  // (ix-1, iy) corner 1, (ix, iy) corner 0 -- local elements (lx, ly), (lx+1, ly),
  // (lx, ly+1), (lx+1, ly+1)
  const int ix = x0 + lx, iy = y0 + ly;
  if (lx < kPhiTX - 1 && ly < kPhiTY - 1 && ix < T.nx && iy < T.ny) {
    double s0 = 0.0, s1 = 0.0;
    if (ix >= 1 && iy >= 1) {
      s0 = __dadd_rn(s0, contrib[4][tid]);
      s1 = __dadd_rn(s1, contrib[5][tid]);
    }
    if (ix < A.ex && iy >= 1) {
      s0 = __dadd_rn(s0, contrib[6][tid + 1]);
      s1 = __dadd_rn(s1, contrib[7][tid + 1]);
    }
    if (ix >= 1 && iy < T.ey) {
      s0 = __dadd_rn(s0, contrib[2][tid + kPhiTX]);
      s1 = __dadd_rn(s1, contrib[3][tid + kPhiTX]);
    }
    if (ix < A.ex && iy < T.ey) {
      s0 = __dadd_rn(s0, contrib[0][tid + kPhiTX + 1]);
      s1 = __dadd_rn(s1, contrib[1][tid + kPhiTX + 1]);
    }
    const int nd = ix + A.nx * iy;
    const int f0 = T.g2f[2 * nd], f1 = T.g2f[2 * nd + 1];
    if (f0 >= 0) {
      const double r = __dsub_rn(s0, T.f[f0]);
      T.res_u[f0] = r;
      acc[7] = fma(r, r, acc[7]);
      acc[8] = fma(T.f[f0], A.ug[2 * nd], acc[8]);
    }
    if (f1 >= 0) {
      const double r = __dsub_rn(s1, T.f[f1]);
      T.res_u[f1] = r;
      acc[7] = fma(r, r, acc[7]);
      acc[8] = fma(T.f[f1], A.ug[2 * nd + 1], acc[8]);
    }
  }
  if (sat) atomicOr(flags, 1u);
  double t[9];
  if (last_block_reduce<9>(acc, scratch, partials, counter, t) && threadIdx.x == 0) {
    // k_phi_finish: dual_objective (model.py:61-66) + the penalty sums (pbm.py:161-166)
    const double fu = t[8];
    const double dual = ((alpha * T.volume - fu) - t[5]) + t[6];
    const double value = ((dual + t[0]) + t[1]) + t[2];
    const double res_alpha = T.volume - t[3];
    const double tau = (sqrt(t[7]) / T.norm_f + fabs(res_alpha) / T.volume) + sqrt(t[4]) / T.norm_bounds;
    T.out[0] = value;
    T.out[1] = res_alpha;
    T.out[2] = tau;
    T.out[3] = fu;
    T.out[4] = t[3];
    T.out[5] = sqrt(t[7]);
    T.out[6] = sqrt(t[4]);
    T.out[7] = 0.0;
  }
}

// sums the two partial arrays and forms the eval scalars
__global__ void k_phi_finish(int nb_e, const double* __restrict__ pe, int nb_n,
                             const double* __restrict__ pn, double alpha, double volume,
                             double norm_f, double norm_bounds, double* out, const double* alpha_dev = nullptr,
                             const int* skip = nullptr) {
  if (skip && *skip) return;
  if (alpha_dev) alpha = *alpha_dev;
  __shared__ double scratch[9 * kThreads / 32];
  double t[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int b = threadIdx.x; b < nb_e; b += blockDim.x)
    for (int i = 0; i < 7; ++i) t[i] += pe[b * 7 + i];
  for (int b = threadIdx.x; b < nb_n; b += blockDim.x)
    for (int i = 0; i < 2; ++i) t[7 + i] += pn[b * 2 + i];
  block_sum<9>(t, scratch);
  if (threadIdx.x == 0) {
    const double fu = t[8];
    // dual_objective (model.py:61-66) + the three penalty sums (pbm.py:161-166)
    const double dual = ((alpha * volume - fu) - t[5]) + t[6];
    const double value = ((dual + t[0]) + t[1]) + t[2];
    const double res_alpha = volume - t[3];
    const double tau = (sqrt(t[7]) / norm_f + fabs(res_alpha) / volume) + sqrt(t[4]) / norm_bounds;
    out[0] = value;
    out[1] = res_alpha;
    out[2] = tau;
    out[3] = fu;
    out[4] = t[3];
    out[5] = sqrt(t[7]);
    out[6] = sqrt(t[4]);
    out[7] = 0.0;
  }
}

// ---------------------------------------------------------------------------
// schur_system
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_schur_elem(int m, const double* __restrict__ a,
                                                       const double* __restrict__ b_lo,
                                                       const double* __restrict__ b_up,
                                                       const double* __restrict__ res_lo,
                                                       const double* __restrict__ res_up,
                                                       const double* __restrict__ rho_hat,
                                                       double* chat_out, double* chat_ctx,
                                                       double* rho_hat_ctx, double* t_out,
                                                       double* partials) {
  __shared__ double scratch[2 * kThreads / 32];
  double acc[2] = {0, 0};
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    const double ae = a[e], bl = b_lo[e], bu = b_up[e];
    // pbm.py:210-212, evaluated in the reference's operation order
    const double det = __dadd_rn(__dadd_rn(__dmul_rn(ae, bl), __dmul_rn(ae, bu)), __dmul_rn(bl, bu));
    const double ch = __dmul_rn(__dmul_rn(ae, bl), bu) / det;
    const double tt = __dmul_rn(ae, __dsub_rn(__dmul_rn(bu, res_lo[e]), __dmul_rn(bl, res_up[e]))) / det;
    if (chat_out) chat_out[e] = ch;
    chat_ctx[e] = ch;
    rho_hat_ctx[e] = rho_hat[e];
    t_out[e] = tt;
    acc[0] += tt;
    acc[1] += ch;
  }
  block_partials<2>(acc, scratch, partials);
}

// rhs_u = -res_u + scatter(t w);  border = -scatter(chat w)  (pbm.py:216, fem.py:206)
__global__ void __launch_bounds__(kThreads) k_schur_node(int nnodes, int nx, int ex, int ey,
                                                       const double* __restrict__ ug,
                                                       const double* __restrict__ tcoef,
                                                       const double* __restrict__ chat,
                                                       const double* __restrict__ res_u,
                                                       const int32_t* __restrict__ g2f,
                                                       double* __restrict__ rhs,
                                                       double* __restrict__ border_free,
                                                       double* __restrict__ border_grid) {
  for (int nd = blockIdx.x * blockDim.x + threadIdx.x; nd < nnodes; nd += gridDim.x * blockDim.x) {
    const int ix = nd % nx, iy = nd / nx;
    const NodeElems ne = node_elems(ix, iy, ex, ey);
    double t0 = 0.0, t1 = 0.0, c0 = 0.0, c1 = 0.0;
    for (int k = 0; k < ne.cnt; ++k) {
      int n4[4];
      elem_nodes(ne.e[k], ex, nx, n4);
      double ue[8];
      gather8(ug, n4, ue);
      double w0, w1;
      ke_rows(ue, ne.li[k], w0, w1);
      const double tt = tcoef[ne.e[k]], ch = chat[ne.e[k]];
      t0 = __dadd_rn(t0, __dmul_rn(tt, w0));
      t1 = __dadd_rn(t1, __dmul_rn(tt, w1));
      c0 = __dadd_rn(c0, __dmul_rn(ch, w0));
      c1 = __dadd_rn(c1, __dmul_rn(ch, w1));
    }
    const int f0 = g2f[2 * nd], f1 = g2f[2 * nd + 1];
    double bg0 = 0.0, bg1 = 0.0;
    if (f0 >= 0) {
      rhs[f0] = __dadd_rn(-res_u[f0], t0);
      bg0 = -c0;
      if (border_free) border_free[f0] = bg0;
    }
    if (f1 >= 0) {
      rhs[f1] = __dadd_rn(-res_u[f1], t1);
      bg1 = -c1;
      if (border_free) border_free[f1] = bg1;
    }
    *reinterpret_cast<double2*>(border_grid + 2 * nd) = make_double2(bg0, bg1);
  }
}

__global__ void k_schur_finish(int nb, const double* __restrict__ pe, double res_alpha, double sign, int n,
                               double* rhs, double* d_corner, double* out, const double* res_alpha_dev = nullptr) {
  if (res_alpha_dev) res_alpha = *res_alpha_dev;
  __shared__ double scratch[2 * kThreads / 32];
  double t[2] = {0, 0};
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    t[0] += pe[b * 2];
    t[1] += pe[b * 2 + 1];
  }
  block_sum<2>(t, scratch);
  if (threadIdx.x == 0) {
    rhs[n] = sign * (-res_alpha - t[0]);
    *d_corner = t[1];
    out[0] = t[1];
    out[1] = t[0];
  }
}

// ---------------------------------------------------------------------------
// reconstruct_nu + slope partials (element part)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_recon_elem(int m, int ex, int nx,
                                                       const double* __restrict__ ug,
                                                       const double* __restrict__ dug, double dalpha,
                                                       const double* __restrict__ res_lo,
                                                       const double* __restrict__ res_up,
                                                       const double* __restrict__ a,
                                                       const double* __restrict__ b_lo,
                                                       const double* __restrict__ b_up,
                                                       double* dnu_lo, double* dnu_up,
                                                       double* partials, const double* dalpha_dev = nullptr) {
  __shared__ double scratch[2 * kThreads / 32];
  double acc[2] = {0, 0};
  if (dalpha_dev) dalpha = *dalpha_dev;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    int nd[4];
    elem_nodes(e, ex, nx, nd);
    double ue[8], w[8], de[8];
    gather8(ug, nd, ue);
    ke_times(ue, w);
    gather8(dug, nd, de);
    const double theta = __dsub_rn(dot8(w, de), dalpha);
    const double ae = a[e], bl = b_lo[e], bu = b_up[e];
    const double det = __dadd_rn(__dadd_rn(__dmul_rn(ae, bl), __dmul_rn(ae, bu)), __dmul_rn(bl, bu));
    const double glo = __dadd_rn(res_lo[e], __dmul_rn(ae, theta));
    const double gup = __dsub_rn(res_up[e], __dmul_rn(ae, theta));
    const double dl = -__dadd_rn(__dmul_rn(__dadd_rn(ae, bu), glo), __dmul_rn(ae, gup)) / det;
    const double du = -__dadd_rn(__dmul_rn(ae, glo), __dmul_rn(__dadd_rn(ae, bl), gup)) / det;
    dnu_lo[e] = dl;
    dnu_up[e] = du;
    acc[0] = fma(res_lo[e], dl, acc[0]);
    acc[1] = fma(res_up[e], du, acc[1]);
  }
  block_partials<2>(acc, scratch, partials);
}

// slope = res_u.du + res_alpha dalpha + res_lo.dnu_lo + res_up.dnu_up (pbm.py:290-295): the
// element partials of k_recon_elem summed in block order, then the reference's sum order
__global__ void k_slope_finish(int nb, const double* __restrict__ pe, const double* __restrict__ dot, double res_alpha,
                               double dalpha, double* out) {
  double s_lo = 0.0, s_up = 0.0;
  for (int b = 0; b < nb; ++b) {
    s_lo = __dadd_rn(s_lo, pe[2 * b]);
    s_up = __dadd_rn(s_up, pe[2 * b + 1]);
  }
  *out = __dadd_rn(__dadd_rn(__dadd_rn(*dot, __dmul_rn(res_alpha, dalpha)), s_lo), s_up);
}

// ---------------------------------------------------------------------------
// _al_value at the trial point (element part)
// ---------------------------------------------------------------------------
struct AlElemArgs {
  int m, ex, nx;
  const double* ug;  // trial u on the grid
  double alpha, kappa, branch;
  const double *nu_lo, *nu_up, *dnu_lo, *dnu_up, *rho, *p, *mu_lo, *mu_up, *q_lo, *q_up, *lower, *upper;
  // device-resident Newton step: alpha, kappa and dalpha from device memory (the trial
  // alpha + kappa dalpha then formed here, in pbm.py:301's two roundings); skip: the
  // line search has decided
  const double *alpha_dev = nullptr, *kappa_dev = nullptr, *dalpha_dev = nullptr;
  const int* skip = nullptr;
};

VTS_DEVICE_INLINE double trial_alpha(double alpha, double kappa, double dalpha) {
  return __dadd_rn(alpha, __dmul_rn(kappa, dalpha));
}

__global__ void __launch_bounds__(kThreads) k_al_elem(AlElemArgs A, double* partials, unsigned* flags) {
  if (A.skip && *A.skip) return;
  __shared__ double scratch[5 * kThreads / 32];
  double acc[5] = {0, 0, 0, 0, 0};
  unsigned sat = 0;
  if (A.kappa_dev) {
    A.kappa = *A.kappa_dev;
    A.alpha = trial_alpha(*A.alpha_dev, A.kappa, *A.dalpha_dev);
  }
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < A.m; e += gridDim.x * blockDim.x) {
    int nd[4];
    elem_nodes(e, A.ex, A.nx, nd);
    double ue[8], w[8];
    gather8(A.ug, nd, ue);
    ke_times(ue, w);
    double qq = w[0] * ue[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) qq = fma(w[i], ue[i], qq);
    qq = 0.5 * qq;
    const double nlo = __dadd_rn(A.nu_lo[e], __dmul_rn(A.kappa, A.dnu_lo[e]));
    const double nup = __dadd_rn(A.nu_up[e], __dmul_rn(A.kappa, A.dnu_up[e]));
    const double pe = A.p[e], qlo = A.q_lo[e], qup = A.q_up[e];
    const double s = __dsub_rn(__dadd_rn(__dsub_rn(qq, A.alpha), nlo), nup);
    const PhiOut f1 = phi_eval(s / pe, A.branch, &sat);
    const PhiOut f2 = phi_eval(-nlo / qlo, A.branch, &sat);
    const PhiOut f3 = phi_eval(-nup / qup, A.branch, &sat);
    acc[0] += A.rho[e] * __dmul_rn(pe, f1.v);
    acc[1] += A.mu_lo[e] * __dmul_rn(qlo, f2.v);
    acc[2] += A.mu_up[e] * __dmul_rn(qup, f3.v);
    acc[3] = fma(A.lower[e], nlo, acc[3]);
    acc[4] = fma(A.upper[e], nup, acc[4]);
  }
  if (sat) atomicOr(flags, 1u);
  block_partials<5>(acc, scratch, partials);
}

__global__ void k_al_finish(int nb, const double* __restrict__ pe, const double* __restrict__ fu_ptr,
                            double alpha, double volume, double* out, const double* alpha_dev = nullptr,
                            const double* kappa_dev = nullptr, const double* dalpha_dev = nullptr,
                            const int* skip = nullptr) {
  if (skip && *skip) return;
  if (kappa_dev) alpha = trial_alpha(*alpha_dev, *kappa_dev, *dalpha_dev);
  __shared__ double scratch[5 * kThreads / 32];
  double t[5] = {0, 0, 0, 0, 0};
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    for (int i = 0; i < 5; ++i) t[i] += pe[b * 5 + i];
  block_sum<5>(t, scratch);
  if (threadIdx.x == 0) {
    const double dual = ((alpha * volume - *fu_ptr) - t[3]) + t[4];
    out[0] = ((dual + t[0]) + t[1]) + t[2];
  }
}

// ---------------------------------------------------------------------------
// outer loop pieces
// ---------------------------------------------------------------------------
VTS_DEVICE_INLINE double clip_ref(double v, double lo, double hi) { return fmin(fmax(v, lo), hi); }

__global__ void k_outer_update(int m, double beta, double gamma, double floor_p,
                               const double* __restrict__ rho_hat, const double* __restrict__ mhl,
                               const double* __restrict__ mhu, double* rho, double* mu_lo,
                               double* mu_up, double* p, double* q_lo, double* q_up, int pen) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    if (rho_hat) {
      const double r = rho[e];
      rho[e] = clip_ref(rho_hat[e], beta * r, r / beta);
      if (mhl) {
        const double a = mu_lo[e], b = mu_up[e];
        mu_lo[e] = clip_ref(mhl[e], beta * a, a / beta);
        mu_up[e] = clip_ref(mhu[e], beta * b, b / beta);
      }
    }
    if (pen) {
      p[e] = fmax(gamma * p[e], floor_p);
      q_lo[e] = fmax(gamma * q_lo[e], floor_p);
      q_up[e] = fmax(gamma * q_up[e], floor_p);
    }
  }
}

__global__ void __launch_bounds__(kThreads) k_gap_elem(int m, double alpha, const double* __restrict__ q,
                                                     const double* __restrict__ nu_lo,
                                                     const double* __restrict__ nu_up,
                                                     const double* __restrict__ lower,
                                                     const double* __restrict__ upper,
                                                     const double* __restrict__ rho, double* partials) {
  __shared__ double scratch[4 * kThreads / 32];
  double acc[4] = {0, 0, 0, 0};
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    const double slack = __dsub_rn(alpha, q[e]);
    const double lo = lower[e], up = upper[e];
    acc[0] += fmin(__dmul_rn(lo, slack), __dmul_rn(up, slack));
    acc[1] = fma(lo, nu_lo[e], acc[1]);
    acc[2] = fma(up, nu_up[e], acc[2]);
    acc[3] += rho ? rho[e] : 0.0;
  }
  block_partials<4>(acc, scratch, partials);
}

__global__ void k_gap_finish(int nb, const double* __restrict__ pe, const double* __restrict__ fu_ptr,
                             double alpha, double volume, double* out) {
  __shared__ double scratch[4 * kThreads / 32];
  double t[4] = {0, 0, 0, 0};
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    for (int i = 0; i < 4; ++i) t[i] += pe[b * 4 + i];
  block_sum<4>(t, scratch);
  if (threadIdx.x == 0) {
    const double fu = *fu_ptr;
    out[0] = ((alpha * volume - fu) - t[1]) + t[2];    // dual_objective (model.py:61-66)
    out[1] = (-0.5 * fu + alpha * volume) - t[0];       // duality_gap (model.py:77-79)
    out[2] = fu;
    out[3] = t[3];
  }
}

// ---------------------------------------------------------------------------
// host wrappers
// ---------------------------------------------------------------------------
// border-slot mode of an API vector of the bound system (k_free_to_grid / k_grid_to_free)
static int border_mode(const Ctx* c, bool bordered) {
  if (!bordered) return 0;
  if (c->unbordered) return 2;
  return c->border_flip ? -1 : 1;
}

static int reduce_grid(long long work) {
  return (int)std::min<long long>(std::max<long long>(1, (work + kThreads - 1) / kThreads), kReduceGridCap);
}

static int sync_scalars(Ctx* c, int count) {
  VTS_CUDA(cudaMemcpyAsync(c->hscal, c->dscal, sizeof(double) * count, cudaMemcpyDeviceToHost, c->stream));
  VTS_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

// VTS_PHI_SPLIT=1: the evaluation as k_phi_elem + k_phi_node + k_phi_finish (A/B checks)
static bool phi_fused() {
  static const bool on = [] {
    const char* e = getenv("VTS_PHI_SPLIT");
    return !(e && e[0] == '1');
  }();
  return on;
}

int free_to_grid(Ctx* c, int level, const double* src, double* dst, bool bordered, const int* skip) {
  const LevelBuf& L = c->lv[level];
  const int total = L.d.ngrid + 1;
  k_free_to_grid<<<div_up(total, kThreads), kThreads, 0, c->stream>>>(L.d.ngrid, L.d.nfree, L.grid2free,
                                                                      src, dst, border_mode(c, bordered), skip);
  VTS_LAUNCHED(c);
  return 0;
}

int grid_to_free(Ctx* c, int level, const double* src, double* dst, bool bordered) {
  const LevelBuf& L = c->lv[level];
  const int total = L.d.nfree + 1;
  k_grid_to_free<<<div_up(total, kThreads), kThreads, 0, c->stream>>>(L.d.nfree, L.d.ngrid, L.d.free2grid,
                                                                      src, dst, border_mode(c, bordered));
  VTS_LAUNCHED(c);
  return 0;
}

int dot_grid(Ctx* c, int level, const double* a, const double* b, bool bordered, double* dst,
             const int* skip) {
  const long long len = c->lv[level].d.ngrid + (bordered ? 1 : 0);
  k_dot<<<reduce_grid(len), kThreads, 0, c->stream>>>(len, a, b, c->partials, c->counters + 0, dst, skip);
  VTS_LAUNCHED(c);
  return 0;
}

// alpha_dev != null (device-resident Newton step, step.inc.cu): alpha is read from
// device memory, nothing is read back (the eight scalars stay in dscal[0..7], the
// saturation bit accumulates in dflags) and the stream is not synchronised
int eval_lagrangian(Ctx* c, const double* u, double alpha, const double* nu_lo, const double* nu_up,
                    const double* rho, const double* mu_lo, const double* mu_up, const double* p,
                    const double* q_lo, const double* q_up, const double* f, const double* lower,
                    const double* upper, double volume, double norm_f, double norm_bounds,
                    double branch, double* res_u, double* res_lo, double* res_up, double* q,
                    double* mu_hat_lo, double* mu_hat_up, double* a, double* b_lo, double* b_up,
                    double* rho_hat, double* w_out, double* scalars, unsigned* warn, const double* alpha_dev,
                    const int* skip) {
  const int F = c->L - 1;
  const LevelDev& d = c->lv[F].d;
  double* ug = c->fvec[0];
  if (int rc = free_to_grid(c, F, u, ug, false, skip)) return rc;
  if (!alpha_dev) VTS_CUDA(cudaMemsetAsync(c->dflags, 0, sizeof(unsigned), c->stream));
  PhiElemArgs A{c->m, d.ex, d.nx, ug, alpha, branch, nu_lo, nu_up, rho, mu_lo, mu_up, p, q_lo,
                q_up, lower, upper, q, rho_hat, mu_hat_lo, mu_hat_up, a, b_lo, b_up, res_lo,
                res_up, w_out, alpha_dev, skip};
  const int tiles_x = div_up(d.nx, kPhiTX - 1), tiles = tiles_x * div_up(d.ny, kPhiTY - 1);
  // one tile per CTA; the last-block reduction holds 9 partials per CTA
  if (phi_fused() && (long long)tiles * 9 <= (long long)kMaxBlocks * kMaxPartials) {
    PhiTileArgs T{d.nx, d.ny, d.ey, tiles_x, tiles, f, c->lv[F].grid2free, res_u, volume, norm_f, norm_bounds,
                  c->dscal};
    k_phi_tile<<<tiles, kPhiTX * kPhiTY, 0, c->stream>>>(A, T, c->partials, c->counters + 15, c->dflags);
    VTS_LAUNCHED(c);
    if (alpha_dev) return 0;
    VTS_CUDA(cudaMemcpyAsync(c->hscal + 16, c->dflags, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
    if (int rc = sync_scalars(c, 8)) return rc;
    for (int i = 0; i < 8; ++i) scalars[i] = c->hscal[i];
    if (warn) *warn = *reinterpret_cast<unsigned*>(c->hscal + 16) ? 1u : 0u;
    return 0;
  }
  const int ge = reduce_grid(c->m);
  k_phi_elem<<<ge, kThreads, 0, c->stream>>>(A, c->partials, c->dflags);
  VTS_LAUNCHED(c);
  const int gn = reduce_grid(d.nnodes);
  double* pn = c->partials + kMaxBlocks * 8;
  k_phi_node<<<gn, kThreads, 0, c->stream>>>(d.nnodes, d.nx, d.ex, d.ey, ug, rho_hat, f, c->lv[F].grid2free,
                                              res_u, pn, skip);
  VTS_LAUNCHED(c);
  k_phi_finish<<<1, kThreads, 0, c->stream>>>(ge, c->partials, gn, pn, alpha, volume, norm_f, norm_bounds,
                                               c->dscal, alpha_dev, skip);
  VTS_LAUNCHED(c);
  if (alpha_dev) return 0;
  VTS_CUDA(cudaMemcpyAsync(c->hscal + 16, c->dflags, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
  if (int rc = sync_scalars(c, 8)) return rc;
  for (int i = 0; i < 8; ++i) scalars[i] = c->hscal[i];
  if (warn) *warn = *reinterpret_cast<unsigned*>(c->hscal + 16) ? 1u : 0u;
  return 0;
}

// res_alpha_dev != null (device-resident Newton step): res_alpha from device memory,
// no read-back of the corner (it stays in d_corner) and no synchronisation
int schur_system(Ctx* c, const double* u, const double* res_u, double res_alpha,
                 const double* res_lo, const double* res_up, const double* a, const double* b_lo,
                 const double* b_up, const double* rho_hat, double* chat, double* rhs,
                 double* border, double* corner, const double* res_alpha_dev) {
  const int F = c->L - 1;
  const LevelDev& d = c->lv[F].d;
  if (int rc = free_to_grid(c, F, u, c->u_grid, false)) return rc;
  double* tcoef = c->fvec[1];  // m <= ngrid, scratch
  const int ge = reduce_grid(c->m);
  k_schur_elem<<<ge, kThreads, 0, c->stream>>>(c->m, a, b_lo, b_up, res_lo, res_up, rho_hat, chat, c->chat,
                                                c->rho_hat, tcoef, c->partials);
  VTS_LAUNCHED(c);
  k_schur_node<<<reduce_grid(d.nnodes), kThreads, 0, c->stream>>>(d.nnodes, d.nx, d.ex, d.ey, c->u_grid,
                                                                   tcoef, c->chat, res_u, c->lv[F].grid2free,
                                                                   rhs, border, c->lv[F].d.border);
  VTS_LAUNCHED(c);
  k_schur_finish<<<1, kThreads, 0, c->stream>>>(ge, c->partials, res_alpha, 1.0, c->n, rhs, c->d_corner, c->dscal,
                                                res_alpha_dev);
  VTS_LAUNCHED(c);
  if (!res_alpha_dev) {
    if (int rc = sync_scalars(c, 2)) return rc;
    c->corner = c->hscal[0];
    if (corner) *corner = c->corner;
  }
  c->system_bound = true;
  c->border_flip = false;
  c->unbordered = false;
  c->mg_ready = false;
  return 0;
}

int reconstruct_nu(Ctx* c, const double* u, const double* du, double dalpha, const double* res_u,
                   double res_alpha, const double* res_lo, const double* res_up, const double* a,
                   const double* b_lo, const double* b_up, double* dnu_lo, double* dnu_up,
                   double* slope) {
  const int F = c->L - 1;
  const LevelDev& d = c->lv[F].d;
  double* ug = c->fvec[0];
  double* dug = c->fvec[2];
  if (int rc = free_to_grid(c, F, u, ug, false)) return rc;
  if (int rc = free_to_grid(c, F, du, dug, false)) return rc;
  const int ge = reduce_grid(c->m);
  k_recon_elem<<<ge, kThreads, 0, c->stream>>>(c->m, d.ex, d.nx, ug, dug, dalpha, res_lo, res_up, a, b_lo,
                                                b_up, dnu_lo, dnu_up, c->partials);
  VTS_LAUNCHED(c);
  k_dot<<<reduce_grid(c->n), kThreads, 0, c->stream>>>(c->n, res_u, du, c->partials + kMaxBlocks * 8,
                                                        c->counters + 1, c->dscal + 8, nullptr);
  VTS_LAUNCHED(c);
  if (slope) {
    k_slope_finish<<<1, 1, 0, c->stream>>>(ge, c->partials, c->dscal + 8, res_alpha, dalpha, c->dscal + 9);
    VTS_LAUNCHED(c);
    if (int rc = sync_scalars(c, 10)) return rc;
    *slope = c->hscal[9];
  }
  return 0;
}

int al_value(Ctx* c, const double* u, double alpha, const double* nu_lo, const double* nu_up,
             const double* du, double dalpha, const double* dnu_lo, const double* dnu_up,
             double kappa, const double* rho, const double* p, const double* mu_lo,
             const double* mu_up, const double* q_lo, const double* q_up, const double* f,
             const double* lower, const double* upper, double volume, double branch,
             double* value, unsigned* warn) {
  const int F = c->L - 1;
  const LevelDev& d = c->lv[F].d;
  double* ug = c->fvec[0];
  k_trial_grid<<<reduce_grid(d.ngrid), kThreads, 0, c->stream>>>(d.ngrid, c->lv[F].grid2free, u, du, kappa, f, ug,
                                                                  c->partials + kMaxBlocks * 8, c->counters + 2,
                                                                  c->dscal + 10);
  VTS_LAUNCHED(c);
  VTS_CUDA(cudaMemsetAsync(c->dflags, 0, sizeof(unsigned), c->stream));
  volatile double kd = kappa * dalpha;  // state.alpha + kappa * dalpha, two roundings (pbm.py:301)
  const double alpha_t = alpha + kd;
  AlElemArgs A{c->m, d.ex, d.nx, ug, alpha_t, kappa, branch, nu_lo, nu_up, dnu_lo, dnu_up, rho, p,
               mu_lo, mu_up, q_lo, q_up, lower, upper};
  const int ge = reduce_grid(c->m);
  k_al_elem<<<ge, kThreads, 0, c->stream>>>(A, c->partials, c->dflags);
  VTS_LAUNCHED(c);
  k_al_finish<<<1, kThreads, 0, c->stream>>>(ge, c->partials, c->dscal + 10, alpha_t, volume, c->dscal);
  VTS_LAUNCHED(c);
  VTS_CUDA(cudaMemcpyAsync(c->hscal + 16, c->dflags, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
  if (int rc = sync_scalars(c, 1)) return rc;
  *value = c->hscal[0];
  if (warn) *warn = *reinterpret_cast<unsigned*>(c->hscal + 16) ? 1u : 0u;
  return 0;
}

int axpy(Ctx* c, long long len, double kappa, const double* dx, double* x) {
  k_axpy<<<reduce_grid(len), kThreads, 0, c->stream>>>(len, kappa, dx, x);
  VTS_LAUNCHED(c);
  return 0;
}

int outer_update(Ctx* c, double beta, double gamma, double floor_p, const double* rho_hat,
                 const double* mu_hat_lo, const double* mu_hat_up, double* rho, double* mu_lo,
                 double* mu_up, double* p, double* q_lo, double* q_up, int update_penalties) {
  k_outer_update<<<reduce_grid(c->m), kThreads, 0, c->stream>>>(c->m, beta, gamma, floor_p, rho_hat, mu_hat_lo,
                                                                mu_hat_up, rho, mu_lo, mu_up, p, q_lo, q_up,
                                                                update_penalties);
  VTS_LAUNCHED(c);
  return 0;
}

int gap(Ctx* c, const double* u, double alpha, const double* q, const double* f,
        const double* nu_lo, const double* nu_up, const double* lower, const double* upper,
        double volume, const double* rho, double* d_val, double* gap_out, double* fu, double* rho_sum) {
  k_dot<<<reduce_grid(c->n), kThreads, 0, c->stream>>>(c->n, f, u, c->partials + kMaxBlocks * 8,
                                                        c->counters + 3, c->dscal + 12, nullptr);
  VTS_LAUNCHED(c);
  const int ge = reduce_grid(c->m);
  k_gap_elem<<<ge, kThreads, 0, c->stream>>>(c->m, alpha, q, nu_lo, nu_up, lower, upper, rho, c->partials);
  VTS_LAUNCHED(c);
  k_gap_finish<<<1, kThreads, 0, c->stream>>>(ge, c->partials, c->dscal + 12, alpha, volume, c->dscal);
  VTS_LAUNCHED(c);
  if (int rc = sync_scalars(c, 4)) return rc;
  if (d_val) *d_val = c->hscal[0];
  if (gap_out) *gap_out = c->hscal[1];
  if (fu) *fu = c->hscal[2];
  if (rho_sum) *rho_sum = c->hscal[3];
  return 0;
}

}  // namespace vts

namespace vts {

// phi, phi', phi'' of a vector (PenaltyBarrier.value/deriv/deriv2, penalty.py:49-82)
__global__ void k_penalty_eval(long long n, const double* __restrict__ tau, double branch, double* v, double* d1,
                               double* d2, unsigned* flags) {
  unsigned sat = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const PhiOut o = phi_eval(tau[i], branch, &sat);
    if (v) v[i] = o.v;
    if (d1) d1[i] = o.d1;
    if (d2) d2[i] = o.d2;
  }
  if (sat) atomicOr(flags, 1u);
}

int penalty_eval(Ctx* c, long long n, const double* tau, double branch, double* v, double* d1, double* d2,
                 unsigned* warn) {
  VTS_CUDA(cudaMemsetAsync(c->dflags, 0, sizeof(unsigned), c->stream));
  k_penalty_eval<<<reduce_grid(n), kThreads, 0, c->stream>>>(n, tau, branch, v, d1, d2, c->dflags);
  VTS_LAUNCHED(c);
  unsigned h = 0;
  VTS_CUDA(cudaMemcpyAsync(c->hscal + 16, c->dflags, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
  VTS_CUDA(cudaStreamSynchronize(c->stream));
  h = *reinterpret_cast<unsigned*>(c->hscal + 16);
  if (warn) *warn = h ? 1u : 0u;
  return 0;
}

}  // namespace vts
