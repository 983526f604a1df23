// Newton-matrix and level-operator applies (unity-built into vts_b200.cu).
//
// k_newton_apply: matrix-free y = S x for the bordered Schur matrix
//   S = [[sum_e rho_hat_e K_e + sum_e chat_e w_e w_e^T, -sum_e chat_e w_e],
//        [.^T, sum_e chat_e]],  w_e = K_e u_e
// i.e. BorderedMatrix.matvec (linalg.py:56-62) of ElementOps.assemble
// (fem.py:188-209) without ever forming the CSR matrix.  One CTA (32 x 8
// threads) owns a 31 x 7 tile of nodes: it stages x and u of the (33 x 9)-node
// halo in shared memory, computes the 32 x 8 touching elements, one per thread
// (w_e, theta_e = w_e.x_e - x_alpha, K_e x_e, the 8-vector
// rho_hat K_e x_e + chat theta w_e), then every owning thread gathers its
// node's four element contributions in the reference's scatter order.  No
// atomics; y_alpha = -sum chat_e theta_e is a deterministic last-block
// reduction over the elements each tile owns.
//
// k_level_apply: y = A_k x + border x_alpha, y_alpha = border.x + corner x_alpha
// on a stored 9-point block stencil (the residual of multigrid.py:125 and the
// parity probe of MgPreconditioner.mats[k].matvec).

namespace vts {

constexpr int kBX = 32, kBY = 8;            // threads = touching elements
constexpr int kTX = kBX - 1, kTY = kBY - 1;  // owned nodes
constexpr int kHX = kTX + 2, kHY = kTY + 2;  // halo nodes (33 x 9)
constexpr int kEX = kBX, kEY = kBY;
constexpr int kES = kEX * kEY;               // elements per tile
#ifndef VTS_APPLY_STAGES
#define VTS_APPLY_STAGES 2
#endif
constexpr int kApplyStages = VTS_APPLY_STAGES;  // halo boxes in flight per CTA
#ifndef VTS_APPLY_MINB
#define VTS_APPLY_MINB 3
#endif

// TMA boxes of the tile's halo nodes (x, u).  The element arrays are read
// directly: a 2-D box starting at element column x0 - 1 has an inner start
// offset that is not 16-B aligned, which TMA rejects for negative starts.
struct __align__(128) ApplyStage {
  double2 xs[kHY * kHX];
  double pad0[(128 - (kHY * kHX * 16) % 128) / 8];
  double2 us[kHY * kHX];
};
struct ApplySmem {
  ApplyStage st[kApplyStages];
  double contrib[8 * kES];  // structure of arrays: conflict-free
  unsigned long long full[kApplyStages];
  double scratch[kES / 32];
};
static_assert(offsetof(ApplyStage, us) % 128 == 0, "TMA alignment");
constexpr unsigned kApplyTxBytes = 2 * kHY * kHX * 16;

// Element phase of one tile (thread = element): contrib = rho_hat K_e x_e +
// chat theta w_e with w_e = K_e u_e, theta = w_e.x_e - x_alpha; returns theta.
// `ke` is c_ke offset by an opaque zero produced inside the tile loop: NVVM
// would otherwise hoist the 64 loop-invariant K_e loads into registers (and
// spill); ptxas still folds them into constant-bank operands.
VTS_DEVICE_INLINE double apply_element(const ApplyStage& G, double* contrib, int tid, int h0, double xa, double rh,
                                       double ch, const double* __restrict__ ke) {
  const int hn[4] = {h0, h0 + 1, h0 + kHX + 1, h0 + kHX};
  double w[8], kx[8], xe[8];
  {
    double ue[8];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const double2 uv = G.us[hn[a]];
      ue[2 * a] = uv.x;
      ue[2 * a + 1] = uv.y;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double sw = ue[0] * ke[j];
#pragma unroll
      for (int i = 1; i < 8; ++i) sw = fma(ue[i], ke[i * 8 + j], sw);
      w[j] = sw;
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const double2 xv = G.xs[hn[a]];
    xe[2 * a] = xv.x;
    xe[2 * a + 1] = xv.y;
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    double sk = xe[0] * ke[j];
#pragma unroll
    for (int i = 1; i < 8; ++i) sk = fma(xe[i], ke[i * 8 + j], sk);
    kx[j] = sk;
  }
  double wx = w[0] * xe[0];
#pragma unroll
  for (int i = 1; i < 8; ++i) wx = fma(w[i], xe[i], wx);
  const double theta = wx - xa;
  const double ct = ch * theta;
#pragma unroll
  for (int j = 0; j < 8; ++j) contrib[j * kES + tid] = fma(ct, w[j], rh * kx[j]);
  return theta;
}

// The same element phase in the corner-mode basis (modal_form, vts_b200.cu):
// u~ = T^T u_e and x~ = T^T x_e by differences, w~ = K' u~ (K' = T^T K_e T / 16,
// 8 coefficients), theta = w~ . x~ - x_alpha (= w_e . x_e - x_alpha since
// w_e = T w~), and contrib = K_e (rho_hat x_e + chat theta u_e) = T K' z~ with
// z~ = rho_hat x~ + chat theta u~ -- one modal product instead of two dense ones.
struct Modes {
  double xi_x, eta_x, h_x, xi_y, eta_y, h_y;
};
VTS_DEVICE_INLINE Modes to_modes(const double2 (&v)[4]) {
  Modes m;
  {
    const double d10 = v[1].x - v[0].x, d23 = v[2].x - v[3].x, d30 = v[3].x - v[0].x, d21 = v[2].x - v[1].x;
    m.xi_x = d10 + d23;
    m.eta_x = d30 + d21;
    m.h_x = d21 - d30;
  }
  {
    const double d10 = v[1].y - v[0].y, d23 = v[2].y - v[3].y, d30 = v[3].y - v[0].y, d21 = v[2].y - v[1].y;
    m.xi_y = d10 + d23;
    m.eta_y = d30 + d21;
    m.h_y = d21 - d30;
  }
  return m;
}
VTS_DEVICE_INLINE Modes modal_k(const Modes& a, const double* __restrict__ km) {
  Modes y;
  y.xi_x = fma(km[2], a.eta_y, km[0] * a.xi_x);
  y.eta_y = fma(km[2], a.xi_x, km[1] * a.eta_y);
  y.xi_y = fma(km[5], a.eta_x, km[3] * a.xi_y);
  y.eta_x = fma(km[5], a.xi_y, km[4] * a.eta_x);
  y.h_x = km[6] * a.h_x;
  y.h_y = km[7] * a.h_y;
  return y;
}
VTS_DEVICE_INLINE double apply_element_modal(const ApplyStage& G, double* contrib, int tid, int h0, double xa,
                                             double rh, double ch, const double* __restrict__ km) {
  const int hn[4] = {h0, h0 + 1, h0 + kHX + 1, h0 + kHX};
  double2 uv[4], xv[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    uv[a] = G.us[hn[a]];
    xv[a] = G.xs[hn[a]];
  }
  const Modes ut = to_modes(uv), xt = to_modes(xv);
  const Modes wt = modal_k(ut, km);
  double wx = wt.xi_x * xt.xi_x;
  wx = fma(wt.eta_x, xt.eta_x, wx);
  wx = fma(wt.h_x, xt.h_x, wx);
  wx = fma(wt.xi_y, xt.xi_y, wx);
  wx = fma(wt.eta_y, xt.eta_y, wx);
  wx = fma(wt.h_y, xt.h_y, wx);
  const double theta = wx - xa;
  const double ct = ch * theta;
  Modes z;
  z.xi_x = fma(ct, ut.xi_x, rh * xt.xi_x);
  z.eta_x = fma(ct, ut.eta_x, rh * xt.eta_x);
  z.h_x = fma(ct, ut.h_x, rh * xt.h_x);
  z.xi_y = fma(ct, ut.xi_y, rh * xt.xi_y);
  z.eta_y = fma(ct, ut.eta_y, rh * xt.eta_y);
  z.h_y = fma(ct, ut.h_y, rh * xt.h_y);
  const Modes y = modal_k(z, km);
  // back to the corners: node (sign of xi, eta, h) = 0 (-,-,+), 1 (+,-,-), 2 (+,+,+), 3 (-,+,-)
  {
    const double a = y.xi_x + y.eta_x, b = y.xi_x - y.eta_x;
    contrib[0 * kES + tid] = y.h_x - a;
    contrib[2 * kES + tid] = b - y.h_x;
    contrib[4 * kES + tid] = a + y.h_x;
    contrib[6 * kES + tid] = -b - y.h_x;
  }
  {
    const double a = y.xi_y + y.eta_y, b = y.xi_y - y.eta_y;
    contrib[1 * kES + tid] = y.h_y - a;
    contrib[3 * kES + tid] = b - y.h_y;
    contrib[5 * kES + tid] = a + y.h_y;
    contrib[7 * kES + tid] = -b - y.h_y;
  }
  return theta;
}

// Persistent: CTA b takes tiles b, b + grid, ...; the halo boxes (TMA, OOB
// zero fill) and element coefficients of the next tile are in flight while
// the current tile computes (2 stages).
template <bool MODAL>
__global__ void __launch_bounds__(kBX* kBY, VTS_APPLY_MINB) k_newton_apply(const __grid_constant__ CUtensorMap mapX,
                                                             const __grid_constant__ CUtensorMap mapU,
                                                             const double* __restrict__ rho_hat,
                                                             const double* __restrict__ chat, int nx, int ny,
                                                             int ex, int ey, int ngrid, int tiles_x, int ntiles,
                                                             const uint8_t* __restrict__ fmask,
                                                             const double* __restrict__ x, double* __restrict__ y,
                                                             double* partials, unsigned* counter, const int* skip) {
  pdl_enter();
  if (skip && *skip) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  ApplySmem& S = *reinterpret_cast<ApplySmem*>(smem_raw);
  const int tid = threadIdx.x;
  const int lx = tid % kEX, ly = tid / kEX;
  const int h0 = lx + kHX * ly;
  auto issue = [&](int t, int s) {
    const int x0 = (t % tiles_x) * kTX, y0 = (t / tiles_x) * kTY;
    mbar_expect_tx(&S.full[s], kApplyTxBytes);
    tma_load_3d(S.st[s].xs, &mapX, 0, x0 - 1, y0 - 1, &S.full[s]);
    tma_load_3d(S.st[s].us, &mapU, 0, x0 - 1, y0 - 1, &S.full[s]);
  };
  auto coeffs = [&](int t, double& rh, double& ch) {
    const int gx = (t % tiles_x) * kTX - 1 + lx, gy = (t / tiles_x) * kTY - 1 + ly;
    rh = 0.0;
    ch = 0.0;
    if (t < ntiles && gx >= 0 && gx < ex && gy >= 0 && gy < ey) {
      rh = rho_hat[gx + ex * gy];
      ch = chat[gx + ex * gy];
    }
  };
  if (tid == 0) {
    for (int i = 0; i < kApplyStages; ++i) mbar_init(&S.full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < kApplyStages; ++i)
      if ((int)blockIdx.x + i * (int)gridDim.x < ntiles) issue(blockIdx.x + i * gridDim.x, i);
  }
  const double xa = x[ngrid];
  double rh, ch;
  coeffs(blockIdx.x, rh, ch);
  __syncthreads();

  double acc = 0.0;
  int k = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    const int s = k % kApplyStages;
    const int x0 = (t % tiles_x) * kTX, y0 = (t / tiles_x) * kTY;
    double rh_n, ch_n;
    coeffs(t + gridDim.x, rh_n, ch_n);  // next tile's coefficients, in flight during this one
    mbar_wait(&S.full[s], (k / kApplyStages) & 1);
    int z;
    asm volatile("mov.u32 %0, 0;" : "=r"(z));
    double* contrib = S.contrib;
    const double theta = MODAL ? apply_element_modal(S.st[s], contrib, tid, h0, xa, rh, ch, c_modal + z)
                               : apply_element(S.st[s], contrib, tid, h0, xa, rh, ch, c_ke + z);
    // y_alpha sums the elements this tile owns (ch = 0 outside the mesh)
    {
      const int gx = x0 - 1 + lx, gy = y0 - 1 + ly;
      if (gx >= x0 && gx < x0 + kTX && gy >= y0 && gy < y0 + kTY) acc = fma(ch, theta, acc);
    }
    rh = rh_n;
    ch = ch_n;
    __syncthreads();  // stage s consumed, contrib complete
    if (tid == 0 && t + kApplyStages * (int)gridDim.x < ntiles) issue(t + kApplyStages * gridDim.x, s);
    const int ix = x0 + lx, iy = y0 + ly;
    if (lx < kTX && ly < kTY && ix < nx && iy < ny) {
      // elements (ix-1,iy-1) c2, (ix,iy-1) c3, (ix-1,iy) c1, (ix,iy) c0: the reference's scatter order
      double s0 = 0.0, s1 = 0.0;
      if (ix >= 1 && iy >= 1) {
        const double* cb = contrib + (lx + kEX * ly);
        s0 += cb[4 * kES]; s1 += cb[5 * kES];
      }
      if (ix < ex && iy >= 1) {
        const double* cb = contrib + (lx + 1 + kEX * ly);
        s0 += cb[6 * kES]; s1 += cb[7 * kES];
      }
      if (ix >= 1 && iy < ey) {
        const double* cb = contrib + (lx + kEX * (ly + 1));
        s0 += cb[2 * kES]; s1 += cb[3 * kES];
      }
      if (ix < ex && iy < ey) {
        const double* cb = contrib + (lx + 1 + kEX * (ly + 1));
        s0 += cb[0]; s1 += cb[kES];
      }
      const int nd = ix + nx * iy;
      const uchar2 fm = *reinterpret_cast<const uchar2*>(fmask + 2 * nd);
      *reinterpret_cast<double2*>(y + 2 * nd) = make_double2(fm.x ? s0 : 0.0, fm.y ? s1 : 0.0);
    }
    __syncthreads();  // contrib reused by the next tile
  }
  double a1[1] = {acc}, tot[1];
  if (last_block_reduce<1>(a1, S.scratch, partials, counter, tot) && tid == 0) y[ngrid] = -tot[0];
}

// y = A_k x (+ border x_alpha) on a block stencil; with `b` given, computes
// r = b - (A x + border x_alpha) instead.  Border dot partials for y_alpha.
// Row sums follow the CSR column order SW S SE W C E NW N NE (linalg.py:58).
// one node of A_k x + border x_alpha (or b - that); also its border.x term
// (CG: x and b through L2 only -- k_residual_restrict_rows reads them while they are written)
template <bool RESIDUAL, bool CG = false>
VTS_DEVICE_INLINE double2 level_apply_node(int nx, int ny, const double* __restrict__ stL,
                                           const double* __restrict__ stU, const double* border, const double* x,
                                           const double* b, double xa, int nd, double& acc) {
  const int ix = nd % nx, iy = nd / nx;
  const double* l = stL + (size_t)nd * kHalf;
  const double* u = stU + (size_t)nd * kHalf;
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int blk = 0; blk < 9; ++blk) {
    const int dx = blk % 3 - 1, dy = blk / 3 - 1;
    const int jx = ix + dx, jy = iy + dy;
    double2 xv = make_double2(0.0, 0.0);
    if (jx >= 0 && jx < nx && jy >= 0 && jy < ny) xv = ld2<CG>(x + 2 * (jx + nx * jy));
    double2 c01, c23;
    if (blk == kBlockCenter) {
      c01 = make_double2(l[kHDiag], u[kHC]);
      c23 = make_double2(l[kHC], u[kHDiag]);
    } else {
      const double* h = (blk < 4 ? l : u) + half_offset(blk);
      c01 = *reinterpret_cast<const double2*>(h);
      c23 = *reinterpret_cast<const double2*>(h + 2);
    }
    s0 = fma(c01.x, xv.x, s0);
    s0 = fma(c01.y, xv.y, s0);
    s1 = fma(c23.x, xv.x, s1);
    s1 = fma(c23.y, xv.y, s1);
  }
  const double2 bd = *reinterpret_cast<const double2*>(border + 2 * nd);
  s0 = fma(bd.x, xa, s0);
  s1 = fma(bd.y, xa, s1);
  const double2 xv = ld2<CG>(x + 2 * nd);
  acc = fma(bd.x, xv.x, acc);
  acc = fma(bd.y, xv.y, acc);
  if (RESIDUAL) {
    const double2 bv = ld2<CG>(b + 2 * nd);
    s0 = bv.x - s0;
    s1 = bv.y - s1;
  }
  return make_double2(s0, s1);
}

// y = A_k x (+ border x_alpha) on a block stencil; with `b` given, computes
// r = b - (A x + border x_alpha) instead.  Border dot partials for y_alpha.
// Row sums follow the CSR column order SW S SE W C E NW N NE (linalg.py:58).
template <bool RESIDUAL>
__global__ void __launch_bounds__(256) k_level_apply(int nx, int ny, int ngrid, const double* __restrict__ stL,
                                                   const double* __restrict__ stU,
                                                   const double* __restrict__ border,
                                                   const double* __restrict__ corner_ptr,
                                                   const double* __restrict__ x,
                                                   const double* __restrict__ b, double* __restrict__ y,
                                                   double* partials, unsigned* counter, const int* skip) {
  pdl_enter();
  if (skip && *skip) return;
  __shared__ double scratch[256 / 32];
  VTS_TL_BEGIN(RESIDUAL ? 6 : 9, nx);
  const int nnodes = nx * ny;
  const double xa = x[ngrid];
  double acc[1] = {0.0};
  for (int nd = blockIdx.x * blockDim.x + threadIdx.x; nd < nnodes; nd += gridDim.x * blockDim.x)
    *reinterpret_cast<double2*>(y + 2 * nd) = level_apply_node<RESIDUAL>(nx, ny, stL, stU, border, x, b, xa, nd, acc[0]);
  double tot[1];
  if (last_block_reduce<1>(acc, scratch, partials, counter, tot) && threadIdx.x == 0) {
    const double ya = fma(*corner_ptr, xa, tot[0]);
    y[ngrid] = RESIDUAL ? b[ngrid] - ya : ya;
  }
}

static bool g_apply_attr_set = false;

// VTS_DENSE_APPLY=1 keeps the dense K_e products even when the modal form exists (A/B checks)
static bool modal_apply_enabled() {
  static const bool on = [] {
    const char* e = getenv("VTS_DENSE_APPLY");
    return !(e && e[0] == '1');
  }();
  return on;
}

int newton_apply_grid(Ctx* c, const double* x, double* y, const int* skip) {
  const LevelBuf& F = c->lv[c->L - 1];
  if (!g_apply_attr_set) {
    VTS_CUDA(cudaFuncSetAttribute(k_newton_apply<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sizeof(ApplySmem)));
    VTS_CUDA(cudaFuncSetAttribute(k_newton_apply<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sizeof(ApplySmem)));
    g_apply_attr_set = true;
  }
  const bool modal = c->modal_ok && modal_apply_enabled();
  const auto kern = modal ? k_newton_apply<true> : k_newton_apply<false>;
  const int tiles_x = div_up(F.d.nx, kTX), tiles_y = div_up(F.d.ny, kTY);
  const int ntiles = tiles_x * tiles_y;
  int dev = 0, sms = 148, per_sm = 2;
  VTS_CUDA(cudaGetDevice(&dev));
  VTS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  VTS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBX * kBY, sizeof(ApplySmem)));
  const int grid = std::max(1, std::min(ntiles, sms * std::max(per_sm, 1)));
  if (grid > kMaxBlocks * 8) {
    set_error(4, "apply grid exceeds the partial buffer");
    return 4;
  }
  CUtensorMap mX, mU;
  const cuuint64_t nd3[3] = {2, (cuuint64_t)F.d.nx, (cuuint64_t)F.d.ny};
  const cuuint64_t ns3[2] = {16, (cuuint64_t)F.d.nx * 16};
  const cuuint32_t nb3[3] = {2, kHX, kHY};
  if (int rc = encode_tiled(&mX, x, 3, nd3, ns3, nb3)) return rc;
  if (int rc = encode_tiled(&mU, c->u_grid, 3, nd3, ns3, nb3)) return rc;
  VTS_CUDA(launch_pdl(kern, dim3(grid), dim3(kBX * kBY), sizeof(ApplySmem), c->stream, 
      mX, mU, c->rho_hat, c->chat, F.d.nx, F.d.ny, F.d.ex, F.d.ey, F.d.ngrid, tiles_x, ntiles, F.d.free_mask, x, y,
      c->partials + kMaxBlocks * 8, c->counters + 4, skip));
  VTS_LAUNCHED(c);
  return 0;
}

int level_apply_grid(Ctx* c, int k, const double* x, double* y, const int* skip) {
  const LevelBuf& L = c->lv[k];
  const int grid = (int)std::min<long long>(div_up(L.d.nnodes, 256), kReduceGridCap);
  VTS_CUDA(launch_pdl(k_level_apply<false>, dim3(grid), dim3(256), 0, c->stream, L.d.nx, L.d.ny, L.d.ngrid, L.d.stL, L.d.stU, L.d.border,
                                                     c->d_corner, x, nullptr, y, c->partials, c->counters + 5,
                                                     skip));
  VTS_LAUNCHED(c);
  return 0;
}

int level_residual_grid(Ctx* c, int k, const double* x, const double* b, double* r, const int* skip) {
  const LevelBuf& L = c->lv[k];
  const int grid = (int)std::min<long long>(div_up(L.d.nnodes, 256), kReduceGridCap);
  VTS_CUDA(launch_pdl(k_level_apply<true>, dim3(grid), dim3(256), 0, c->stream, L.d.nx, L.d.ny, L.d.ngrid, L.d.stL, L.d.stU, L.d.border,
                                                    c->d_corner, x, b, r, c->partials, c->counters + 5, skip));
  VTS_LAUNCHED(c);
  return 0;
}

}  // namespace vts
