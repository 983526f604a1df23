// Fused bottom of the V-cycle (included by mg.inc.cu inside namespace vts).
//
// MgPreconditioner._cycle (multigrid.py:113-143) on the coarse levels 0..kb
// in ONE single-CTA launch: on those levels every sweep is a few dozen
// dependent wavefront steps, and as separate launches each level costs ~60 us
// of fixed launch / barrier-init / TMA-descriptor latency per V-cycle.  Here
// the level vectors live in shared memory, each sweep stages its half-stencil
// into shared memory, the parallel passes (old values, residual, restriction,
// prolongation) use all 512 threads, the wavefront runs on one warp (lane =
// grid row; kb is the largest level with <= 32 node rows), and the coarsest
// bordered system is solved with the Cholesky factor from mg_setup.
//
// Arithmetic is the multi-launch path's, operation for operation
// (gs_old_node, the wavefront step of k_gs_tri, level_apply_node with the
// same fixed reduction tree, restrict_node, prolong_node, k_coarse_solve's
// column order), so the fused and unfused V-cycles agree bit for bit up to
// the sign of zeros.

constexpr int kBotThreads = 512;  // 128 registers: the wavefront warp keeps two steps of operands live
#ifdef VTS_BOT_PROBE
__device__ long long g_bot_probe[64];
__device__ int g_bot_n;
#define BOT_MARK()                                                           \
  do {                                                                       \
    if (threadIdx.x == 0) {                                                  \
      long long t_;                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                 \
      if (g_bot_n < 64) g_bot_probe[g_bot_n++] = t_;                         \
    }                                                                        \
  } while (0)
#else
#define BOT_MARK() \
  do {             \
  } while (0)
#endif
constexpr int kBotMaxLevels = 8;

struct BotLevel {
  int nx, ny, nn, ngrid;
  const uint8_t* fm;
  const double* stL;
  const double* stU;
  const double* border;
  int off_b, off_x, off_r;  // shared-memory offsets (doubles) of b, x, r/P (ngrid + 1 each)
};

struct BotArgs {
  int kb;  // highest fused level (>= 1)
  BotLevel lv[kBotMaxLevels];
  const double* gb;  // level kb right-hand side (global, bordered grid vector)
  double* gx;        // level kb result (global)
  const double* corner;
  // coarsest bordered Cholesky solve (k_coarse_solve)
  int N0, nfree0;
  const int32_t* f2g0;
  const double* chol;
  const double* rdiag;  // reciprocals of the factor's diagonal (div_by)
  int off_chol;  // -1: factor read from global memory
  int off_y;
  int off_stage, off_q;  // staged half-stencil and right-hand side, padded ((nn + 2 kBotPad) nodes)
  int off_red;           // reduction scratch: 32 virtual-block partials + 8 x 32 warp sums
};

// one Gauss-Seidel sweep of level L: x <- sweep(x; b) (zero_guess: x_old = 0)
// (not inlined: one copy of each sweep's code, warm in the instruction cache
// after its first use; inlined copies per call site ran 3.6x slower cold)
constexpr int kBotPad = 64;  // zero nodes before/after the staged level (>= 2 x 31, the largest skew)
template <bool FWD, bool ZERO>
__device__ __noinline__ void bot_sweep(const BotLevel& L, double* sm, const BotArgs& A, bool restage) {
  double* sb = sm + L.off_b;
  double* sx = sm + L.off_x;
  double* stage = sm + A.off_stage;  // [(nn + 2 pad) * kHalf] the half the wavefront solves with
  double* pst = sm + A.off_q;        // [(nn + 2 pad) * 2] its right-hand side P
  const int tid = threadIdx.x;
  const int nn = L.nn;
  const double* solve_half = FWD ? L.stL : L.stU;
  // stage the solve half and P = b - border x_alpha [- U x_old / - L x_old] (the
  // old-value pass, gs_old_node) in padded node order; the pads are zeros
  {
    const double2* src = reinterpret_cast<const double2*>(solve_half);
    double2* dst = reinterpret_cast<double2*>(stage);
    const int lo = kBotPad * kHalf / 2, hi = (kBotPad + nn) * kHalf / 2, end = (2 * kBotPad + nn) * kHalf / 2;
    if (restage)  // the second sweep of a smoothing step solves with the same half: still staged
      for (int i = tid; i < end; i += blockDim.x) dst[i] = (i >= lo && i < hi) ? src[i - lo] : make_double2(0.0, 0.0);
    const double xa = sx[L.ngrid];
    double2* pd = reinterpret_cast<double2*>(pst);
    for (int i = tid; i < nn + 2 * kBotPad; i += blockDim.x) {
      const int nd = i - kBotPad;
      double2 pv = make_double2(0.0, 0.0);
      if (nd >= 0 && nd < nn) {
        if (ZERO) {
          const double2 bb = *reinterpret_cast<const double2*>(sb + 2 * nd);
          const double2 qq = *reinterpret_cast<const double2*>(L.border + 2 * nd);
          pv = make_double2(__dsub_rn(bb.x, __dmul_rn(qq.x, xa)), __dsub_rn(bb.y, __dmul_rn(qq.y, xa)));
        } else {
          pv = gs_old_node<FWD>(L.nx, L.ny, FWD ? L.stU : L.stL, sb, L.border, sx, xa, nd);
        }
      }
      pd[i] = pv;
    }
  }
  __syncthreads();
  BOT_MARK();  // staged
  BOT_MARK();  // (old pass: part of staging)
  if (tid < 32) {
    // the wavefront of k_gs_tri on a single band: lane l = sweep row, skew 2,
    // software-pipelined, branch-free like k_gs_tri: every lane streams its row
    // through the padded stage with a pointer that moves one node per step;
    // positions off the row (and lanes below the grid, clamped to the last row)
    // compute on finite real-neighbour or zero-pad data and are never stored;
    // every coupling that reads them at a valid position is an exact zero
    const int l = tid;
    const int nx = L.nx, ny = L.ny;  // registers: the loop must not re-read L through a generic pointer
    const int lc = l < ny ? l : ny - 1;
    constexpr int d0 = FWD ? 0 : 1;
    constexpr int d1 = 1 - d0;
    constexpr int dir = FWD ? 1 : -1;
    // node of (row lc, sweep column t - 2 l) at t = 0, in padded stage order
    const int n0 = FWD ? lc * nx - 2 * l : (ny - 1 - lc) * nx + nx - 1 + 2 * l;
    const double* ap = stage + (size_t)(kBotPad + n0) * kHalf;
    const double* pp = pst + (size_t)(kBotPad + n0) * 2;
    double* xp_out = sx + 2 * (ptrdiff_t)n0;
    struct StepData {
      double q0, q1, e00, e01, e10, e11, w00, w01, w10, w11, c, r0, r1;
    };
    // gs_pre / gs_rec2 of k_gs_tri's skew-2 steps, so both paths compute the same bits
    auto prepare = [&](const double* a, const double* pv, const double2 xm, const double2 xz) {
      double r[19];
#pragma unroll
      for (int i = 0; i < 9; ++i) {
        const double2 v = reinterpret_cast<const double2*>(a)[i];
        r[2 * i] = v.x;
        r[2 * i + 1] = v.y;
      }
      r[18] = a[18];
      const double2 pq = *reinterpret_cast<const double2*>(pv);
      StepData o;
      gs_pre<d0>(r, pq.x, pq.y, xm, xz, o.q0, o.q1);
      o.e00 = r[8 + 2 * d0];
      o.e01 = r[9 + 2 * d0];
      o.e10 = r[8 + 2 * d1];
      o.e11 = r[9 + 2 * d1];
      o.w00 = r[12 + 2 * d0];
      o.w01 = r[13 + 2 * d0];
      o.w10 = r[12 + 2 * d1];
      o.w11 = r[13 + 2 * d1];
      o.c = r[kHC];
      o.r0 = r[d0 == 0 ? kHRd0 : kHRd1];
      o.r1 = r[d1 == 0 ? kHRd0 : kHRd1];
      return o;
    };
    double2 win[3] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
    double2 wprev = make_double2(0.0, 0.0);
    const int T = nx + 2 * (ny - 1);
    StepData cur = prepare(ap, pp, win[0], win[1]);
    const bool row_ok = l < ny;
    double* const trash = sm + A.off_red;  // stores of off-row positions land here (unused during sweeps)
#pragma unroll 4
    for (int t = 0; t < T; ++t) {
      const int j = t - 2 * l;
      const double2 nv = gs_rec2<d0>(cur.q0, cur.q1, cur.w00, cur.w01, cur.w10, cur.w11, cur.e00, cur.e01, cur.e10,
                                     cur.e11, cur.c, cur.r0, cur.r1, wprev, win[2]);
      // the next step's loads before this step's store (shared memory: the store
      // would otherwise order them behind it)
      const StepData nxt = prepare(ap + (size_t)((t + 1) * dir * kHalf), pp + 2 * dir * (t + 1), win[1], win[2]);
      // branch-free store: off-row positions write the scratch slot instead
      double* dst = (row_ok && j >= 0 && j < nx) ? xp_out + 2 * dir * t : trash;
      *reinterpret_cast<double2*>(dst) = nv;
      wprev = nv;
      double2 up;
      up.x = __shfl_up_sync(0xffffffffu, nv.x, 1);
      up.y = __shfl_up_sync(0xffffffffu, nv.y, 1);
      if (l == 0) up = make_double2(0.0, 0.0);  // a single band: no previous row
      win[0] = win[1];
      win[1] = win[2];
      win[2] = up;
      cur = nxt;
    }
  }
  __syncthreads();
  BOT_MARK();  // wavefront
}

// r = b - (A x + border x_alpha) with k_level_apply<true>'s reduction tree for
// the border row (virtual blocks of 256 threads, last-block sum)
__device__ __noinline__ void bot_residual(const BotLevel& L, double* sm, const BotArgs& A) {
  double* sb = sm + L.off_b;
  double* sx = sm + L.off_x;
  double* sr = sm + L.off_r;
  double* part = sm + A.off_red;         // [32] virtual-block partials
  double* wsum = sm + A.off_red + 32;    // [32 blocks][8 warps]
  const int tid = threadIdx.x, g = tid >> 8, t = tid & 255, w = t >> 5, lane = tid & 31;
  const int nvb = (L.nn + 255) / 256;
  const double xa = sx[L.ngrid];
  for (int vb0 = 0; vb0 < nvb; vb0 += kBotThreads / 256) {
    const int vb = vb0 + g;
    double acc = 0.0;
    if (vb < nvb) {
      const int nd = vb * 256 + t;
      if (nd < L.nn)
        *reinterpret_cast<double2*>(sr + 2 * nd) =
            level_apply_node<true>(L.nx, L.ny, L.stL, L.stU, L.border, sx, sb, xa, nd, acc);
    }
    acc = warp_sum(acc);
    if (lane == 0 && vb < nvb) wsum[vb * 8 + w] = acc;
  }
  __syncthreads();
  if (tid < nvb) {
    double s = 0.0;
    for (int i = 0; i < 8; ++i) s += wsum[tid * 8 + i];
    part[tid] = s;
  }
  __syncthreads();
  if (tid < 32) {
    double v = tid < nvb ? part[tid] : 0.0;
    v = warp_sum(v);
    if (tid == 0) {
      // block_sum's thread 0 adds the 8 warp totals of the finishing block (7 zeros)
      double s = 0.0;
      s += v;
      for (int i = 1; i < 8; ++i) s += 0.0;
      sr[L.ngrid] = sb[L.ngrid] - fma(*A.corner, xa, s);
    }
  }
  __syncthreads();
}

// x0 = chol^-1 b0 (k_coarse_solve's column order)
__device__ void bot_coarse(const BotLevel& C, double* sm, const BotArgs& A) {
  double* sb = sm + C.off_b;
  double* sx = sm + C.off_x;
  double* y = sm + A.off_y;
  const double* Lf = A.off_chol >= 0 ? sm + A.off_chol : A.chol;
  const int N = A.N0, tid = threadIdx.x;
  if (A.off_chol >= 0)
    for (int i = tid; i < N * N; i += blockDim.x) sm[A.off_chol + i] = A.chol[i];
  for (int i = tid; i < N; i += blockDim.x) y[i] = (i < A.nfree0) ? sb[A.f2g0[i]] : sb[C.ngrid];
  __syncthreads();
  BOT_MARK();  // coarse: factor staged, y gathered
  if (N <= 32) {
    // one warp, lane i owns y[i]; same column order and operations as below
    if (tid < 32) {
      // every lane forms the quotient (div_by, as k_coarse_solve), lane j keeps its own
      double yi = tid < N ? y[tid] : 0.0;
      for (int j = 0; j < N; ++j) {
        const double q = div_by(yi, Lf[(size_t)j * N + j], A.rdiag[j]);
        yi = tid == j ? q : yi;
        const double yj = __shfl_sync(0xffffffffu, yi, j);
        const double lij = (tid > j && tid < N) ? Lf[(size_t)tid * N + j] : 0.0;
        yi = (tid > j && tid < N) ? fma(-lij, yj, yi) : yi;
      }
      for (int j = N - 1; j >= 0; --j) {
        const double q = div_by(yi, Lf[(size_t)j * N + j], A.rdiag[j]);
        yi = tid == j ? q : yi;
        const double yj = __shfl_sync(0xffffffffu, yi, j);
        const double lji = tid < j ? Lf[(size_t)j * N + tid] : 0.0;
        yi = tid < j ? fma(-lji, yj, yi) : yi;
      }
      if (tid < N) y[tid] = yi;
    }
    __syncthreads();
    BOT_MARK();  // coarse: both substitutions
  } else {
  for (int j = 0; j < N; ++j) {
    if (tid == 0) y[j] = div_by(y[j], Lf[(size_t)j * N + j], A.rdiag[j]);
    __syncthreads();
    const double yj = y[j];
    for (int i = j + 1 + tid; i < N; i += blockDim.x) y[i] = fma(-Lf[(size_t)i * N + j], yj, y[i]);
    __syncthreads();
  }
  for (int j = N - 1; j >= 0; --j) {
    if (tid == 0) y[j] = div_by(y[j], Lf[(size_t)j * N + j], A.rdiag[j]);
    __syncthreads();
    const double yj = y[j];
    for (int i = tid; i < j; i += blockDim.x) y[i] = fma(-Lf[(size_t)j * N + i], yj, y[i]);
    __syncthreads();
  }
  }
  for (int i = tid; i <= C.ngrid; i += blockDim.x) sx[i] = 0.0;
  __syncthreads();
  for (int i = tid; i < N; i += blockDim.x) {
    if (i < A.nfree0) sx[A.f2g0[i]] = y[i];
    else sx[C.ngrid] = y[i];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kBotThreads, 1) k_vcycle_bottom(const __grid_constant__ BotArgs A, const int* skip) {
  pdl_enter();
  if (skip && *skip) return;
  VTS_TL_BEGIN(4, 5);
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x;
  {
    const BotLevel& T = A.lv[A.kb];
    for (int i = tid; i <= T.ngrid; i += blockDim.x) sm[T.off_b + i] = A.gb[i];
  }
  __syncthreads();
  for (int k = A.kb; k >= 1; --k) {  // descent (multigrid.py:115-131)
    const BotLevel& L = A.lv[k];
    if (tid == 0) sm[L.off_x + L.ngrid] = 0.0;  // k_alpha_init on a coarse level
    __syncthreads();
    bot_sweep<true, true>(L, sm, A, true);
    bot_sweep<true, false>(L, sm, A, false);
    bot_residual(L, sm, A);
    BOT_MARK();  // residual
    const BotLevel& C = A.lv[k - 1];
    for (int cn = tid; cn <= C.nn; cn += blockDim.x) {
      if (cn == C.nn) sm[C.off_b + C.ngrid] = sm[L.off_r + L.ngrid];
      else
        *reinterpret_cast<double2*>(sm + C.off_b + 2 * cn) =
            restrict_node(L.nx, L.ny, L.fm, sm + L.off_r, C.nx, C.fm, cn);
    }
    __syncthreads();
  }
  BOT_MARK();
  bot_coarse(A.lv[0], sm, A);
  BOT_MARK();
  for (int k = 1; k <= A.kb; ++k) {  // ascent (multigrid.py:132-139)
    const BotLevel& L = A.lv[k];
    const BotLevel& C = A.lv[k - 1];
    for (int fi = tid; fi <= L.nn; fi += blockDim.x) {
      if (fi == L.nn) sm[L.off_x + L.ngrid] += sm[C.off_x + C.ngrid];
      else
        *reinterpret_cast<double2*>(sm + L.off_x + 2 * fi) =
            prolong_node(L.nx, L.fm, sm + L.off_x, C.nx, C.fm, sm + C.off_x, fi);
    }
    __syncthreads();
    bot_sweep<false, false>(L, sm, A, true);
    bot_sweep<false, false>(L, sm, A, false);
  }
  {
    const BotLevel& T = A.lv[A.kb];
    for (int i = tid; i <= T.ngrid; i += blockDim.x) A.gx[i] = sm[T.off_x + i];
  }
  VTS_TL_END(4, 5);
}

// Highest level the fused kernel can take (0 = none): below the top, <= 32
// node rows, and its vectors + one staged half-stencil fit in shared memory.
static int bottom_plan(Ctx* c, BotArgs* A, size_t* smem_bytes) {
  const int top = c->L - 1;
  int kb = 0;
  for (int k = 1; k < top && k < kBotMaxLevels; ++k) {
    if (c->lv[k].d.ny > 32) break;
    kb = k;
  }
  while (kb >= 1) {
    size_t off = 0;
    for (int k = 0; k <= kb; ++k) {
      const LevelDev& d = c->lv[k].d;
      BotLevel& b = A->lv[k];
      b.nx = d.nx;
      b.ny = d.ny;
      b.nn = d.nnodes;
      b.ngrid = d.ngrid;
      b.fm = d.free_mask;
      b.stL = d.stL;
      b.stU = d.stU;
      b.border = d.border;
      const size_t v = (size_t)d.ngrid + 2;  // ngrid + 1, kept even for double2 alignment
      b.off_b = (int)off;
      off += v;
      b.off_x = (int)off;
      off += v;
      b.off_r = (int)off;
      off += v;
    }
    A->off_stage = (int)off;
    off += ((size_t)c->lv[kb].d.nnodes + 2 * kBotPad) * kHalf;
    A->off_q = (int)off;
    off += 2 * ((size_t)c->lv[kb].d.nnodes + 2 * kBotPad);
    A->off_red = (int)off;
    off += 32 + 32 * 8;
    A->off_y = (int)off;
    off += (size_t)c->N0 + (c->N0 & 1);
    const size_t base = off * 8;
    const size_t chol = (size_t)c->N0 * c->N0 * 8;
    A->off_chol = -1;
    if (base + chol <= 200 * 1024) {
      A->off_chol = (int)off;
      off += (size_t)c->N0 * c->N0;
    }
    if (off * 8 <= 200 * 1024) {
      *smem_bytes = off * 8;
      A->kb = kb;
      return kb;
    }
    --kb;  // too big: fuse one level less
  }
  return 0;
}

static bool g_bot_attr_set = false;

// levels 0..kb of the V-cycle in one launch; L(kb).b must hold the restricted
// right-hand side, L(kb).x receives the level's result
static int vcycle_bottom(Ctx* c, const BotArgs& plan, size_t smem, const int* skip) {
  if (!g_bot_attr_set) {
    VTS_CUDA(cudaFuncSetAttribute(k_vcycle_bottom, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    g_bot_attr_set = true;
  }
  BotArgs A = plan;
  LevelBuf& T = c->lv[A.kb];
  A.gb = T.b;
  A.gx = T.x;
  A.corner = c->d_corner;
  A.N0 = c->N0;
  A.nfree0 = c->lv[0].d.nfree;
  A.f2g0 = c->lv[0].d.free2grid;
  A.chol = c->chol;
  A.rdiag = c->chol_rdiag;
  VTS_CUDA(launch_pdl(k_vcycle_bottom, dim3(1), dim3(kBotThreads), smem, c->stream, A, skip));
  VTS_LAUNCHED(c);
  return 0;
}

