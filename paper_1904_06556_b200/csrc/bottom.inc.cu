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
// time marks of one launch: kept in shared memory while the kernel runs (a global
// read-modify-write per mark cost ~2 us each and hid the picture), written out at the end
__device__ long long g_bot_probe[64];
__device__ int g_bot_n;
__shared__ long long s_bot_marks[64];
__shared__ int s_bot_n;
#define BOT_MARK()                                                 \
  do {                                                             \
    if (threadIdx.x == 0 && s_bot_n < 64) {                        \
      long long t_;                                                \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));       \
      s_bot_marks[s_bot_n++] = t_;                                 \
    }                                                              \
  } while (0)
#else
#define BOT_MARK() \
  do {             \
  } while (0)
#endif
constexpr int kBotMaxLevels = 8;
#ifndef VTS_BOT_EXP
#define VTS_BOT_EXP 0  // probe-only timing experiments on bot_coarse (results then wrong)
#endif
// the opt-in shared memory limit of one CTA less 1 KB of static shared memory (the prefetch
// barrier, the probe's marks)
constexpr size_t kBotSmemMax = 226 * 1024;
// The top fused level's first half-stencil (99 KB on C3) is fetched by one bulk copy issued
// BEFORE the kernel waits for the grids ahead of it (the stencils date from mg_setup): the
// first sweep's staging, 8.5 us of dependent global loads, shrinks to a barrier wait.
// VTS_BOT_PREFETCH=0: every staging by the block's threads.
#ifndef VTS_BOT_UNROLL
#define VTS_BOT_UNROLL 4  // steps per trip of the wavefront loop (code size against loop overhead)
#endif
constexpr int kBotUnroll = VTS_BOT_UNROLL;
#ifndef VTS_BOT_PREFETCH
#define VTS_BOT_PREFETCH 1
#endif
__shared__ unsigned long long s_bot_bar;

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
  int off_dblk;          // N0 > 32: two buffers of bot_coarse's diagonal + sub-diagonal blocks
};

// one Gauss-Seidel sweep of level L: x <- sweep(x; b) (zero_guess: x_old = 0)
// (not inlined: one copy of each sweep's code, warm in the instruction cache
// after its first use; inlined copies per call site ran 3.6x slower cold)
constexpr int kBotPad = 64;  // zero nodes before/after the staged level (>= 2 x 31, the largest skew)
template <bool FWD, bool ZERO>
// restage: 0 the stage still holds this level's half, 1 copy it, 2 it was prefetched (wait for the bulk copy)
__device__ __noinline__ void bot_sweep(const BotLevel& L, double* sm, const BotArgs& A, int restage) {
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
    if (restage == 1)  // the second sweep of a smoothing step solves with the same half: still staged
      for (int i = tid; i < end; i += blockDim.x) dst[i] = (i >= lo && i < hi) ? src[i - lo] : make_double2(0.0, 0.0);
    if (restage == 2) mbar_wait(&s_bot_bar, 0);  // the prefetched half has landed (its pads were zeroed at the start)
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
  // only the lanes that own a row: every shared-memory load and store of the loop costs
  // issue time per 128-byte wavefront
  const int nlanes = min(L.ny, 32);
  if (tid < nlanes) {
    // the wavefront of k_gs_tri on a single band: lane l = sweep row, skew 2,
    // software-pipelined, branch-free like k_gs_tri: every lane streams its row
    // through the padded stage with a pointer that moves one node per step;
    // positions off the row compute on finite real-neighbour or zero-pad data and
    // are never stored; every coupling that reads them at a valid position is an
    // exact zero
    const unsigned lanes = nlanes == 32 ? 0xffffffffu : ((1u << nlanes) - 1u);
    const int l = tid;
    const int nx = L.nx, ny = L.ny;  // registers: the loop must not re-read L through a generic pointer
    constexpr int d0 = FWD ? 0 : 1;
    constexpr int d1 = 1 - d0;
    constexpr int dir = FWD ? 1 : -1;
    // node of (row l, sweep column t - 2 l) at t = 0, in padded stage order
    const int n0 = FWD ? l * nx - 2 * l : (ny - 1 - l) * nx + nx - 1 + 2 * l;
    const double* ap = stage + (size_t)(kBotPad + n0) * kHalf;
    const double* pp = pst + (size_t)(kBotPad + n0) * 2;
    double* xp_out = sx + 2 * (ptrdiff_t)n0;
    struct StepData {
      double q0, q1, e00, e01, e10, e11, w00, w01, w10, w11, c, r0, r1;
    };
    // a step's shared-memory operands, loaded two steps ahead of the step that uses
    // them (as gs_compute): the loads' latency and gs_pre run in the shadow of the
    // recurrence of the steps in between
    struct Raw {
      double r[19];
      double2 pq;
    };
    auto load_raw = [&](int t, Raw& o) {
      const double* a = ap + (ptrdiff_t)t * dir * kHalf;
#pragma unroll
      for (int i = 0; i < 9; ++i) {
        const double2 v = reinterpret_cast<const double2*>(a)[i];
        o.r[2 * i] = v.x;
        o.r[2 * i + 1] = v.y;
      }
      o.r[18] = a[18];
      o.pq = *reinterpret_cast<const double2*>(pp + 2 * dir * t);
    };
    // gs_pre / gs_rec2 of k_gs_tri's skew-2 steps, so both paths compute the same bits
    auto prepare = [&](const Raw& in, const double2 xm, const double2 xz) {
      const double* r = in.r;
      StepData o;
      gs_pre<d0>(r, in.pq.x, in.pq.y, xm, xz, o.q0, o.q1);
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
    Raw ra;
    load_raw(0, ra);
    StepData cur = prepare(ra, win[0], win[1]);
    load_raw(1, ra);  // (reads at most two nodes past the last step: inside the stage's zero pad)
    double* const trash = sm + A.off_red;  // stores of off-row positions land here (unused during sweeps)
#pragma unroll kBotUnroll
    for (int t = 0; t < T; ++t) {
      const int j = t - 2 * l;
      const double2 nv = gs_rec2<d0>(cur.q0, cur.q1, cur.w00, cur.w01, cur.w10, cur.w11, cur.e00, cur.e01, cur.e10,
                                     cur.e11, cur.c, cur.r0, cur.r1, wprev, win[2]);
      const StepData nxt = prepare(ra, win[1], win[2]);
      load_raw(t + 2, ra);
      // branch-free store: off-row positions write the scratch slot instead
      double* dst = (j >= 0 && j < nx) ? xp_out + 2 * dir * t : trash;
      *reinterpret_cast<double2*>(dst) = nv;
      wprev = nv;
      double2 up;
      up.x = __shfl_up_sync(lanes, nv.x, 1);
      up.y = __shfl_up_sync(lanes, nv.y, 1);
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
__device__ __noinline__ void bot_coarse(const BotLevel& C, double* sm, const BotArgs& A) {
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
    // Blocked by 32 columns, bit-identical to the column-by-column substitution of
    // k_coarse_solve: every y[i] still receives its updates fma(-L[i][j], y[j], .) in
    // increasing j (decreasing j going back) and is divided right after its last one.
    // Per block: warp 0 solves the 32 x 32 diagonal block by shuffles (as the N <= 32
    // path), then every thread applies the block's 32 columns to its own later rows in
    // column order -- two barriers per block instead of two per column.
    // Blocks of 32 columns with one block of look-ahead, bit-identical to the
    // column-by-column substitution of k_coarse_solve: every y[i] still receives its
    // updates fma(-L[i][j], y[j], .) in increasing j (decreasing j going back) and is
    // divided right after its last one.  Phase k: warp 0 applies block k-1's columns
    // to block k's rows, then solves block k's 32 x 32 diagonal block by shuffles;
    // meanwhile warps 1.. apply block k-1's columns to the rows below block k and
    // stage block k+1's diagonal and sub-diagonal blocks into shared memory, so the
    // serial chain of warp 0 reads only shared memory.  One barrier per block.
    // The loops stay rolled: the fused kernel's sweeps run from the instruction
    // cache, and fully unrolled substitutions here evicted them (sweeps 6 -> 41 us).
    // The factor is read from global memory (ld.global.nc): N0 > 32 keeps no copy
    // in shared memory.
    const double* __restrict__ G = A.chol;
    const int lane = tid & 31, warp = tid >> 5;
    const int nb = (N + 31) / 32;
    constexpr int kBuf = 2 * 32 * 33 + 32;  // diagonal [32][33], sub-diagonal [32][33], rdiag [32]
    double* const buf0 = sm + A.off_dblk;
    // forward block k = columns [32k, min(32k + 32, N)); backward block b = [max(N - 32b - 32, 0), N - 32b)
    // stage the diagonal block [lo, hi) and the coupling block with [plo, phi) (forward:
    // sub[r][t] = L[lo + r][plo + t]; backward: sub[r][t] = L[plo + t][lo + r])
    auto stage = [&](double* B, int lo, int hi, int plo, int phi, bool fwd) {
      double* D = B;
      double* S = B + 32 * 33;
      for (int idx = tid - 32; idx < 32 * 32; idx += blockDim.x - 32) {
        const int a = idx >> 5, e = idx & 31;
        const double d = (e <= a && lo + a < hi) ? __ldg(G + (size_t)(lo + a) * N + lo + e) : 0.0;
        double v = 0.0;
        if (fwd && lo + a < hi && plo + e < phi) v = __ldg(G + (size_t)(lo + a) * N + plo + e);
        if (!fwd && plo + a < phi && lo + e < hi) v = __ldg(G + (size_t)(plo + a) * N + lo + e);
        D[a * 33 + e] = d;
        S[fwd ? a * 33 + e : e * 33 + a] = v;
      }
      if (tid >= 32 && tid < 64 && lo + tid - 32 < hi) B[2 * 32 * 33 + tid - 32] = __ldg(A.rdiag + lo + tid - 32);
    };
    if (warp > 0) stage(buf0, 0, min(32, N), 0, 0, true);
    __syncthreads();
    for (int ph = 0; ph < 2 * nb; ++ph) {
      const bool fwd = ph < nb;
      const int k = fwd ? ph : ph - nb;  // block index in this direction
      const int lo = fwd ? 32 * k : max(N - 32 * k - 32, 0), hi = fwd ? min(32 * k + 32, N) : N - 32 * k;
      const int plo = k == 0 ? 0 : fwd ? lo - 32 : hi, phi = k == 0 ? 0 : fwd ? lo : min(hi + 32, N);
      double* const B = buf0 + (ph & 1) * kBuf;
      if (warp == 0) {
        // block k-1's columns on block k's rows, then block k's diagonal solve
        const int r = lo + lane;
        const bool own = r < hi;
        double yi = own ? y[r] : 0.0;
        const double* S = B + 32 * 33 + lane * 33;
        const int np = phi - plo;
        if (fwd)
          for (int t = 0; t < np; ++t) yi = fma(-S[t], y[plo + t], yi);
        else
          for (int t = np - 1; t >= 0; --t) yi = fma(-S[t], y[plo + t], yi);
        const double* D = B;
        const double* rd = B + 2 * 32 * 33;
        const int n = hi - lo;
        for (int u = 0; u < n && VTS_BOT_EXP != 2; ++u) {
          const int t = fwd ? u : n - 1 - u;
          const double q = div_by(yi, D[t * 33 + t], rd[t]);
          yi = lane == t ? q : yi;
          const double yt = __shfl_sync(0xffffffffu, yi, t);
          const bool below = fwd ? lane > t : lane < t;
          const double l = below ? D[fwd ? lane * 33 + t : t * 33 + lane] : 0.0;
          yi = below ? fma(-l, yt, yi) : yi;
        }
        if (own) y[r] = yi;
      } else {
        // block k-1's columns on the rows beyond block k; stage block k+1
        if (k > 0 && VTS_BOT_EXP != 1) {
          const int i0 = fwd ? hi : 0, i1 = fwd ? N : lo;
          for (int i = i0 + tid - 32; i < i1; i += blockDim.x - 32) {
            double yi = y[i];
            if (fwd) {
              const double* li = G + (size_t)i * N + plo;
#pragma unroll 8
              for (int t = 0; t < 32; ++t) yi = fma(-__ldg(li + t), y[plo + t], yi);  // forward blocks k-1 are full
            } else {
#pragma unroll 8
              for (int t = phi - plo - 1; t >= 0; --t) yi = fma(-__ldg(G + (size_t)(plo + t) * N + i), y[plo + t], yi);
            }
            y[i] = yi;
          }
        }
        double* const Bn = buf0 + ((ph + 1) & 1) * kBuf;
        if (ph + 1 < nb) stage(Bn, lo + 32, min(hi + 32, N), lo, hi, true);
        else if (ph + 1 == nb) stage(Bn, max(N - 32, 0), N, 0, 0, false);
        else if (ph + 1 < 2 * nb) stage(Bn, max(lo - 32, 0), lo, lo, hi, false);
      }
      __syncthreads();
    }
    BOT_MARK();  // coarse: both substitutions
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
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x;
#if VTS_BOT_PREFETCH
  {
    // before the wait: nothing here depends on the grids ahead (read-only setup data -> shared memory)
    const BotLevel& T = A.lv[A.kb];
    double* stage = sm + A.off_stage;
    const unsigned bytes = (unsigned)((size_t)T.nn * kHalf * sizeof(double));
    if (tid == 0) {
      mbar_init(&s_bot_bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&s_bot_bar, bytes);
      bulk_g2s(stage + (size_t)kBotPad * kHalf, T.stL, bytes, &s_bot_bar);
    }
    double2* dst = reinterpret_cast<double2*>(stage);
    const int lo = kBotPad * kHalf / 2, hi = (kBotPad + T.nn) * kHalf / 2, end = (2 * kBotPad + T.nn) * kHalf / 2;
    for (int i = tid; i < lo; i += blockDim.x) dst[i] = make_double2(0.0, 0.0);
    for (int i = hi + tid; i < end; i += blockDim.x) dst[i] = make_double2(0.0, 0.0);
  }
#endif
  pdl_enter();
  if (skip && *skip) {
#if VTS_BOT_PREFETCH
    __syncthreads();  // (the barrier's initialisation)
    mbar_wait(&s_bot_bar, 0);  // no bulk copy may still be writing into this CTA's shared memory
#endif
    return;
  }
  VTS_TL_BEGIN(4, 5);
#ifdef VTS_BOT_PROBE
  if (tid == 0) s_bot_n = 0;
  __syncthreads();
  BOT_MARK();
#endif
  {
    const BotLevel& T = A.lv[A.kb];
    for (int i = tid; i <= T.ngrid; i += blockDim.x) sm[T.off_b + i] = A.gb[i];
  }
  __syncthreads();
  BOT_MARK();  // right-hand side loaded
  for (int k = A.kb; k >= 1; --k) {  // descent (multigrid.py:115-131)
    const BotLevel& L = A.lv[k];
    if (tid == 0) sm[L.off_x + L.ngrid] = 0.0;  // k_alpha_init on a coarse level
    __syncthreads();
    bot_sweep<true, true>(L, sm, A, (VTS_BOT_PREFETCH && k == A.kb) ? 2 : 1);
    bot_sweep<true, false>(L, sm, A, 0);
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
    BOT_MARK();  // restricted
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
    BOT_MARK();  // prolongated
    bot_sweep<false, false>(L, sm, A, 1);
    bot_sweep<false, false>(L, sm, A, 0);
  }
  {
    const BotLevel& T = A.lv[A.kb];
    for (int i = tid; i <= T.ngrid; i += blockDim.x) A.gx[i] = sm[T.off_x + i];
  }
#ifdef VTS_BOT_PROBE
  BOT_MARK();
  __syncthreads();
  if (tid == 0) {
    for (int i = 0; i < s_bot_n; ++i) g_bot_probe[i] = s_bot_marks[i];
    g_bot_n = s_bot_n;
  }
#endif
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
    A->off_dblk = (int)off;
    if (c->N0 > 32) off += 2 * (2 * 32 * 33 + 32);  // bot_coarse's double-buffered blocks
    const size_t base = off * 8;
    const size_t chol = (size_t)c->N0 * c->N0 * 8;
    A->off_chol = -1;
    if (c->N0 <= 32 && base + chol <= kBotSmemMax) {
      A->off_chol = (int)off;
      off += (size_t)c->N0 * c->N0;
    }
    if (off * 8 <= kBotSmemMax) {
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
    VTS_CUDA(cudaFuncSetAttribute(k_vcycle_bottom, cudaFuncAttributeMaxDynamicSharedMemorySize, kBotSmemMax));
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

