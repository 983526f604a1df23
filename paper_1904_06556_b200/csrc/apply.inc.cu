// Newton-matrix and level-operator applies (unity-built into vts_b200.cu).
//
// k_newton_apply: matrix-free y = S x for the bordered Schur matrix
//   S = [[sum_e rho_hat_e K_e + sum_e chat_e w_e w_e^T, -sum_e chat_e w_e],
//        [.^T, sum_e chat_e]],  w_e = K_e u_e
// i.e. BorderedMatrix.matvec (linalg.py:56-62) of ElementOps.assemble
// (fem.py:188-209) without ever forming the CSR matrix.  One CTA owns a
// 32 x 8 tile of nodes: it stages x and u of the (34 x 10)-node halo in shared
// memory, computes the 33 x 9 touching elements once each (w_e, theta_e =
// w_e.x_e - x_alpha, K_e x_e, the 8-vector rho_hat K_e x_e + chat theta w_e),
// then every thread gathers its node's four element contributions in the
// reference's scatter order.  No atomics; y_alpha = -sum chat_e theta_e is a
// deterministic last-block reduction over the elements each tile owns.
//
// k_level_apply: y = A_k x + border x_alpha, y_alpha = border.x + corner x_alpha
// on a stored 9-point block stencil (the residual of multigrid.py:125 and the
// parity probe of MgPreconditioner.mats[k].matvec).

namespace vts {

constexpr int kTX = 32, kTY = 8;
constexpr int kHX = kTX + 2, kHY = kTY + 2;  // halo nodes
constexpr int kEX = kTX + 1, kEY = kTY + 1;  // touching elements

__global__ void __launch_bounds__(kTX* kTY) k_newton_apply(int nx, int ny, int ex, int ey, int ngrid,
                                                         const double* __restrict__ ug,
                                                         const double* __restrict__ rho_hat,
                                                         const double* __restrict__ chat,
                                                         const uint8_t* __restrict__ fmask,
                                                         const double* __restrict__ x,
                                                         double* __restrict__ y, double* partials,
                                                         unsigned* counter, const int* skip) {
  if (skip && *skip) return;
  __shared__ double2 xs[kHY * kHX];
  __shared__ double2 us[kHY * kHX];
  __shared__ double contrib[kEY * kEX * 8];
  __shared__ double scratch[kTX * kTY / 32];
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY;
  const double xa = x[ngrid];

  for (int h = tid; h < kHY * kHX; h += blockDim.x) {
    const int gx = x0 - 1 + h % kHX, gy = y0 - 1 + h / kHX;
    double2 xv = make_double2(0.0, 0.0), uv = make_double2(0.0, 0.0);
    if (gx >= 0 && gx < nx && gy >= 0 && gy < ny) {
      const int nd = gx + nx * gy;
      xv = *reinterpret_cast<const double2*>(x + 2 * nd);
      uv = *reinterpret_cast<const double2*>(ug + 2 * nd);
    }
    xs[h] = xv;
    us[h] = uv;
  }
  __syncthreads();

  double acc[1] = {0.0};
  for (int le = tid; le < kEY * kEX; le += blockDim.x) {
    const int lx = le % kEX, ly = le / kEX;
    const int gx = x0 - 1 + lx, gy = y0 - 1 + ly;
    if (gx < 0 || gx >= ex || gy < 0 || gy >= ey) continue;
    const int e = gx + ex * gy;
    const int h0 = lx + kHX * ly;
    const int hn[4] = {h0, h0 + 1, h0 + kHX + 1, h0 + kHX};
    double ue[8], xe[8];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const double2 uv = us[hn[a]], xv = xs[hn[a]];
      ue[2 * a] = uv.x;
      ue[2 * a + 1] = uv.y;
      xe[2 * a] = xv.x;
      xe[2 * a + 1] = xv.y;
    }
    double w[8], kx[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double sw = ue[0] * c_ke[j], sk = xe[0] * c_ke[j];
#pragma unroll
      for (int i = 1; i < 8; ++i) {
        sw = fma(ue[i], c_ke[i * 8 + j], sw);
        sk = fma(xe[i], c_ke[i * 8 + j], sk);
      }
      w[j] = sw;
      kx[j] = sk;
    }
    double wx = w[0] * xe[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) wx = fma(w[i], xe[i], wx);
    const double ch = chat[e], rh = rho_hat[e];
    const double theta = wx - xa;
    const double ct = ch * theta;
#pragma unroll
    for (int j = 0; j < 8; ++j) contrib[le * 8 + j] = fma(ct, w[j], rh * kx[j]);
    if (gx >= x0 && gx < x0 + kTX && gy >= y0 && gy < y0 + kTY) acc[0] = fma(ch, theta, acc[0]);
  }
  __syncthreads();

  const int tx = tid % kTX, ty = tid / kTX;
  const int ix = x0 + tx, iy = y0 + ty;
  if (ix < nx && iy < ny) {
    // elements (ix-1,iy-1) c2, (ix,iy-1) c3, (ix-1,iy) c1, (ix,iy) c0  -> local (tx,ty) (tx+1,ty) (tx,ty+1) (tx+1,ty+1)
    double s0 = 0.0, s1 = 0.0;
    if (ix >= 1 && iy >= 1) {
      const double* cb = contrib + (tx + kEX * ty) * 8;
      s0 += cb[4]; s1 += cb[5];
    }
    if (ix < ex && iy >= 1) {
      const double* cb = contrib + (tx + 1 + kEX * ty) * 8;
      s0 += cb[6]; s1 += cb[7];
    }
    if (ix >= 1 && iy < ey) {
      const double* cb = contrib + (tx + kEX * (ty + 1)) * 8;
      s0 += cb[2]; s1 += cb[3];
    }
    if (ix < ex && iy < ey) {
      const double* cb = contrib + (tx + 1 + kEX * (ty + 1)) * 8;
      s0 += cb[0]; s1 += cb[1];
    }
    const int nd = ix + nx * iy;
    const uchar2 fm = *reinterpret_cast<const uchar2*>(fmask + 2 * nd);
    *reinterpret_cast<double2*>(y + 2 * nd) = make_double2(fm.x ? s0 : 0.0, fm.y ? s1 : 0.0);
  }
  double tot[1];
  // flatten the 2D grid for the last-block protocol
  __shared__ bool s_last;
  block_sum<1>(acc, scratch);
  const int bid = blockIdx.x + gridDim.x * blockIdx.y, nb = gridDim.x * gridDim.y;
  if (tid == 0) {
    partials[bid] = acc[0];
    __threadfence();
    s_last = (atomicAdd(counter, 1u) == (unsigned)nb - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  tot[0] = 0.0;
  for (int b = tid; b < nb; b += blockDim.x) tot[0] += __ldcg(partials + b);
  block_sum<1>(tot, scratch);
  if (tid == 0) {
    y[ngrid] = -tot[0];
    *counter = 0u;
  }
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
  if (skip && *skip) return;
  __shared__ double scratch[256 / 32];
  const int nnodes = nx * ny;
  const double xa = x[ngrid];
  double acc[1] = {0.0};
  for (int nd = blockIdx.x * blockDim.x + threadIdx.x; nd < nnodes; nd += gridDim.x * blockDim.x) {
    const int ix = nd % nx, iy = nd / nx;
    const double* l = stL + (size_t)nd * kHalf;
    const double* u = stU + (size_t)nd * kHalf;
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int blk = 0; blk < 9; ++blk) {
      const int dx = blk % 3 - 1, dy = blk / 3 - 1;
      const int jx = ix + dx, jy = iy + dy;
      double2 xv = make_double2(0.0, 0.0);
      if (jx >= 0 && jx < nx && jy >= 0 && jy < ny) xv = *reinterpret_cast<const double2*>(x + 2 * (jx + nx * jy));
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
    const double2 xv = *reinterpret_cast<const double2*>(x + 2 * nd);
    acc[0] = fma(bd.x, xv.x, acc[0]);
    acc[0] = fma(bd.y, xv.y, acc[0]);
    if (RESIDUAL) {
      const double2 bv = *reinterpret_cast<const double2*>(b + 2 * nd);
      s0 = bv.x - s0;
      s1 = bv.y - s1;
    }
    *reinterpret_cast<double2*>(y + 2 * nd) = make_double2(s0, s1);
  }
  double tot[1];
  if (last_block_reduce<1>(acc, scratch, partials, counter, tot) && threadIdx.x == 0) {
    const double ya = fma(*corner_ptr, xa, tot[0]);
    y[ngrid] = RESIDUAL ? b[ngrid] - ya : ya;
  }
}

int newton_apply_grid(Ctx* c, const double* x, double* y, const int* skip) {
  const LevelBuf& F = c->lv[c->L - 1];
  dim3 grid(div_up(F.d.nx, kTX), div_up(F.d.ny, kTY));
  if ((long long)grid.x * grid.y > kMaxBlocks * kMaxPartials) {
    set_error(4, "mesh too large for the apply partial buffer");
    return 4;
  }
  k_newton_apply<<<grid, kTX * kTY, 0, c->stream>>>(F.d.nx, F.d.ny, F.d.ex, F.d.ey, F.d.ngrid, c->u_grid,
                                                     c->rho_hat, c->chat, F.d.free_mask, x, y,
                                                     c->partials + kMaxBlocks * 8, c->counters + 4, skip);
  VTS_LAUNCHED(c);
  return 0;
}

int level_apply_grid(Ctx* c, int k, const double* x, double* y, const int* skip) {
  const LevelBuf& L = c->lv[k];
  const int grid = (int)std::min<long long>(div_up(L.d.nnodes, 256), kReduceGridCap);
  k_level_apply<false><<<grid, 256, 0, c->stream>>>(L.d.nx, L.d.ny, L.d.ngrid, L.d.stL, L.d.stU, L.d.border,
                                                     c->d_corner, x, nullptr, y, c->partials, c->counters + 5,
                                                     skip);
  VTS_LAUNCHED(c);
  return 0;
}

int level_residual_grid(Ctx* c, int k, const double* x, const double* b, double* r, const int* skip) {
  const LevelBuf& L = c->lv[k];
  const int grid = (int)std::min<long long>(div_up(L.d.nnodes, 256), kReduceGridCap);
  k_level_apply<true><<<grid, 256, 0, c->stream>>>(L.d.nx, L.d.ny, L.d.ngrid, L.d.stL, L.d.stU, L.d.border,
                                                    c->d_corner, x, b, r, c->partials, c->counters + 5, skip);
  VTS_LAUNCHED(c);
  return 0;
}

}  // namespace vts
