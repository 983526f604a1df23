// Galerkin V(2,2) multigrid on the node-block stencils (unity-built).
//
//  mg_setup  : MgPreconditioner.__init__ (multigrid.py:82-103)
//    k_fine_stencil  finest-level stencil of S straight from the element data
//                    (the CSR values of fem.py:199-204, summed per entry in
//                    element order like _AssemblyPattern.build, fem.py:132-139)
//    k_rap           coarse block stencil P^T A P (linalg.py:78), structured:
//                    every coarse node gathers its 3x3 fine support
//    k_symmetrize    (C + C^T)/2 (linalg.py:79) + reciprocal diagonals
//    k_restrict      P^T v (border chain linalg.py:80, residual restriction)
//    k_dense_coarse + k_cholesky   dense bordered coarsest matrix and its
//                    Cholesky factor with the trace-scaled shift fallback
//  vcycle_grid : MgPreconditioner.apply/_cycle (multigrid.py:109-143)
//    k_gs_sweep      exact-order lexicographic Gauss-Seidel (multigrid.py:35-64):
//                    wavefront, one lane per grid row, 32 rows per warp,
//                    rows skewed by two nodes, new values of the row before
//                    passed lane to lane with shuffles, warps chained through
//                    release/acquire progress counters in global memory
//    k_level_apply<true>  residual, then k_restrict / k_prolong_add
//    k_coarse_solve  two triangular solves with the coarsest factor

namespace vts {

// weight of coarse node (cx, cy) in the interpolant at fine node (fx, fy)
// (mesh.py:304-306: 1 on coinciding coordinates, 1/2 on odd ones)
VTS_DEVICE_INLINE double pweight(int fx, int fy, int cx, int cy) {
  const int dx = fx - 2 * cx, dy = fy - 2 * cy;
  if (dx < -1 || dx > 1 || dy < -1 || dy > 1) return 0.0;
  return (dx == 0 ? 1.0 : 0.5) * (dy == 0 ? 1.0 : 0.5);
}

// coarse parents of a fine coordinate, increasing (mesh.py:314-316)
VTS_DEVICE_INLINE int parents(int f, int (&q)[2]) {
  if (f & 1) {
    q[0] = (f - 1) >> 1;
    q[1] = (f + 1) >> 1;
    return 2;
  }
  q[0] = f >> 1;
  return 1;
}

// ---------------------------------------------------------------------------
// finest-level stencil of the Schur matrix from (u, rho_hat, chat)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_fine_stencil(int nx, int ny, int ex, int ey,
                                                    const double* __restrict__ ug,
                                                    const double* __restrict__ rho_hat,
                                                    const double* __restrict__ chat,
                                                    const uint8_t* __restrict__ fm,
                                                    double* __restrict__ st) {
  const int nd = blockIdx.x * blockDim.x + threadIdx.x;
  if (nd >= nx * ny) return;
  const int ix = nd % nx, iy = nd / nx;
  const NodeElems ne = node_elems(ix, iy, ex, ey);
  // corner offsets of the element's local nodes relative to its node 0
  const int cdx[4] = {0, 1, 1, 0}, cdy[4] = {0, 0, 1, 1};
  double blk[36];
#pragma unroll
  for (int i = 0; i < 36; ++i) blk[i] = 0.0;
  bool seen[36];
#pragma unroll
  for (int i = 0; i < 36; ++i) seen[i] = false;
  for (int k = 0; k < ne.cnt; ++k) {
    const int e = ne.e[k], li = ne.li[k];
    int n4[4];
    elem_nodes(e, ex, nx, n4);
    double ue[8], w[8];
    gather8(ug, n4, ue);
    ke_times(ue, w);
    const double rh = rho_hat[e], ch = chat[e];
#pragma unroll
    for (int lj = 0; lj < 4; ++lj) {
      const int dx = cdx[lj] - cdx[li], dy = cdy[lj] - cdy[li];
      const int b = (dy + 1) * 3 + (dx + 1);
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          // fem.py:199-201: rho_hat*K + chat*(w_i*w_j), summed over elements in order
          const double v = __dadd_rn(__dmul_rn(rh, c_ke[(2 * li + r) * 8 + 2 * lj + cc]),
                                     __dmul_rn(ch, __dmul_rn(w[2 * li + r], w[2 * lj + cc])));
          const int slot = 4 * b + 2 * r + cc;
          blk[slot] = seen[slot] ? __dadd_rn(blk[slot], v) : v;
          seen[slot] = true;
        }
    }
  }
  // drop rows/cols of Dirichlet dofs (fem.py:157-161)
  const uchar2 fi = *reinterpret_cast<const uchar2*>(fm + 2 * nd);
#pragma unroll
  for (int b = 0; b < 9; ++b) {
    const int jx = ix + b % 3 - 1, jy = iy + b / 3 - 1;
    uchar2 fj = make_uchar2(0, 0);
    if (jx >= 0 && jx < nx && jy >= 0 && jy < ny) fj = *reinterpret_cast<const uchar2*>(fm + 2 * (jx + nx * jy));
    if (!fi.x || !fj.x) blk[4 * b + 0] = 0.0;
    if (!fi.x || !fj.y) blk[4 * b + 1] = 0.0;
    if (!fi.y || !fj.x) blk[4 * b + 2] = 0.0;
    if (!fi.y || !fj.y) blk[4 * b + 3] = 0.0;
  }
  double* out = st + (size_t)nd * kStencilStride;
#pragma unroll
  for (int i = 0; i < 36; i += 2) *reinterpret_cast<double2*>(out + i) = make_double2(blk[i], blk[i + 1]);
  const double rd0 = fi.x ? 1.0 / blk[16] : 0.0;
  const double rd1 = fi.y ? 1.0 / blk[19] : 0.0;
  *reinterpret_cast<double2*>(out + 36) = make_double2(rd0, rd1);
  *reinterpret_cast<double2*>(out + 38) = make_double2(0.0, 0.0);
}

// ---------------------------------------------------------------------------
// coarse operator P^T A P (unsymmetrised) on coarse node I
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_rap(int fnx, int fny, const double* __restrict__ fst,
                                           const uint8_t* __restrict__ ffm, int cnx, int cny,
                                           const uint8_t* __restrict__ cfm, double* __restrict__ out) {
  const int cn = blockIdx.x * blockDim.x + threadIdx.x;
  if (cn >= cnx * cny) return;
  const int cx = cn % cnx, cy = cn / cnx;
  double acc[36];
#pragma unroll
  for (int i = 0; i < 36; ++i) acc[i] = 0.0;
  const uchar2 fI = *reinterpret_cast<const uchar2*>(cfm + 2 * cn);
  for (int fy = 2 * cy - 1; fy <= 2 * cy + 1; ++fy) {
    if (fy < 0 || fy >= fny) continue;
    for (int fx = 2 * cx - 1; fx <= 2 * cx + 1; ++fx) {
      if (fx < 0 || fx >= fnx) continue;
      const int fi = fx + fnx * fy;
      const uchar2 ff = *reinterpret_cast<const uchar2*>(ffm + 2 * fi);
      const double wI = pweight(fx, fy, cx, cy);
      const double pr0 = (ff.x && fI.x) ? wI : 0.0, pr1 = (ff.y && fI.y) ? wI : 0.0;
      if (pr0 == 0.0 && pr1 == 0.0) continue;
      const double* a = fst + (size_t)fi * kStencilStride;
      for (int b = 0; b < 9; ++b) {
        const int jx = fx + b % 3 - 1, jy = fy + b / 3 - 1;
        if (jx < 0 || jx >= fnx || jy < 0 || jy >= fny) continue;
        const double a00 = a[4 * b], a01 = a[4 * b + 1], a10 = a[4 * b + 2], a11 = a[4 * b + 3];
        const uchar2 fj = *reinterpret_cast<const uchar2*>(ffm + 2 * (jx + fnx * jy));
        // coarse parents of fine node j (one per even, two per odd coordinate)
        int qxs[2], qys[2];
        const int nqx = parents(jx, qxs), nqy = parents(jy, qys);
        for (int iqy = 0; iqy < nqy; ++iqy) {
          for (int iqx = 0; iqx < nqx; ++iqx) {
            const int qx = qxs[iqx], qy = qys[iqy];
            const int Dx = qx - cx, Dy = qy - cy;
            if (Dx < -1 || Dx > 1 || Dy < -1 || Dy > 1) continue;
            const double wJ = pweight(jx, jy, qx, qy);
            const uchar2 fJ = *reinterpret_cast<const uchar2*>(cfm + 2 * (qx + cnx * qy));
            const double pc0 = (fj.x && fJ.x) ? wJ : 0.0, pc1 = (fj.y && fJ.y) ? wJ : 0.0;
            const int D = (Dy + 1) * 3 + (Dx + 1);
            acc[4 * D + 0] = fma(pr0 * a00, pc0, acc[4 * D + 0]);
            acc[4 * D + 1] = fma(pr0 * a01, pc1, acc[4 * D + 1]);
            acc[4 * D + 2] = fma(pr1 * a10, pc0, acc[4 * D + 2]);
            acc[4 * D + 3] = fma(pr1 * a11, pc1, acc[4 * D + 3]);
          }
        }
      }
    }
  }
  double* o = out + (size_t)cn * kStencilStride;
#pragma unroll
  for (int i = 0; i < 36; i += 2) *reinterpret_cast<double2*>(o + i) = make_double2(acc[i], acc[i + 1]);
}

// (C + C^T)/2 and reciprocal diagonals
__global__ void k_symmetrize(int nx, int ny, const double* __restrict__ raw, const uint8_t* __restrict__ fm,
                             double* __restrict__ st) {
  const int nd = blockIdx.x * blockDim.x + threadIdx.x;
  if (nd >= nx * ny) return;
  const int ix = nd % nx, iy = nd / nx;
  const double* a = raw + (size_t)nd * kStencilStride;
  double* o = st + (size_t)nd * kStencilStride;
  for (int b = 0; b < 9; ++b) {
    const int dx = b % 3 - 1, dy = b / 3 - 1;
    const int jx = ix + dx, jy = iy + dy;
    double t[4] = {0.0, 0.0, 0.0, 0.0};
    if (jx >= 0 && jx < nx && jy >= 0 && jy < ny) {
      const double* bt = raw + (size_t)(jx + nx * jy) * kStencilStride + 4 * (8 - b);  // mirrored block
      t[0] = (a[4 * b + 0] + bt[0]) * 0.5;
      t[1] = (a[4 * b + 1] + bt[2]) * 0.5;
      t[2] = (a[4 * b + 2] + bt[1]) * 0.5;
      t[3] = (a[4 * b + 3] + bt[3]) * 0.5;
    }
    *reinterpret_cast<double2*>(o + 4 * b) = make_double2(t[0], t[1]);
    *reinterpret_cast<double2*>(o + 4 * b + 2) = make_double2(t[2], t[3]);
  }
  const uchar2 f = *reinterpret_cast<const uchar2*>(fm + 2 * nd);
  const double a00 = o[16], a11 = o[19];
  *reinterpret_cast<double2*>(o + 36) = make_double2(f.x ? 1.0 / a00 : 0.0, f.y ? 1.0 / a11 : 0.0);
  *reinterpret_cast<double2*>(o + 38) = make_double2(0.0, 0.0);
}

// ---------------------------------------------------------------------------
// transfers
// ---------------------------------------------------------------------------
// vc = P^T vf on free dofs (csc_matvec order: fine dofs in increasing index);
// with `bordered` the border slot is copied (multigrid.py:128-130)
__global__ void k_restrict(int fnx, int fny, const uint8_t* __restrict__ ffm, const double* __restrict__ vf,
                           int cnx, int cny, const uint8_t* __restrict__ cfm, double* __restrict__ vc,
                           int bordered, const int* skip) {
  if (skip && *skip) return;
  const int cn = blockIdx.x * blockDim.x + threadIdx.x;
  const int cnn = cnx * cny;
  if (cn > cnn) return;
  if (cn == cnn) {
    if (bordered) vc[2 * cnn] = vf[2 * fnx * fny];
    return;
  }
  const int cx = cn % cnx, cy = cn / cnx;
  const uchar2 fc = *reinterpret_cast<const uchar2*>(cfm + 2 * cn);
  double s0 = 0.0, s1 = 0.0;
  for (int fy = 2 * cy - 1; fy <= 2 * cy + 1; ++fy) {
    if (fy < 0 || fy >= fny) continue;
    for (int fx = 2 * cx - 1; fx <= 2 * cx + 1; ++fx) {
      if (fx < 0 || fx >= fnx) continue;
      const int fi = fx + fnx * fy;
      const double wv = pweight(fx, fy, cx, cy);
      const uchar2 ff = *reinterpret_cast<const uchar2*>(ffm + 2 * fi);
      const double2 v = *reinterpret_cast<const double2*>(vf + 2 * fi);
      if (ff.x) s0 += wv * v.x;
      if (ff.y) s1 += wv * v.y;
    }
  }
  *reinterpret_cast<double2*>(vc + 2 * cn) = make_double2(fc.x ? s0 : 0.0, fc.y ? s1 : 0.0);
}

// xf += P xc (multigrid.py:134-136): parents in increasing coarse index
__global__ void k_prolong_add(int fnx, int fny, const uint8_t* __restrict__ ffm, double* __restrict__ xf,
                              int cnx, int cny, const uint8_t* __restrict__ cfm, const double* __restrict__ xc,
                              const int* skip) {
  if (skip && *skip) return;
  const int fi = blockIdx.x * blockDim.x + threadIdx.x;
  const int fnn = fnx * fny;
  if (fi > fnn) return;
  if (fi == fnn) {
    xf[2 * fnn] += xc[2 * cnx * cny];
    return;
  }
  const int fx = fi % fnx, fy = fi / fnx;
  const uchar2 ff = *reinterpret_cast<const uchar2*>(ffm + 2 * fi);
  double s0 = 0.0, s1 = 0.0;
  int qxs[2], qys[2];
  const int nqx = parents(fx, qxs), nqy = parents(fy, qys);
  for (int iqy = 0; iqy < nqy; ++iqy) {
    for (int iqx = 0; iqx < nqx; ++iqx) {
      const int qx = qxs[iqx], qy = qys[iqy];
      const double wv = pweight(fx, fy, qx, qy);
      const int cn = qx + cnx * qy;
      const uchar2 fc = *reinterpret_cast<const uchar2*>(cfm + 2 * cn);
      const double2 v = *reinterpret_cast<const double2*>(xc + 2 * cn);
      if (fc.x) s0 += wv * v.x;
      if (fc.y) s1 += wv * v.y;
    }
  }
  double2 o = *reinterpret_cast<double2*>(xf + 2 * fi);
  if (ff.x) o.x += s0;
  if (ff.y) o.y += s1;
  *reinterpret_cast<double2*>(xf + 2 * fi) = o;
}

// ---------------------------------------------------------------------------
// exact-order Gauss-Seidel sweep (wavefront), v1
// ---------------------------------------------------------------------------
VTS_DEVICE_INLINE unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
VTS_DEVICE_INLINE void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <bool FWD>
__global__ void __launch_bounds__(32) k_gs_sweep(int nx, int ny, int ngrid, const double* __restrict__ st,
                                               const double* __restrict__ b, const double* __restrict__ border,
                                               double* x, unsigned long long* flags, const int* skip) {
  if (skip && *skip) return;
  const int lane = threadIdx.x, grp = blockIdx.x;
  const int r = grp * 32 + lane;  // row in sweep order
  const bool row_ok = r < ny;
  const int iy = FWD ? r : ny - 1 - r;
  const double xa = x[ngrid];
  const int nsteps = nx + 62;
  double pm0 = 0.0, pm1 = 0.0, pz0 = 0.0, pz1 = 0.0, pp0 = 0.0, pp1 = 0.0;  // previous row (new), cols j-1, j, j+1
  double w0 = 0.0, w1 = 0.0;                                                // own row, col j-1 (new)
  unsigned long long seen = 0;
  const int prev_row_y = FWD ? iy - 1 : iy + 1;  // grid row of the sweep-previous row
  const int next_row_y = FWD ? iy + 1 : iy - 1;
  if (lane == 0 && grp > 0) {
    // first two sweep columns of the previous group's last row (later ones arrive each step)
    const unsigned long long need = (unsigned long long)((nx > 1 ? 1 : 0) + 62 + 1);
    while (seen < need) seen = ld_acquire(flags + grp - 1);
    const int q0 = FWD ? 0 : nx - 1;
    const double2 v0 = __ldcg(reinterpret_cast<const double2*>(x + 2 * (q0 + nx * prev_row_y)));
    pz0 = v0.x;
    pz1 = v0.y;
    if (nx > 1) {
      const int q1 = FWD ? 1 : nx - 2;
      const double2 v1 = __ldcg(reinterpret_cast<const double2*>(x + 2 * (q1 + nx * prev_row_y)));
      pp0 = v1.x;
      pp1 = v1.y;
    }
  }
  for (int t = 0; t < nsteps; ++t) {
    const int j = t - 2 * lane;
    const bool active = row_ok && j >= 0 && j < nx;
    double n0 = 0.0, n1 = 0.0;
    if (active) {
      const int ix = FWD ? j : nx - 1 - j;
      const int nd = ix + nx * iy;
      const double* a = st + (size_t)nd * kStencilStride;
      double c[38];
#pragma unroll
      for (int k = 0; k < 19; ++k) {
        const double2 v = *reinterpret_cast<const double2*>(a + 2 * k);
        c[2 * k] = v.x;
        c[2 * k + 1] = v.y;
      }
      const double2 bv = *reinterpret_cast<const double2*>(b + 2 * nd);
      const double2 bd = *reinterpret_cast<const double2*>(border + 2 * nd);
      const double badj0 = __dsub_rn(bv.x, __dmul_rn(bd.x, xa));
      const double badj1 = __dsub_rn(bv.y, __dmul_rn(bd.y, xa));
      const double2 xo = *reinterpret_cast<const double2*>(x + 2 * nd);  // own old values
      // neighbour values by block index (dy+1)*3 + (dx+1) in grid coordinates
      double v0[9], v1[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) { v0[k] = 0.0; v1[k] = 0.0; }
      // sweep-previous row (new): sweep cols j-1, j, j+1
      if (FWD) {  // row iy-1: SW(0) S(1) SE(2) at ix-1, ix, ix+1
        v0[0] = pm0; v1[0] = pm1; v0[1] = pz0; v1[1] = pz1; v0[2] = pp0; v1[2] = pp1;
        v0[3] = w0; v1[3] = w1;  // W new
      } else {    // row iy+1: sweep col j-1 -> ix+1 (NE 8), j -> N 7, j+1 -> ix-1 (NW 6)
        v0[8] = pm0; v1[8] = pm1; v0[7] = pz0; v1[7] = pz1; v0[6] = pp0; v1[6] = pp1;
        v0[5] = w0; v1[5] = w1;  // E new
      }
      // old values: own row next node, sweep-next row three nodes
      {
        const int ox = FWD ? ix + 1 : ix - 1;
        if (ox >= 0 && ox < nx) {
          const double2 v = *reinterpret_cast<const double2*>(x + 2 * (ox + nx * iy));
          if (FWD) { v0[5] = v.x; v1[5] = v.y; } else { v0[3] = v.x; v1[3] = v.y; }
        }
        if (next_row_y >= 0 && next_row_y < ny) {
#pragma unroll
          for (int d = -1; d <= 1; ++d) {
            const int qx = ix + d;
            if (qx < 0 || qx >= nx) continue;
            const double2 v = *reinterpret_cast<const double2*>(x + 2 * (qx + nx * next_row_y));
            const int blk = (FWD ? 6 : 0) + (d + 1);
            v0[blk] = v.x;
            v1[blk] = v.y;
          }
        }
      }
      if (FWD) {
        // dof 0 then dof 1 (node-major, x then y)
        double s = badj0;
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          if (k == kBlockCenter) { s = fma(-c[4 * k + 1], xo.y, s); continue; }
          s = fma(-c[4 * k], v0[k], s);
          s = fma(-c[4 * k + 1], v1[k], s);
        }
        n0 = s * c[kRd0];
        s = badj1;
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          if (k == kBlockCenter) { s = fma(-c[4 * k + 2], n0, s); continue; }
          s = fma(-c[4 * k + 2], v0[k], s);
          s = fma(-c[4 * k + 3], v1[k], s);
        }
        n1 = s * c[kRd1];
      } else {
        // backward order: dof 1 then dof 0
        double s = badj1;
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          if (k == kBlockCenter) { s = fma(-c[4 * k + 2], xo.x, s); continue; }
          s = fma(-c[4 * k + 2], v0[k], s);
          s = fma(-c[4 * k + 3], v1[k], s);
        }
        n1 = s * c[kRd1];
        s = badj0;
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          if (k == kBlockCenter) { s = fma(-c[4 * k + 1], n1, s); continue; }
          s = fma(-c[4 * k], v0[k], s);
          s = fma(-c[4 * k + 1], v1[k], s);
        }
        n0 = s * c[kRd0];
      }
      *reinterpret_cast<double2*>(x + 2 * nd) = make_double2(n0, n1);
      w0 = n0;
      w1 = n1;
    }
    // hand the new value to the next row (it needs sweep col j+1 at its step t+1 ... as its col j+2)
    double r0 = __shfl_up_sync(0xffffffffu, n0, 1);
    double r1 = __shfl_up_sync(0xffffffffu, n1, 1);
    if (lane == 0) {
      r0 = 0.0;
      r1 = 0.0;
      const int jn = t + 2;  // sweep column needed next step (+1 ahead)
      if (grp > 0 && row_ok && jn < nx && prev_row_y >= 0 && prev_row_y < ny) {
        const unsigned long long need = (unsigned long long)(jn + 62 + 1);
        while (seen < need) seen = ld_acquire(flags + grp - 1);
        const int qx = FWD ? jn : nx - 1 - jn;
        const double2 v = __ldcg(reinterpret_cast<const double2*>(x + 2 * (qx + nx * prev_row_y)));
        r0 = v.x;
        r1 = v.y;
      }
    }
    pm0 = pz0; pm1 = pz1;
    pz0 = pp0; pz1 = pp1;
    pp0 = r0; pp1 = r1;
    __syncwarp();
    if (lane == 31 && ((t & 7) == 7 || t == nsteps - 1)) st_release(flags + grp, (unsigned long long)(t + 1));
  }
  // lane 0 consumed flags[grp-1]; nobody reads it again in this launch
  if (lane == 0 && grp > 0) flags[grp - 1] = 0ull;
}

// ---------------------------------------------------------------------------
// finest-level border unknown relaxation (multigrid.py:121-122, 141-142)
// ---------------------------------------------------------------------------
__global__ void k_alpha_init(int ngrid, const double* b, double* x, const double* corner, const int* skip) {
  if (skip && *skip) return;
  x[ngrid] = b[ngrid] / *corner;
}

__global__ void k_alpha_relax(int ngrid, const double* __restrict__ border, const double* b, double* x,
                              const double* corner, double* partials, unsigned* counter, const int* skip) {
  if (skip && *skip) return;
  __shared__ double scratch[256 / 32];
  double acc[1] = {0.0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ngrid; i += gridDim.x * blockDim.x)
    acc[0] = fma(border[i], x[i], acc[0]);
  double tot[1];
  if (last_block_reduce<1>(acc, scratch, partials, counter, tot) && threadIdx.x == 0) {
    const double cr = *corner, xa = x[ngrid];
    x[ngrid] = xa + ((b[ngrid] - tot[0]) - cr * xa) / cr;
  }
}

// ---------------------------------------------------------------------------
// coarsest level: dense bordered matrix, Cholesky, triangular solves
// ---------------------------------------------------------------------------
__global__ void k_dense_coarse(int nx, int ny, const double* __restrict__ st, const double* __restrict__ border,
                               const int32_t* __restrict__ g2f, const double* corner, int N, double shift,
                               double* __restrict__ A) {
  // one thread per (free row, neighbour block) ; zero-fill first via memset
  const int nd = blockIdx.x * blockDim.x + threadIdx.x;
  if (nd >= nx * ny) return;
  const int ix = nd % nx, iy = nd / nx;
  for (int r = 0; r < 2; ++r) {
    const int fi = g2f[2 * nd + r];
    if (fi < 0) continue;
    for (int b = 0; b < 9; ++b) {
      const int jx = ix + b % 3 - 1, jy = iy + b / 3 - 1;
      if (jx < 0 || jx >= nx || jy < 0 || jy >= ny) continue;
      for (int cc = 0; cc < 2; ++cc) {
        const int fj = g2f[2 * (jx + nx * jy) + cc];
        if (fj < 0) continue;
        A[(size_t)fi * N + fj] = st[(size_t)nd * kStencilStride + 4 * b + 2 * r + cc];
      }
    }
    A[(size_t)fi * N + (N - 1)] = border[2 * nd + r];
    A[(size_t)(N - 1) * N + fi] = border[2 * nd + r];
  }
  if (nd == 0) A[(size_t)(N - 1) * N + (N - 1)] = *corner;
}

__global__ void k_add_shift(int N, double scale, double* A, double* trace_out) {
  // single block: trace, then A += scale * trace / N * I
  __shared__ double scratch[1024 / 32];
  double t[1] = {0.0};
  for (int i = threadIdx.x; i < N; i += blockDim.x) t[0] += A[(size_t)i * N + i];
  block_sum<1>(t, scratch);
  __shared__ double s_shift;
  if (threadIdx.x == 0) {
    s_shift = scale * t[0] / N;
    *trace_out = s_shift;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < N; i += blockDim.x) A[(size_t)i * N + i] += s_shift;
}

// in-place lower Cholesky, left-looking by columns, one CTA; status 0 ok, 1 fail
__global__ void __launch_bounds__(1024) k_cholesky(int N, double* A, int* status) {
  __shared__ double scratch[1024 / 32];
  __shared__ double s_diag;
  __shared__ int s_fail;
  if (threadIdx.x == 0) s_fail = 0;
  __syncthreads();
  for (int j = 0; j < N; ++j) {
    double t[1] = {0.0};
    for (int k = threadIdx.x; k < j; k += blockDim.x) t[0] = fma(A[(size_t)j * N + k], A[(size_t)j * N + k], t[0]);
    block_sum<1>(t, scratch);
    if (threadIdx.x == 0) {
      const double d = A[(size_t)j * N + j] - t[0];
      if (!(d > 0.0)) s_fail = 1;
      s_diag = sqrt(d);
      A[(size_t)j * N + j] = s_diag;
    }
    __syncthreads();
    if (s_fail) break;
    const double dj = s_diag;
    for (int i = j + 1 + threadIdx.x; i < N; i += blockDim.x) {
      double s = A[(size_t)i * N + j];
      for (int k = 0; k < j; ++k) s = fma(-A[(size_t)i * N + k], A[(size_t)j * N + k], s);
      A[(size_t)i * N + j] = s / dj;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *status = s_fail;
}

__global__ void __launch_bounds__(1024) k_coarse_solve(int N, int nfree, int ngrid, const double* __restrict__ Lf,
                                                     const int32_t* __restrict__ f2g, const double* __restrict__ b,
                                                     double* __restrict__ x, const int* skip) {
  if (skip && *skip) return;
  extern __shared__ double y[];
  for (int i = threadIdx.x; i < N; i += blockDim.x) y[i] = (i < nfree) ? b[f2g[i]] : b[ngrid];
  __syncthreads();
  for (int j = 0; j < N; ++j) {  // L y = b
    if (threadIdx.x == 0) y[j] = y[j] / Lf[(size_t)j * N + j];
    __syncthreads();
    const double yj = y[j];
    for (int i = j + 1 + threadIdx.x; i < N; i += blockDim.x) y[i] = fma(-Lf[(size_t)i * N + j], yj, y[i]);
    __syncthreads();
  }
  for (int j = N - 1; j >= 0; --j) {  // L^T x = y
    if (threadIdx.x == 0) y[j] = y[j] / Lf[(size_t)j * N + j];
    __syncthreads();
    const double yj = y[j];
    for (int i = threadIdx.x; i < j; i += blockDim.x) y[i] = fma(-Lf[(size_t)j * N + i], yj, y[i]);
    __syncthreads();
  }
  for (int i = threadIdx.x; i <= ngrid; i += blockDim.x) x[i] = 0.0;
  __syncthreads();
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    if (i < nfree) x[f2g[i]] = y[i];
    else x[ngrid] = y[i];
  }
}

// ---------------------------------------------------------------------------
// host drivers
// ---------------------------------------------------------------------------
static int gs_sweep(Ctx* c, int k, const double* b, double* x, bool forward, const int* skip) {
  LevelBuf& L = c->lv[k];
  const int groups = div_up(L.d.ny, 32);
  if (forward)
    k_gs_sweep<true><<<groups, 32, 0, c->stream>>>(L.d.nx, L.d.ny, L.d.ngrid, L.d.stencil, b, L.d.border, x,
                                                    L.gs_flags, skip);
  else
    k_gs_sweep<false><<<groups, 32, 0, c->stream>>>(L.d.nx, L.d.ny, L.d.ngrid, L.d.stencil, b, L.d.border, x,
                                                     L.gs_flags, skip);
  VTS_LAUNCHED(c);
  return 0;
}

int level_residual_grid(Ctx* c, int k, const double* x, const double* b, double* r, const int* skip);

int vcycle_grid(Ctx* c, const double* b_top, double* z_top, const int* skip) {
  const int top = c->L - 1;
  // descent
  for (int k = top; k >= 1; --k) {
    LevelBuf& L = c->lv[k];
    const double* b = (k == top) ? b_top : L.b;
    double* x = (k == top) ? z_top : L.x;
    VTS_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * (L.d.ngrid + 1), c->stream));
    if (k == top) {
      k_alpha_init<<<1, 1, 0, c->stream>>>(L.d.ngrid, b, x, c->d_corner, skip);
      VTS_LAUNCHED(c);
    }
    for (int s = 0; s < 2; ++s)
      if (int rc = gs_sweep(c, k, b, x, true, skip)) return rc;
    if (int rc = level_residual_grid(c, k, x, b, L.r, skip)) return rc;
    LevelBuf& C = c->lv[k - 1];
    k_restrict<<<div_up(C.d.nnodes + 1, 256), 256, 0, c->stream>>>(L.d.nx, L.d.ny, L.d.free_mask, L.r, C.d.nx,
                                                                     C.d.ny, C.d.free_mask, C.b, 1, skip);
    VTS_LAUNCHED(c);
  }
  {
    LevelBuf& C = c->lv[0];
    double* x0 = (top == 0) ? z_top : C.x;
    const double* b0 = (top == 0) ? b_top : C.b;
    k_coarse_solve<<<1, 1024, sizeof(double) * c->N0, c->stream>>>(c->N0, C.d.nfree, C.d.ngrid, c->chol,
                                                                    C.d.free2grid, b0, x0, skip);
    VTS_LAUNCHED(c);
  }
  // ascent
  for (int k = 1; k <= top; ++k) {
    LevelBuf& L = c->lv[k];
    LevelBuf& C = c->lv[k - 1];
    const double* b = (k == top) ? b_top : L.b;
    double* x = (k == top) ? z_top : L.x;
    k_prolong_add<<<div_up(L.d.nnodes + 1, 256), 256, 0, c->stream>>>(L.d.nx, L.d.ny, L.d.free_mask, x, C.d.nx,
                                                                        C.d.ny, C.d.free_mask, C.x, skip);
    VTS_LAUNCHED(c);
    for (int s = 0; s < 2; ++s)
      if (int rc = gs_sweep(c, k, b, x, false, skip)) return rc;
    if (k == top) {
      const int grid = (int)std::min<long long>(div_up(L.d.ngrid, 256), kReduceGridCap);
      k_alpha_relax<<<grid, 256, 0, c->stream>>>(L.d.ngrid, L.d.border, b, x, c->d_corner, c->partials,
                                                  c->counters + 6, skip);
      VTS_LAUNCHED(c);
    }
  }
  return 0;
}

int mg_setup(Ctx* c, double shift_scale) {
  if (!c->system_bound) {
    set_error(4, "mg_setup: no Newton system bound (call vts_schur_system first)");
    return 4;
  }
  const int top = c->L - 1;
  {
    LevelBuf& F = c->lv[top];
    k_fine_stencil<<<div_up(F.d.nnodes, 128), 128, 0, c->stream>>>(F.d.nx, F.d.ny, F.d.ex, F.d.ey, c->u_grid,
                                                                    c->rho_hat, c->chat, F.d.free_mask,
                                                                    F.d.stencil);
    VTS_LAUNCHED(c);
  }
  for (int k = top; k >= 1; --k) {
    LevelBuf& F = c->lv[k];
    LevelBuf& C = c->lv[k - 1];
    double* tmp = c->rap_tmp;
    k_rap<<<div_up(C.d.nnodes, 128), 128, 0, c->stream>>>(F.d.nx, F.d.ny, F.d.stencil, F.d.free_mask, C.d.nx,
                                                           C.d.ny, C.d.free_mask, tmp);
    VTS_LAUNCHED(c);
    k_symmetrize<<<div_up(C.d.nnodes, 128), 128, 0, c->stream>>>(C.d.nx, C.d.ny, tmp, C.d.free_mask, C.d.stencil);
    VTS_LAUNCHED(c);
    k_restrict<<<div_up(C.d.nnodes + 1, 256), 256, 0, c->stream>>>(F.d.nx, F.d.ny, F.d.free_mask, F.d.border,
                                                                     C.d.nx, C.d.ny, C.d.free_mask, C.d.border, 0,
                                                                     nullptr);
    VTS_LAUNCHED(c);
  }
  // coarsest dense factor
  LevelBuf& C = c->lv[0];
  const int N = c->N0;
  auto build = [&](double shift_scale_now) -> int {
    VTS_CUDA(cudaMemsetAsync(c->chol, 0, sizeof(double) * N * N, c->stream));
    k_dense_coarse<<<div_up(C.d.nnodes, 128), 128, 0, c->stream>>>(C.d.nx, C.d.ny, C.d.stencil, C.d.border,
                                                                    C.grid2free, c->d_corner, N, 0.0, c->chol);
    VTS_LAUNCHED(c);
    if (shift_scale_now != 0.0) {
      k_add_shift<<<1, 1024, 0, c->stream>>>(N, shift_scale_now, c->chol, c->dscal + 20);
      VTS_LAUNCHED(c);
    }
    k_cholesky<<<1, 1024, 0, c->stream>>>(N, c->chol, c->chol_status);
    VTS_LAUNCHED(c);
    int st = 0;
    VTS_CUDA(cudaMemcpyAsync(&st, c->chol_status, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    VTS_CUDA(cudaStreamSynchronize(c->stream));
    return st ? -1 : 0;
  };
  int rc = build(0.0);
  if (rc > 0) return rc;
  c->shifted = 0;
  if (rc < 0) {
    rc = build(shift_scale);
    if (rc > 0) return rc;
    if (rc < 0) {
      set_error(6, "coarse Cholesky failed even with the shift");
      return 6;
    }
    c->shifted = 1;
  }
  c->mg_ready = true;
  return 0;
}

}  // namespace vts

namespace vts {

// Per-kernel device times (CUDA events on the context stream, averaged over
// `reps` back-to-back launches) for bench.py's roofline: ms[0] Newton apply,
// ms[1] one V-cycle, ms[2] one forward GS sweep on the finest level, ms[3] one
// forward GS sweep on the second-finest level, ms[4] finest residual,
// ms[5] mg_setup (stencil + Galerkin chain + coarse factor, incl. one sync).
int time_kernels(Ctx* c, int reps, double* ms) {
  if (!c->mg_ready) {
    set_error(4, "time_kernels: multigrid not set up");
    return 4;
  }
  const int top = c->L - 1;
  LevelBuf& F = c->lv[top];
  double* xin = c->fvec[10];
  double* yout = c->fvec[11];
  cudaEvent_t e0, e1;
  VTS_CUDA(cudaEventCreate(&e0));
  VTS_CUDA(cudaEventCreate(&e1));
  auto timed = [&](auto&& body, double* out) -> int {
    if (int rc = body()) return rc;  // warm
    VTS_CUDA(cudaEventRecord(e0, c->stream));
    for (int r = 0; r < reps; ++r)
      if (int rc = body()) return rc;
    VTS_CUDA(cudaEventRecord(e1, c->stream));
    VTS_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    VTS_CUDA(cudaEventElapsedTime(&t, e0, e1));
    *out = (double)t / reps;
    return 0;
  };
  int rc = 0;
  rc = rc ? rc : timed([&] { return newton_apply_grid(c, xin, yout, nullptr); }, ms + 0);
  rc = rc ? rc : timed([&] { return vcycle_grid(c, xin, yout, nullptr); }, ms + 1);
  rc = rc ? rc : timed([&] { return gs_sweep(c, top, xin, F.x, true, nullptr); }, ms + 2);
  if (top >= 1) {
    LevelBuf& G = c->lv[top - 1];
    rc = rc ? rc : timed([&] { return gs_sweep(c, top - 1, G.b, G.x, true, nullptr); }, ms + 3);
  } else {
    ms[3] = 0.0;
  }
  rc = rc ? rc : timed([&] { return level_residual_grid(c, top, F.x, xin, F.r, nullptr); }, ms + 4);
  rc = rc ? rc : timed([&] { return mg_setup(c, 1e-12); }, ms + 5);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return rc;
}

}  // namespace vts
