// The reference's own discretisation: trilinear hexahedra.
//
// The reference is 3D (mesh.py, fem.py:31-97: 8-node hexahedra, 24 dofs per
// element, 81 nonzeros per row).  This file runs the same PBM Newton step on
// its `CANT/BRIDGE-mx-my-mz-L` hierarchies, so the unmodified reference is the
// oracle with no glue.  Same contract and entry points as the 2D path (the
// context carries dim = 3); what differs is the data layout:
//
//  * node grid nx*ny*nz (x fastest), 3 dofs per node: grid index 3 node + c,
//    the border unknown after it; Dirichlet dofs stored as 0;
//  * every level operator (the finest one assembled at schur_system time, as
//    the reference assembles its CSR, fem.py:188-209) is a full 27-point block
//    stencil: per node, neighbour b = (dz, dy, dx) in increasing node order,
//    3 x 3 block row-major -- 243 doubles, i.e. the CSR row's columns in order;
//  * element products w_e = u_e K_e (24 each) are stored by the element pass
//    and read by the node passes (no 8-fold recomputation).
//
// Kernels (one per reference operation, fp64):
//   k3_phi_elem / k3_phi_node   eval_lagrangian (pbm.py:150-199)
//   k3_w_elem, k3_schur_node    schur_system's scatters (pbm.py:202-218)
//   k3_fine_stencil             ElementOps.assemble (fem.py:188-209)
//   k3_rap, k3_symmetrize       BorderedMatrix.galerkin (linalg.py:76-81), in
//                               the reference's summation order (inner A P sums
//                               in column order, then the outer sum over fine rows)
//   k3_restrict, k3_prolong     P^T r / x + P e with trilinear weights (mesh.py:290-332)
//   k3_level_apply<R>           BorderedMatrix.matvec / the V-cycle residual
//   k3_gs<FWD>                  lexicographic Gauss-Seidel (multigrid.py:35-64)
//                               as a row pipeline: one warp per grid row (x
//                               pencil), rows taken by ticket in sweep order,
//                               each row waiting only for the rows before it
//                               to pass column i+1 (per-row progress counters);
//                               the sums are the reference's exact sequence
//                               (CSR order, separate multiply and subtract)
//   k3_dense_coarse             the coarsest bordered matrix for k_cholesky
//   k3_recon_elem, k3_al_elem   reconstruct_nu, _al_value
// The Cholesky factor, the coarse solve, the border relaxation, MINRES's
// recurrences, the outer update and the gap are the 2D path's kernels: they
// never look at the grid shape.

namespace vts {

constexpr int kNb3 = 27;
constexpr int kRow3 = kNb3 * 9;  // doubles of one node's stencil row

__constant__ double c_ke3[576];  // finest K_e, row-major 24 x 24

struct Level3 {
  int ex = 0, ey = 0, ez = 0, nx = 0, ny = 0, nz = 0, nnodes = 0, ngrid = 0, nfree = 0;
  uint8_t* fmask = nullptr;   // [ngrid]
  int32_t* g2f = nullptr;     // [ngrid]
  int32_t* f2g = nullptr;     // [nfree]
  double* st = nullptr;       // [nnodes * 243]
  double* border = nullptr;   // [ngrid + 1]
  double *b = nullptr, *x = nullptr, *r = nullptr;  // [ngrid + 1]
  unsigned* progress = nullptr;  // [ny * nz + 1]: per row, then the ticket counter
};

struct Hex {
  std::vector<Level3> lv;
  double* w = nullptr;       // [m * 24] element products of the bound / evaluated u
  double* u_grid = nullptr;  // [ngrid + 1]
  double* g[6] = {};         // finest grid work vectors [ngrid + 1]
  double* rap_tmp = nullptr; // unsymmetrised coarse stencil
  double ke[576];
};

// ---------------------------------------------------------------------------
// element helpers
// ---------------------------------------------------------------------------
VTS_DEVICE_INLINE void elem3_nodes(int e, int ex, int ey, int nx, int ny, int (&nd)[8]) {
  const int exi = e % ex, eyi = (e / ex) % ey, ezi = e / (ex * ey);
  const int b = exi + nx * (eyi + ny * ezi);
  const int sz = nx * ny;
  nd[0] = b;
  nd[1] = b + 1;
  nd[2] = b + nx + 1;
  nd[3] = b + nx;
  nd[4] = b + sz;
  nd[5] = b + sz + 1;
  nd[6] = b + sz + nx + 1;
  nd[7] = b + sz + nx;
}

VTS_DEVICE_INLINE void gather24(const double* __restrict__ g, const int (&nd)[8], double (&v)[24]) {
#pragma unroll
  for (int a = 0; a < 8; ++a) {
#pragma unroll
    for (int c = 0; c < 3; ++c) v[3 * a + c] = g[3 * nd[a] + c];
  }
}

// w = u_e K_e (fem.py:178 `ue @ ke`)
VTS_DEVICE_INLINE void ke3_times(const double (&ue)[24], double (&w)[24]) {
#pragma unroll
  for (int j = 0; j < 24; ++j) {
    double s = ue[0] * c_ke3[j];
#pragma unroll
    for (int i = 1; i < 24; ++i) s = fma(ue[i], c_ke3[i * 24 + j], s);
    w[j] = s;
  }
}

VTS_DEVICE_INLINE double dot24(const double (&a)[24], const double (&b)[24]) {
  double s = a[0] * b[0];
#pragma unroll
  for (int i = 1; i < 24; ++i) s = fma(a[i], b[i], s);
  return s;
}

// corner index (VTK order, mesh.py:47-56) of offset (dx, dy, dz) in {0,1}^3
VTS_DEVICE_INLINE int corner3(int dx, int dy, int dz) {
  const int base = dz ? 4 : 0;
  if (!dy) return base + dx;        // (0,0,z) -> 0/4, (1,0,z) -> 1/5
  return base + (dx ? 2 : 3);       // (1,1,z) -> 2/6, (0,1,z) -> 3/7
}

// the (up to) eight elements around node (ix, iy, iz) in increasing element
// index -- the accumulation order of the reference's bincount scatter
// (fem.py:170-173) -- and the node's corner in each
struct NodeElems3 {
  int e[8];
  int li[8];
  int cnt;
};

VTS_DEVICE_INLINE NodeElems3 node_elems3(int ix, int iy, int iz, int ex, int ey, int ez) {
  NodeElems3 r;
  r.cnt = 0;
  for (int dz = 1; dz >= 0; --dz) {
    const int ez_i = iz - dz;
    if (ez_i < 0 || ez_i >= ez) continue;
    for (int dy = 1; dy >= 0; --dy) {
      const int ey_i = iy - dy;
      if (ey_i < 0 || ey_i >= ey) continue;
      for (int dx = 1; dx >= 0; --dx) {
        const int ex_i = ix - dx;
        if (ex_i < 0 || ex_i >= ex) continue;
        r.e[r.cnt] = ex_i + ex * (ey_i + ey * ez_i);
        r.li[r.cnt++] = corner3(dx, dy, dz);
      }
    }
  }
  return r;
}

// ---------------------------------------------------------------------------
// eval_lagrangian (pbm.py:150-199): element pass (stores w) + node pass
// ---------------------------------------------------------------------------
struct Phi3Args {
  int m, ex, ey, nx, ny;
  const double* ug;
  double alpha, branch;
  const double *nu_lo, *nu_up, *rho, *mu_lo, *mu_up, *p, *q_lo, *q_up, *lower, *upper;
  double *q, *rho_hat, *mu_hat_lo, *mu_hat_up, *a, *b_lo, *b_up, *res_lo, *res_up, *w;
};

__global__ void __launch_bounds__(kThreads) k3_phi_elem(Phi3Args A, double* partials, unsigned* flags) {
  __shared__ double scratch[7 * kThreads / 32];
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  unsigned sat = 0;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < A.m; e += gridDim.x * blockDim.x) {
    int nd[8];
    elem3_nodes(e, A.ex, A.ey, A.nx, A.ny, nd);
    double ue[24], w[24];
    gather24(A.ug, nd, ue);
    ke3_times(ue, w);
    const double qq = 0.5 * dot24(w, ue);
    const double nlo = A.nu_lo[e], nup = A.nu_up[e], pe = A.p[e], qlo = A.q_lo[e], qup = A.q_up[e];
    const double rh = A.rho[e], mlo = A.mu_lo[e], mup = A.mu_up[e];
    const double s = __dsub_rn(__dadd_rn(__dsub_rn(qq, A.alpha), nlo), nup);
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
#pragma unroll
    for (int j = 0; j < 24; ++j) A.w[24 * (size_t)e + j] = w[j];
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

// res_u = scatter(rho_hat w) - f in free order; ||res_u||^2 and f.u partials
__global__ void __launch_bounds__(kThreads) k3_phi_node(int nnodes, int nx, int ny, int ex, int ey, int ez,
                                                      const double* __restrict__ ug, const double* __restrict__ w,
                                                      const double* __restrict__ coef, const double* __restrict__ f,
                                                      const int32_t* __restrict__ g2f, double* __restrict__ res_u,
                                                      double* partials) {
  __shared__ double scratch[2 * kThreads / 32];
  double acc[2] = {0, 0};
  for (int nd = blockIdx.x * blockDim.x + threadIdx.x; nd < nnodes; nd += gridDim.x * blockDim.x) {
    const int ix = nd % nx, iy = (nd / nx) % ny, iz = nd / (nx * ny);
    const NodeElems3 ne = node_elems3(ix, iy, iz, ex, ey, ez);
    double s[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < ne.cnt; ++k) {
      const double* we = w + 24 * (size_t)ne.e[k] + 3 * ne.li[k];
      const double rh = coef[ne.e[k]];
#pragma unroll
      for (int c = 0; c < 3; ++c) s[c] = __dadd_rn(s[c], __dmul_rn(rh, we[c]));
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int fi = g2f[3 * nd + c];
      if (fi < 0) continue;
      const double r = __dsub_rn(s[c], f[fi]);
      res_u[fi] = r;
      acc[0] = fma(r, r, acc[0]);
      acc[1] = fma(f[fi], ug[3 * nd + c], acc[1]);
    }
  }
  block_partials<2>(acc, scratch, partials);
}

// w_e = u_e K_e for every element (and q_e when asked): schur_system and
// element_products (fem.py:175-180) for an arbitrary u
__global__ void __launch_bounds__(kThreads) k3_w_elem(int m, int ex, int ey, int nx, int ny,
                                                    const double* __restrict__ ug, double* __restrict__ w,
                                                    double* __restrict__ q) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    int nd[8];
    elem3_nodes(e, ex, ey, nx, ny, nd);
    double ue[24], we[24];
    gather24(ug, nd, ue);
    ke3_times(ue, we);
#pragma unroll
    for (int j = 0; j < 24; ++j) w[24 * (size_t)e + j] = we[j];
    if (q) q[e] = 0.5 * dot24(we, ue);
  }
}

// rhs_u = -res_u + scatter(t w); border = -scatter(chat w) (pbm.py:214-216, fem.py:206)
__global__ void __launch_bounds__(kThreads) k3_schur_node(int nnodes, int nx, int ny, int ex, int ey, int ez,
                                                        const double* __restrict__ w,
                                                        const double* __restrict__ tcoef,
                                                        const double* __restrict__ chat,
                                                        const double* __restrict__ res_u,
                                                        const int32_t* __restrict__ g2f, double* __restrict__ rhs,
                                                        double* __restrict__ border_free,
                                                        double* __restrict__ border_grid) {
  for (int nd = blockIdx.x * blockDim.x + threadIdx.x; nd < nnodes; nd += gridDim.x * blockDim.x) {
    const int ix = nd % nx, iy = (nd / nx) % ny, iz = nd / (nx * ny);
    const NodeElems3 ne = node_elems3(ix, iy, iz, ex, ey, ez);
    double t[3] = {0.0, 0.0, 0.0}, cb[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < ne.cnt; ++k) {
      const double* we = w + 24 * (size_t)ne.e[k] + 3 * ne.li[k];
      const double tt = tcoef[ne.e[k]], ch = chat[ne.e[k]];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        t[c] = __dadd_rn(t[c], __dmul_rn(tt, we[c]));
        cb[c] = __dadd_rn(cb[c], __dmul_rn(ch, we[c]));
      }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int fi = g2f[3 * nd + c];
      double bg = 0.0;
      if (fi >= 0) {
        rhs[fi] = __dadd_rn(-res_u[fi], t[c]);
        bg = -cb[c];
        if (border_free) border_free[fi] = bg;
      }
      border_grid[3 * nd + c] = bg;
    }
  }
}

// ---------------------------------------------------------------------------
// assembly: finest 27-point stencil (fem.py:188-209)
// ---------------------------------------------------------------------------
// one thread per (node i, neighbour b): the 3 x 3 block of rho_hat K_e +
// chat w w^T summed over the elements holding both nodes, in increasing
// element order (the reference's reduceat over the stable-sorted pattern)
__global__ void __launch_bounds__(128) k3_fine_stencil(int nx, int ny, int nz, int ex, int ey, int ez,
                                                     const double* __restrict__ w, const double* __restrict__ rho_hat,
                                                     const double* __restrict__ chat,
                                                     const uint8_t* __restrict__ fm, double* __restrict__ st) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int nn = nx * ny * nz;
  if (t >= (long long)nn * kNb3) return;
  const int nd = (int)(t / kNb3), b = (int)(t % kNb3);
  const int ix = nd % nx, iy = (nd / nx) % ny, iz = nd / (nx * ny);
  const int bx = b % 3 - 1, by = (b / 3) % 3 - 1, bz = b / 9 - 1;
  const int jx = ix + bx, jy = iy + by, jz = iz + bz;
  double blk[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  if (jx >= 0 && jx < nx && jy >= 0 && jy < ny && jz >= 0 && jz < nz) {
    const NodeElems3 ne = node_elems3(ix, iy, iz, ex, ey, ez);
    bool seen = false;
    for (int k = 0; k < ne.cnt; ++k) {
      const int li = ne.li[k];
      const int lx = (li == 1 || li == 2 || li == 5 || li == 6) ? 1 : 0;
      const int ly = (li == 2 || li == 3 || li == 6 || li == 7) ? 1 : 0;
      const int lz = li >= 4 ? 1 : 0;
      const int mx = lx + bx, my = ly + by, mz = lz + bz;
      if (mx < 0 || mx > 1 || my < 0 || my > 1 || mz < 0 || mz > 1) continue;
      const int lj = corner3(mx, my, mz);
      const int e = ne.e[k];
      const double rh = rho_hat[e], ch = chat[e];
      const double* we = w + 24 * (size_t)e;
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double v = __dadd_rn(__dmul_rn(rh, c_ke3[(3 * li + r) * 24 + 3 * lj + c]),
                                     __dmul_rn(ch, __dmul_rn(we[3 * li + r], we[3 * lj + c])));
          blk[3 * r + c] = seen ? __dadd_rn(blk[3 * r + c], v) : v;
        }
      seen = true;
    }
    const int jd = jx + nx * (jy + ny * jz);
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        if (!fm[3 * nd + r] || !fm[3 * jd + c]) blk[3 * r + c] = 0.0;  // fem.py:157-161
  }
  double* o = st + (size_t)nd * kRow3 + 9 * b;
#pragma unroll
  for (int i = 0; i < 9; ++i) o[i] = blk[i];
}

// ---------------------------------------------------------------------------
// Galerkin coarse operator (linalg.py:76-81), in the reference's order
// ---------------------------------------------------------------------------
VTS_DEVICE_INLINE double tri_weight(int d) { return d == 0 ? 1.0 : 0.5; }  // |fine - 2 coarse| in {0, 1}

// one thread per (coarse node I, coarse neighbour D): block (r, c) =
// sum_{fine i near I, increasing} P(i,I)_r [sum_{j = i + b, increasing} A(i,j)_rc P(j,J)_c]
__global__ void __launch_bounds__(128) k3_rap(int fnx, int fny, int fnz, const double* __restrict__ fst,
                                            const uint8_t* __restrict__ ffm, int cnx, int cny, int cnz,
                                            const uint8_t* __restrict__ cfm, double* __restrict__ out) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int cnn = cnx * cny * cnz;
  if (t >= (long long)cnn * kNb3) return;
  const int cn = (int)(t / kNb3), D = (int)(t % kNb3);
  const int cx = cn % cnx, cy = (cn / cnx) % cny, cz = cn / (cnx * cny);
  const int qx = cx + D % 3 - 1, qy = cy + (D / 3) % 3 - 1, qz = cz + D / 9 - 1;
  double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  if (qx >= 0 && qx < cnx && qy >= 0 && qy < cny && qz >= 0 && qz < cnz) {
    const int qn = qx + cnx * (qy + cny * qz);
    for (int oz = -1; oz <= 1; ++oz) {
      const int fz = 2 * cz + oz;
      if (fz < 0 || fz >= fnz) continue;
      for (int oy = -1; oy <= 1; ++oy) {
        const int fy = 2 * cy + oy;
        if (fy < 0 || fy >= fny) continue;
        for (int ox = -1; ox <= 1; ++ox) {
          const int fx = 2 * cx + ox;
          if (fx < 0 || fx >= fnx) continue;
          const int fi = fx + fnx * (fy + fny * fz);
          const double wI = tri_weight(ox) * tri_weight(oy) * tri_weight(oz);
          double pr[3];
#pragma unroll
          for (int r = 0; r < 3; ++r) pr[r] = (ffm[3 * fi + r] && cfm[3 * cn + r]) ? wI : 0.0;
          if (pr[0] == 0.0 && pr[1] == 0.0 && pr[2] == 0.0) continue;
          double tt[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
          const double* arow = fst + (size_t)fi * kRow3;
          for (int b = 0; b < kNb3; ++b) {
            const int jx = fx + b % 3 - 1, jy = fy + (b / 3) % 3 - 1, jz = fz + b / 9 - 1;
            const int dx = jx - 2 * qx, dy = jy - 2 * qy, dz = jz - 2 * qz;
            if (dx < -1 || dx > 1 || dy < -1 || dy > 1 || dz < -1 || dz > 1) continue;
            if (jx < 0 || jx >= fnx || jy < 0 || jy >= fny || jz < 0 || jz >= fnz) continue;
            const int fj = jx + fnx * (jy + fny * jz);
            const double wJ = tri_weight(dx < 0 ? -dx : dx) * tri_weight(dy < 0 ? -dy : dy) *
                              tri_weight(dz < 0 ? -dz : dz);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              const double pc = (ffm[3 * fj + c] && cfm[3 * qn + c]) ? wJ : 0.0;
#pragma unroll
              for (int r = 0; r < 3; ++r) tt[3 * r + c] = fma(arow[9 * b + 3 * r + c], pc, tt[3 * r + c]);
            }
          }
#pragma unroll
          for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) acc[3 * r + c] = fma(pr[r], tt[3 * r + c], acc[3 * r + c]);
        }
      }
    }
  }
  double* o = out + (size_t)cn * kRow3 + 9 * D;
#pragma unroll
  for (int i = 0; i < 9; ++i) o[i] = acc[i];
}

// (C + C^T) / 2 (linalg.py:79): block b of node i pairs with block 26 - b of node i + b, transposed
__global__ void k3_symmetrize(int nx, int ny, int nz, const double* __restrict__ raw, double* __restrict__ st) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int nn = nx * ny * nz;
  if (t >= (long long)nn * kNb3) return;
  const int nd = (int)(t / kNb3), b = (int)(t % kNb3);
  const int ix = nd % nx, iy = (nd / nx) % ny, iz = nd / (nx * ny);
  const int jx = ix + b % 3 - 1, jy = iy + (b / 3) % 3 - 1, jz = iz + b / 9 - 1;
  double* o = st + (size_t)nd * kRow3 + 9 * b;
  const double* a = raw + (size_t)nd * kRow3 + 9 * b;
  if (jx < 0 || jx >= nx || jy < 0 || jy >= ny || jz < 0 || jz >= nz) {
#pragma unroll
    for (int i = 0; i < 9; ++i) o[i] = 0.0;
    return;
  }
  const double* m = raw + (size_t)(jx + nx * (jy + ny * jz)) * kRow3 + 9 * (26 - b);
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) o[3 * r + c] = (a[3 * r + c] + m[3 * c + r]) * 0.5;
}

// ---------------------------------------------------------------------------
// transfers (mesh.py:290-342)
// ---------------------------------------------------------------------------
// vc = P^T vf (csc_matvec order: fine dofs increasing); border slot copied when bordered
__global__ void k3_restrict(int fnx, int fny, int fnz, const uint8_t* __restrict__ ffm, const double* __restrict__ vf,
                            int cnx, int cny, int cnz, const uint8_t* __restrict__ cfm, double* __restrict__ vc,
                            int bordered) {
  const int cn = blockIdx.x * blockDim.x + threadIdx.x;
  const int cnn = cnx * cny * cnz;
  if (cn > cnn) return;
  if (cn == cnn) {
    if (bordered) vc[3 * cnn] = vf[3 * fnx * fny * fnz];
    return;
  }
  const int cx = cn % cnx, cy = (cn / cnx) % cny, cz = cn / (cnx * cny);
  double s[3] = {0.0, 0.0, 0.0};
  for (int fz = 2 * cz - 1; fz <= 2 * cz + 1; ++fz) {
    if (fz < 0 || fz >= fnz) continue;
    for (int fy = 2 * cy - 1; fy <= 2 * cy + 1; ++fy) {
      if (fy < 0 || fy >= fny) continue;
      for (int fx = 2 * cx - 1; fx <= 2 * cx + 1; ++fx) {
        if (fx < 0 || fx >= fnx) continue;
        const int fi = fx + fnx * (fy + fny * fz);
        const double wv = tri_weight(abs(fx - 2 * cx)) * tri_weight(abs(fy - 2 * cy)) * tri_weight(abs(fz - 2 * cz));
#pragma unroll
        for (int c = 0; c < 3; ++c)
          if (ffm[3 * fi + c]) s[c] += wv * vf[3 * fi + c];
      }
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) vc[3 * cn + c] = cfm[3 * cn + c] ? s[c] : 0.0;
}

// xf += P xc (csr_matvec over the parents in increasing coarse index, then added);
// the border slot gets xc's (multigrid.py:134-136)
__global__ void k3_prolong(int fnx, int fny, int fnz, const uint8_t* __restrict__ ffm, double* __restrict__ xf,
                           int cnx, int cny, const uint8_t* __restrict__ cfm, const double* __restrict__ xc,
                           int cnn) {
  const int fi = blockIdx.x * blockDim.x + threadIdx.x;
  const int fnn = fnx * fny * fnz;
  if (fi > fnn) return;
  if (fi == fnn) {
    xf[3 * fnn] += xc[3 * cnn];
    return;
  }
  const int fx = fi % fnx, fy = (fi / fnx) % fny, fz = fi / (fnx * fny);
  int px[2], py[2], pz[2];
  const int nxp = (fx & 1) ? 2 : 1, nyp = (fy & 1) ? 2 : 1, nzp = (fz & 1) ? 2 : 1;
  px[0] = fx >> 1;
  px[1] = (fx >> 1) + 1;
  py[0] = fy >> 1;
  py[1] = (fy >> 1) + 1;
  pz[0] = fz >> 1;
  pz[1] = (fz >> 1) + 1;
  const double wv = ((fx & 1) ? 0.5 : 1.0) * ((fy & 1) ? 0.5 : 1.0) * ((fz & 1) ? 0.5 : 1.0);
  double s[3] = {0.0, 0.0, 0.0};
  for (int a = 0; a < nzp; ++a)
    for (int bb = 0; bb < nyp; ++bb)
      for (int d = 0; d < nxp; ++d) {
        const int cn = px[d] + cnx * (py[bb] + cny * pz[a]);
#pragma unroll
        for (int c = 0; c < 3; ++c)
          if (cfm[3 * cn + c]) s[c] += wv * xc[3 * cn + c];
      }
#pragma unroll
  for (int c = 0; c < 3; ++c)
    if (ffm[3 * fi + c]) xf[3 * fi + c] += s[c];
}

// ---------------------------------------------------------------------------
// level operator: y = A x + border x_a, y_a = border.x + corner x_a (linalg.py:56-62);
// RESID: r = b - y (multigrid.py:125)
// ---------------------------------------------------------------------------
template <bool RESID>
__global__ void __launch_bounds__(256) k3_level_apply(int nx, int ny, int nz, const double* __restrict__ st,
                                                    const double* __restrict__ border, const double* corner,
                                                    const double* __restrict__ x, const double* __restrict__ b,
                                                    double* __restrict__ y, double* partials, unsigned* counter) {
  __shared__ double scratch[256 / 32];
  const int nn = nx * ny * nz, ngrid = 3 * nn;
  const double xa = x[ngrid];
  double acc[1] = {0.0};
  for (int nd = blockIdx.x * blockDim.x + threadIdx.x; nd < nn; nd += gridDim.x * blockDim.x) {
    const int ix = nd % nx, iy = (nd / nx) % ny, iz = nd / (nx * ny);
    const double* row = st + (size_t)nd * kRow3;
    double s[3] = {0.0, 0.0, 0.0};
    for (int bz = -1; bz <= 1; ++bz) {
      if (iz + bz < 0 || iz + bz >= nz) continue;
      for (int by = -1; by <= 1; ++by) {
        if (iy + by < 0 || iy + by >= ny) continue;
        for (int bx = -1; bx <= 1; ++bx) {
          if (ix + bx < 0 || ix + bx >= nx) continue;
          const int b9 = 9 * ((bz + 1) * 9 + (by + 1) * 3 + (bx + 1));
          const double* xj = x + 3 * (nd + bx + nx * (by + ny * bz));
#pragma unroll
          for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) s[r] = fma(row[b9 + 3 * r + c], xj[c], s[r]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int gi = 3 * nd + r;
      const double bd = border[gi];
      const double v = s[r] + bd * xa;
      y[gi] = RESID ? b[gi] - v : v;
      acc[0] = fma(bd, x[gi], acc[0]);
    }
  }
  double tot[1];
  if (last_block_reduce<1>(acc, scratch, partials, counter, tot) && threadIdx.x == 0) {
    const double v = tot[0] + *corner * xa;
    y[ngrid] = RESID ? b[ngrid] - v : v;
  }
}

// ---------------------------------------------------------------------------
// lexicographic Gauss-Seidel (multigrid.py:35-64) as a row pipeline
// ---------------------------------------------------------------------------
// Rows are x pencils (iy, iz).  A sweep visits dofs in free-dof order (forward)
// or its reverse; row (iy, iz) can process column i once every earlier row it
// couples to -- (iy-1, iz) and (iy-1..iy+1, iz-1) -- has finished column i+1
// (forward; mirrored backward), because node i's earlier neighbours in those
// rows sit at columns i-1..i+1 and its later ones are not touched until this
// row passes them.  One warp per row; rows are taken by an atomic ticket in
// sweep order, so a row only ever waits on rows held by running warps.
// Lane 0 does the reference's exact arithmetic: acc = b_adj; acc -= a x for
// every off-diagonal column in CSR order; x = acc / a_ii.
template <bool FWD>
__global__ void __launch_bounds__(128) k3_gs(int nx, int ny, int nz, const double* __restrict__ st,
                                           const uint8_t* __restrict__ fm, const double* __restrict__ b,
                                           const double* __restrict__ border, double* x, unsigned* progress) {
  const int lane = threadIdx.x & 31;
  const int rows = ny * nz;
  const int ngrid = 3 * nx * ny * nz;
  unsigned* ticket = progress + rows;
  const double xa = __ldcg(x + ngrid);
  __shared__ double s_coef[4][kRow3];
  __shared__ double s_x[4][81];
  const int wslot = threadIdx.x >> 5;
  double* coef = s_coef[wslot];
  double* xs = s_x[wslot];
  for (;;) {
    unsigned t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    if ((int)t >= rows) return;
    const int row = FWD ? (int)t : rows - 1 - (int)t;
    const int iy = row % ny, iz = row / ny;
    // rows this one waits on (sweep order): same plane one row before, previous plane three rows
    int dep[4];
    int ndep = 0;
    const int sy = FWD ? -1 : 1, sz = FWD ? -1 : 1;
    if (iy + sy >= 0 && iy + sy < ny) dep[ndep++] = (iy + sy) + ny * iz;
    if (iz + sz >= 0 && iz + sz < nz)
      for (int d = -1; d <= 1; ++d)
        if (iy + d >= 0 && iy + d < ny) dep[ndep++] = (iy + d) + ny * (iz + sz);
    for (int pos = 0; pos < nx; ++pos) {
      const int ix = FWD ? pos : nx - 1 - pos;
      const int nd = ix + nx * (iy + ny * iz);
      // wait until the dependency rows passed column ix +- 1 (positions pos + 1)
      const unsigned need = (unsigned)min(pos + 2, nx);
      if (lane < ndep) {
        const volatile unsigned* pr = progress + dep[lane];
        unsigned ns = 32;
        while (*pr < need) {
          __nanosleep(ns);
          ns = min(ns * 2, 1024u);
        }
      }
      __syncwarp();
      __threadfence();
      // stage the node's stencil row and its 27 neighbours' values
      const double* row_c = st + (size_t)nd * kRow3;
      for (int i = lane; i < kRow3; i += 32) coef[i] = row_c[i];
      for (int i = lane; i < 81; i += 32) {
        const int bb = i / 3, c = i % 3;
        const int jx = ix + bb % 3 - 1, jy = iy + (bb / 3) % 3 - 1, jz = iz + bb / 9 - 1;
        double v = 0.0;
        if (jx >= 0 && jx < nx && jy >= 0 && jy < ny && jz >= 0 && jz < nz)
          v = __ldcg(x + 3 * (jx + nx * (jy + ny * jz)) + c);
        xs[i] = v;
      }
      __syncwarp();
      if (lane == 0) {
        const int order[3] = {FWD ? 0 : 2, 1, FWD ? 2 : 0};
        for (int k = 0; k < 3; ++k) {
          const int r = order[k];
          const int gi = 3 * nd + r;
          if (!fm[gi]) continue;
          // b_adj = b - border x_alpha (multigrid.py:148-149), then CSR order
          double acc = __dsub_rn(b[gi], __dmul_rn(border[gi], xa));
          double diag = 0.0;
          for (int bb = 0; bb < kNb3; ++bb) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              const double v = coef[9 * bb + 3 * r + c];
              if (bb == 13 && c == r) {
                diag = v;
              } else {
                acc = __dsub_rn(acc, __dmul_rn(v, xs[3 * bb + c]));
              }
            }
          }
          const double nv = acc / diag;
          xs[3 * 13 + r] = nv;
          x[gi] = nv;
        }
        __threadfence();
        atomicExch(progress + row, (unsigned)(pos + 1));
      }
      __syncwarp();
    }
  }
}

// coarsest bordered dense matrix (free order, border last) for k_cholesky
__global__ void k3_dense_coarse(int nx, int ny, int nz, const double* __restrict__ st,
                                const double* __restrict__ border, const int32_t* __restrict__ g2f,
                                const double* corner, int N, double* __restrict__ A) {
  const int nd = blockIdx.x * blockDim.x + threadIdx.x;
  if (nd >= nx * ny * nz) return;
  const int ix = nd % nx, iy = (nd / nx) % ny, iz = nd / (nx * ny);
  for (int r = 0; r < 3; ++r) {
    const int fi = g2f[3 * nd + r];
    if (fi < 0) continue;
    for (int b = 0; b < kNb3; ++b) {
      const int jx = ix + b % 3 - 1, jy = iy + (b / 3) % 3 - 1, jz = iz + b / 9 - 1;
      if (jx < 0 || jx >= nx || jy < 0 || jy >= ny || jz < 0 || jz >= nz) continue;
      const int jd = jx + nx * (jy + ny * jz);
      for (int c = 0; c < 3; ++c) {
        const int fj = g2f[3 * jd + c];
        if (fj < 0) continue;
        A[(size_t)fi * N + fj] = st[(size_t)nd * kRow3 + 9 * b + 3 * r + c];
      }
    }
    A[(size_t)fi * N + (N - 1)] = border[3 * nd + r];
    A[(size_t)(N - 1) * N + fi] = border[3 * nd + r];
  }
  if (nd == 0) A[(size_t)(N - 1) * N + (N - 1)] = *corner;
}

// ---------------------------------------------------------------------------
// reconstruct_nu (pbm.py:221-232): theta = w . du_e - dalpha with w = u_e K_e
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k3_recon_elem(int m, int ex, int ey, int nx, int ny,
                                                        const double* __restrict__ ug,
                                                        const double* __restrict__ dug, double dalpha,
                                                        const double* __restrict__ res_lo,
                                                        const double* __restrict__ res_up,
                                                        const double* __restrict__ a,
                                                        const double* __restrict__ b_lo,
                                                        const double* __restrict__ b_up, double* dnu_lo,
                                                        double* dnu_up, double* partials) {
  __shared__ double scratch[2 * kThreads / 32];
  double acc[2] = {0, 0};
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    int nd[8];
    elem3_nodes(e, ex, ey, nx, ny, nd);
    double ue[24], w[24], de[24];
    gather24(ug, nd, ue);
    ke3_times(ue, w);
    gather24(dug, nd, de);
    const double theta = __dsub_rn(dot24(w, de), dalpha);
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

// _al_value at the trial point (pbm.py:135-147): element part
struct Al3Args {
  int m, ex, ey, nx, ny;
  const double* ug;
  double alpha, kappa, branch;
  const double *nu_lo, *nu_up, *dnu_lo, *dnu_up, *rho, *p, *mu_lo, *mu_up, *q_lo, *q_up, *lower, *upper;
};

__global__ void __launch_bounds__(kThreads) k3_al_elem(Al3Args A, double* partials, unsigned* flags) {
  __shared__ double scratch[5 * kThreads / 32];
  double acc[5] = {0, 0, 0, 0, 0};
  unsigned sat = 0;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < A.m; e += gridDim.x * blockDim.x) {
    int nd[8];
    elem3_nodes(e, A.ex, A.ey, A.nx, A.ny, nd);
    double ue[24], w[24];
    gather24(A.ug, nd, ue);
    ke3_times(ue, w);
    const double qq = 0.5 * dot24(w, ue);
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

}  // namespace vts
