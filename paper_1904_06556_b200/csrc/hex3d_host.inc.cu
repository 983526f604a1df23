// Host drivers of the 3D hexahedral path (kernels in hex3d.inc.cu).  Included
// by vts_b200.cu after the arena/pool helpers; each function mirrors its 2D
// counterpart and the same reference function (cited there).

namespace vts {

static int h3_create(Ctx** out, int levels, const int32_t* ex, const int32_t* ey, const int32_t* ez,
                     const int64_t* const* dof_maps, const double* ke, int64_t stream) {
  if (levels < 1 || !ex || !ey || !ez || !dof_maps || !ke || !out) {
    set_error(VTS_E_ARGUMENT, "vts_ctx_create3: bad arguments");
    return VTS_E_ARGUMENT;
  }
  for (int k = 0; k < levels; ++k) {
    if (ex[k] < 1 || ey[k] < 1 || ez[k] < 1) {
      set_error(VTS_E_ARGUMENT, "vts_ctx_create3: element counts must be positive");
      return VTS_E_ARGUMENT;
    }
    if (k > 0 && (ex[k] != 2 * ex[k - 1] || ey[k] != 2 * ey[k - 1] || ez[k] != 2 * ez[k - 1])) {
      set_error(VTS_E_ARGUMENT, "vts_ctx_create3: each level must refine the previous one by 2 per axis");
      return VTS_E_ARGUMENT;
    }
  }
  Ctx* c = new Ctx();
  c->dim = 3;
  c->hex = new Hex();
  c->L = levels;
  c->stream = reinterpret_cast<cudaStream_t>(stream);
  {
    std::lock_guard<std::mutex> lock(g_ke_mutex);
    ++g_stream_refs[c->stream];
  }
  Hex& H = *c->hex;
  std::memcpy(H.ke, ke, sizeof(double) * 576);
  H.lv.resize(levels);
  auto fail = [&](int rc) {
    free_ctx(c);
    return rc;
  };
  // host maps first (validated), then one arena
  std::vector<std::vector<uint8_t>> masks(levels);
  std::vector<std::vector<int32_t>> g2f(levels), f2g(levels);
  for (int k = 0; k < levels; ++k) {
    Level3& L = H.lv[k];
    L.ex = ex[k];
    L.ey = ey[k];
    L.ez = ez[k];
    L.nx = L.ex + 1;
    L.ny = L.ey + 1;
    L.nz = L.ez + 1;
    L.nnodes = L.nx * L.ny * L.nz;
    L.ngrid = 3 * L.nnodes;
    masks[k].assign(L.ngrid, 0);
    g2f[k].assign(L.ngrid, -1);
    int nfree = 0;
    for (int i = 0; i < L.ngrid; ++i) {
      const int64_t d = dof_maps[k][i];
      if (d >= 0) {
        if (d != nfree) {
          set_error(VTS_E_ARGUMENT, "vts_ctx_create3: dof map must number free dofs node-major in order");
          return fail(VTS_E_ARGUMENT);
        }
        masks[k][i] = 1;
        g2f[k][i] = nfree++;
        f2g[k].push_back(i);
      }
    }
    if (nfree == 0) {
      set_error(VTS_E_ARGUMENT, "vts_ctx_create3: a level has no free dofs");
      return fail(VTS_E_ARGUMENT);
    }
    L.nfree = nfree;
  }
  const Level3& F = H.lv[levels - 1];
  c->n = F.nfree;
  c->m = F.ex * F.ey * F.ez;
  c->N0 = H.lv[0].nfree + 1;
  Arena arena;
  for (int k = 0; k < levels; ++k) {
    Level3& L = H.lv[k];
    dalloc(arena, &L.fmask, (size_t)L.ngrid);
    dalloc(arena, &L.g2f, (size_t)L.ngrid);
    dalloc(arena, &L.f2g, (size_t)L.nfree);
    dalloc(arena, &L.st, (size_t)L.nnodes * kRow3);
    dalloc(arena, &L.border, (size_t)L.ngrid + 1);
    dalloc(arena, &L.b, (size_t)L.ngrid + 1);
    dalloc(arena, &L.x, (size_t)L.ngrid + 1);
    dalloc(arena, &L.r, (size_t)L.ngrid + 1);
    dalloc(arena, &L.progress, (size_t)L.ny * L.nz + 1);
  }
  const size_t len = (size_t)F.ngrid + 1;
  dalloc(arena, &H.w, (size_t)c->m * 24);
  dalloc(arena, &H.u_grid, len);
  for (double*& g : H.g) dalloc(arena, &g, std::max(len, (size_t)c->m + 1));
  dalloc(arena, &H.rap_tmp, levels > 1 ? (size_t)H.lv[levels - 2].nnodes * kRow3 : 1);
  dalloc(arena, &c->rho_hat, (size_t)c->m);
  dalloc(arena, &c->chat, (size_t)c->m);
  dalloc(arena, &c->d_corner, 1);
  dalloc(arena, &c->chol, (size_t)c->N0 * c->N0);
  dalloc(arena, &c->chol_rdiag, (size_t)c->N0);
  dalloc(arena, &c->chol_status, 1);
  dalloc(arena, &c->partials, (size_t)kMaxBlocks * kMaxPartials);
  dalloc(arena, &c->counters, 64);
  dalloc(arena, &c->dscal, 64);
  dalloc(arena, &c->dflags, 4);
  dalloc(arena, &c->mst, 1);
  if (arena.commit(c)) return fail(VTS_E_CUDA);
  for (int k = 0; k < levels; ++k) {
    Level3& L = H.lv[k];
    if (cudaMemcpy(L.fmask, masks[k].data(), L.ngrid, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(L.g2f, g2f[k].data(), sizeof(int32_t) * L.ngrid, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(L.f2g, f2g[k].data(), sizeof(int32_t) * L.nfree, cudaMemcpyHostToDevice) != cudaSuccess) {
      set_error(VTS_E_CUDA, "vts_ctx_create3: device upload failed");
      return fail(VTS_E_CUDA);
    }
  }
  if (!(c->hscal = static_cast<double*>(pinned_acquire()))) {
    set_error(VTS_E_CUDA, "vts_ctx_create3: pinned allocation failed");
    return fail(VTS_E_CUDA);
  }
  c->hmst = reinterpret_cast<MinresDev*>(c->hscal + 64);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    set_error(VTS_E_CUDA, "vts_ctx_create3: device synchronisation failed");
    return fail(VTS_E_CUDA);
  }
  *out = c;
  return 0;
}

static int h3_free_to_grid(Ctx* c, int k, const double* src, double* dst, bool bordered) {
  const Level3& L = c->hex->lv[k];
  k_free_to_grid<<<div_up(L.ngrid + 1, kThreads), kThreads, 0, c->stream>>>(L.ngrid, L.nfree, L.g2f, src, dst,
                                                                          border_mode(c, bordered));
  VTS_LAUNCHED(c);
  return 0;
}

static int h3_grid_to_free(Ctx* c, int k, const double* src, double* dst, bool bordered) {
  const Level3& L = c->hex->lv[k];
  k_grid_to_free<<<div_up(L.nfree + 1, kThreads), kThreads, 0, c->stream>>>(L.nfree, L.ngrid, L.f2g, src, dst,
                                                                          border_mode(c, bordered));
  VTS_LAUNCHED(c);
  return 0;
}

static int h3_eval_lagrangian(Ctx* c, const double* u, double alpha, const double* nu_lo, const double* nu_up,
                              const double* rho, const double* mu_lo, const double* mu_up, const double* p,
                              const double* q_lo, const double* q_up, const double* f, const double* lower,
                              const double* upper, double volume, double norm_f, double norm_bounds, double branch,
                              double* res_u, double* res_lo, double* res_up, double* q, double* mu_hat_lo,
                              double* mu_hat_up, double* a, double* b_lo, double* b_up, double* rho_hat,
                              double* w_out, double* scalars, unsigned* warn) {
  Hex& H = *c->hex;
  const int F = c->L - 1;
  const Level3& L = H.lv[F];
  double* ug = H.g[0];
  if (int rc = h3_free_to_grid(c, F, u, ug, false)) return rc;
  VTS_CUDA(cudaMemsetAsync(c->dflags, 0, sizeof(unsigned), c->stream));
  Phi3Args A{c->m, L.ex, L.ey, L.nx, L.ny, ug, alpha, branch, nu_lo, nu_up, rho, mu_lo, mu_up, p, q_lo, q_up,
             lower, upper, q, rho_hat, mu_hat_lo, mu_hat_up, a, b_lo, b_up, res_lo, res_up, H.w};
  const int ge = reduce_grid(c->m);
  k3_phi_elem<<<ge, kThreads, 0, c->stream>>>(A, c->partials, c->dflags);
  VTS_LAUNCHED(c);
  const int gn = reduce_grid(L.nnodes);
  double* pn = c->partials + kMaxBlocks * 8;
  k3_phi_node<<<gn, kThreads, 0, c->stream>>>(L.nnodes, L.nx, L.ny, L.ex, L.ey, L.ez, ug, H.w, rho_hat, f, L.g2f,
                                               res_u, pn);
  VTS_LAUNCHED(c);
  k_phi_finish<<<1, kThreads, 0, c->stream>>>(ge, c->partials, gn, pn, alpha, volume, norm_f, norm_bounds, c->dscal);
  VTS_LAUNCHED(c);
  if (w_out)
    VTS_CUDA(cudaMemcpyAsync(w_out, H.w, sizeof(double) * 24 * (size_t)c->m, cudaMemcpyDeviceToDevice, c->stream));
  VTS_CUDA(cudaMemcpyAsync(c->hscal + 16, c->dflags, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
  if (int rc = sync_scalars(c, 8)) return rc;
  for (int i = 0; i < 8; ++i) scalars[i] = c->hscal[i];
  if (warn) *warn = *reinterpret_cast<unsigned*>(c->hscal + 16) ? 1u : 0u;
  return 0;
}

static int h3_fine_stencil(Ctx* c) {
  Hex& H = *c->hex;
  const Level3& L = H.lv[c->L - 1];
  const long long work = (long long)L.nnodes * kNb3;
  k3_fine_stencil<<<div_up(work, 128), 128, 0, c->stream>>>(L.nx, L.ny, L.nz, L.ex, L.ey, L.ez, H.w, c->rho_hat,
                                                             c->chat, L.fmask, L.st);
  VTS_LAUNCHED(c);
  return 0;
}

static int h3_schur_system(Ctx* c, const double* u, const double* res_u, double res_alpha, const double* res_lo,
                           const double* res_up, const double* a, const double* b_lo, const double* b_up,
                           const double* rho_hat, double* chat, double* rhs, double* border, double* corner) {
  Hex& H = *c->hex;
  const int F = c->L - 1;
  const Level3& L = H.lv[F];
  if (int rc = h3_free_to_grid(c, F, u, H.u_grid, false)) return rc;
  k3_w_elem<<<reduce_grid(c->m), kThreads, 0, c->stream>>>(c->m, L.ex, L.ey, L.nx, L.ny, H.u_grid, H.w, nullptr);
  VTS_LAUNCHED(c);
  double* tcoef = H.g[1];
  const int ge = reduce_grid(c->m);
  k_schur_elem<<<ge, kThreads, 0, c->stream>>>(c->m, a, b_lo, b_up, res_lo, res_up, rho_hat, chat, c->chat,
                                                c->rho_hat, tcoef, c->partials);
  VTS_LAUNCHED(c);
  k3_schur_node<<<reduce_grid(L.nnodes), kThreads, 0, c->stream>>>(L.nnodes, L.nx, L.ny, L.ex, L.ey, L.ez, H.w,
                                                                    tcoef, c->chat, res_u, L.g2f, rhs, border,
                                                                    L.border);
  VTS_LAUNCHED(c);
  k_schur_finish<<<1, kThreads, 0, c->stream>>>(ge, c->partials, res_alpha, 1.0, c->n, rhs, c->d_corner, c->dscal);
  VTS_LAUNCHED(c);
  // the reference assembles S here (pbm.py:215, fem.py:188-209): the finest stencil
  if (int rc = h3_fine_stencil(c)) return rc;
  if (int rc = sync_scalars(c, 2)) return rc;
  c->corner = c->hscal[0];
  if (corner) *corner = c->corner;
  c->system_bound = true;
  c->border_flip = false;
  c->unbordered = false;
  c->mg_ready = false;
  return 0;
}

static int h3_bind_stiffness(Ctx* c, const double* rho, unsigned* warn) {
  Hex& H = *c->hex;
  const Level3& L = H.lv[c->L - 1];
  VTS_CUDA(cudaMemsetAsync(H.w, 0, sizeof(double) * 24 * (size_t)c->m, c->stream));
  VTS_CUDA(cudaMemsetAsync(L.border, 0, sizeof(double) * (L.ngrid + 1), c->stream));
  VTS_CUDA(cudaMemsetAsync(c->dflags, 0, sizeof(unsigned), c->stream));
  k_bind_stiffness<<<div_up(c->m, kThreads), kThreads, 0, c->stream>>>(c->m, rho, c->rho_hat, c->chat, c->d_corner,
                                                                       c->dflags);
  VTS_LAUNCHED(c);
  if (int rc = h3_fine_stencil(c)) return rc;
  unsigned flags = 0;
  VTS_CUDA(cudaMemcpyAsync(&flags, c->dflags, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
  VTS_CUDA(cudaStreamSynchronize(c->stream));
  if (warn) *warn = flags;
  c->corner = 1.0;
  c->system_bound = true;
  c->border_flip = false;
  c->unbordered = true;
  c->mg_ready = false;
  return 0;
}

static int h3_element_products(Ctx* c, const double* u, double* w, double* q) {
  Hex& H = *c->hex;
  const int F = c->L - 1;
  const Level3& L = H.lv[F];
  double* ug = H.g[0];
  if (int rc = h3_free_to_grid(c, F, u, ug, false)) return rc;
  // without a caller buffer the products land in the context's element array
  // (only read while a system is assembled, which this call does not do)
  k3_w_elem<<<reduce_grid(c->m), kThreads, 0, c->stream>>>(c->m, L.ex, L.ey, L.nx, L.ny, ug, w ? w : H.w, q);
  VTS_LAUNCHED(c);
  return 0;
}

// y = A_k x (bordered grid vectors); RESID: r = b - A_k x
template <bool RESID>
static int h3_apply(Ctx* c, int k, const double* x, const double* b, double* y) {
  const Level3& L = c->hex->lv[k];
  const int grid = (int)std::min<long long>(div_up(L.nnodes, 256), kReduceGridCap);
  k3_level_apply<RESID><<<grid, 256, 0, c->stream>>>(L.nx, L.ny, L.nz, L.st, L.border, c->d_corner, x, b, y,
                                                      c->partials, c->counters + 5);
  VTS_LAUNCHED(c);
  return 0;
}

static int h3_gs(Ctx* c, int k, const double* b, double* x, bool forward) {
  const Level3& L = c->hex->lv[k];
  const int rows = L.ny * L.nz;
  VTS_CUDA(cudaMemsetAsync(L.progress, 0, sizeof(unsigned) * (rows + 1), c->stream));
  const int blocks = std::max(1, std::min(div_up(rows, 4), 148 * 8));
  if (forward)
    k3_gs<true><<<blocks, 128, 0, c->stream>>>(L.nx, L.ny, L.nz, L.st, L.fmask, b, L.border, x, L.progress);
  else
    k3_gs<false><<<blocks, 128, 0, c->stream>>>(L.nx, L.ny, L.nz, L.st, L.fmask, b, L.border, x, L.progress);
  VTS_LAUNCHED(c);
  return 0;
}

static int h3_mg_setup(Ctx* c, double shift_scale) {
  if (!c->system_bound) {
    set_error(4, "mg_setup: no Newton system bound (call vts_schur_system first)");
    return 4;
  }
  Hex& H = *c->hex;
  for (int k = c->L - 1; k >= 1; --k) {
    const Level3& F = H.lv[k];
    const Level3& C = H.lv[k - 1];
    const long long work = (long long)C.nnodes * kNb3;
    k3_rap<<<div_up(work, 128), 128, 0, c->stream>>>(F.nx, F.ny, F.nz, F.st, F.fmask, C.nx, C.ny, C.nz, C.fmask,
                                                     H.rap_tmp);
    VTS_LAUNCHED(c);
    k3_symmetrize<<<div_up(work, 128), 128, 0, c->stream>>>(C.nx, C.ny, C.nz, H.rap_tmp, C.st);
    VTS_LAUNCHED(c);
    k3_restrict<<<div_up(C.nnodes + 1, 256), 256, 0, c->stream>>>(F.nx, F.ny, F.nz, F.fmask, F.border, C.nx, C.ny,
                                                                  C.nz, C.fmask, C.border, 0);
    VTS_LAUNCHED(c);
  }
  const Level3& C = H.lv[0];
  const int N = c->N0;
  auto build = [&](double shift_now) -> int {
    VTS_CUDA(cudaMemsetAsync(c->chol, 0, sizeof(double) * N * N, c->stream));
    k3_dense_coarse<<<div_up(C.nnodes, 128), 128, 0, c->stream>>>(C.nx, C.ny, C.nz, C.st, C.border, C.g2f,
                                                                   c->d_corner, N, c->chol);
    VTS_LAUNCHED(c);
    if (shift_now != 0.0) {
      k_add_shift<<<1, 1024, 0, c->stream>>>(N, shift_now, c->chol, c->dscal + 20);
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
  k_chol_rdiag<<<1, 256, 0, c->stream>>>(c->N0, c->chol, c->chol_rdiag);
  VTS_LAUNCHED(c);
  c->mg_ready = true;
  return 0;
}

// one V(2,2) cycle from a zero guess (multigrid.py:109-143), grid vectors
static int h3_cycle(Ctx* c, int k, const double* b, double* x) {
  Hex& H = *c->hex;
  const Level3& L = H.lv[k];
  const int top = c->L - 1;
  if (k == 0) {
    VTS_CUDA(launch_pdl(k_coarse_solve, dim3(1), dim3(1024), sizeof(double) * c->N0, c->stream, c->N0, L.nfree,
                        L.ngrid, (const double*)c->chol, (const double*)c->chol_rdiag, (const int32_t*)L.f2g, b, x,
                        (const int*)nullptr));
    VTS_LAUNCHED(c);
    return 0;
  }
  VTS_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * L.ngrid, c->stream));
  VTS_CUDA(launch_pdl(k_alpha_init, dim3(1), dim3(1), 0, c->stream, L.ngrid, b, x, (const double*)c->d_corner,
                      k == top ? 1 : 0, (const int*)nullptr));
  VTS_LAUNCHED(c);
  if (int rc = h3_gs(c, k, b, x, true)) return rc;
  if (int rc = h3_gs(c, k, b, x, true)) return rc;
  if (int rc = h3_apply<true>(c, k, x, b, L.r)) return rc;
  const Level3& C = H.lv[k - 1];
  k3_restrict<<<div_up(C.nnodes + 1, 256), 256, 0, c->stream>>>(L.nx, L.ny, L.nz, L.fmask, L.r, C.nx, C.ny, C.nz,
                                                                 C.fmask, C.b, 1);
  VTS_LAUNCHED(c);
  if (int rc = h3_cycle(c, k - 1, C.b, C.x)) return rc;
  k3_prolong<<<div_up(L.nnodes + 1, 256), 256, 0, c->stream>>>(L.nx, L.ny, L.nz, L.fmask, x, C.nx, C.ny, C.fmask,
                                                               C.x, C.nnodes);
  VTS_LAUNCHED(c);
  if (int rc = h3_gs(c, k, b, x, false)) return rc;
  if (int rc = h3_gs(c, k, b, x, false)) return rc;
  if (k == top) {
    const int grid = (int)std::min<long long>(div_up(L.ngrid, 256), kReduceGridCap);
    VTS_CUDA(launch_pdl(k_alpha_relax, dim3(grid), dim3(256), 0, c->stream, L.ngrid, (const double*)L.border, b, x,
                        (const double*)c->d_corner, c->partials, c->counters + 6, (const int*)nullptr));
    VTS_LAUNCHED(c);
  }
  return 0;
}

static int h3_vcycle_grid(Ctx* c, const double* b, double* z) {
  if (!c->mg_ready) {
    set_error(VTS_E_ARGUMENT, "vts_vcycle: multigrid not set up");
    return VTS_E_ARGUMENT;
  }
  return h3_cycle(c, c->L - 1, b, z);
}

// native operator callbacks for minres_generic (grid vectors, context stream)
static int h3_op_cb(void* user, const double* in, double* out) {
  Ctx* c = static_cast<Ctx*>(user);
  return h3_apply<false>(c, c->L - 1, in, nullptr, out);
}

static int h3_prec_cb(void* user, const double* in, double* out) {
  return h3_vcycle_grid(static_cast<Ctx*>(user), in, out);
}

static int h3_minres(Ctx* c, const double* b_free, double* x_free, const double* x0_free, double tol, int max_iters,
                     double floor_tol, int precondition, int* it, double* rel, int* conv, double* history) {
  if (!c->system_bound || (precondition && !c->mg_ready)) {
    set_error(4, "minres: bind the Newton system (and set up the multigrid) first");
    return 4;
  }
  Hex& H = *c->hex;
  const int F = c->L - 1;
  const Level3& L = H.lv[F];
  const long long len = L.ngrid + 1;
  double* B = H.g[4];
  double* X0 = x0_free ? H.g[5] : nullptr;
  if (int rc = h3_free_to_grid(c, F, b_free, B, true)) return rc;
  if (X0)
    if (int rc = h3_free_to_grid(c, F, x0_free, X0, true)) return rc;
  double* X = L.x;  // the top level's V-cycle buffers are unused (its b / z are the callers')
  const int cap = max_iters > 0 ? max_iters : 3 * (c->unbordered ? c->n : c->n + 1);
  const int rc = minres_generic(c, len, B, X, X0, tol, cap, floor_tol, h3_op_cb, precondition ? h3_prec_cb : nullptr,
                                c, it, rel, conv, history, true);
  if (rc == 0 || rc == 1 || rc == 2 || rc == 3) {
    if (int rc2 = h3_grid_to_free(c, F, X, x_free, true)) return rc2;
    VTS_CUDA(cudaStreamSynchronize(c->stream));
  }
  return rc;
}

static int h3_reconstruct_nu(Ctx* c, const double* u, const double* du, double dalpha, const double* res_u,
                             double res_alpha, const double* res_lo, const double* res_up, const double* a,
                             const double* b_lo, const double* b_up, double* dnu_lo, double* dnu_up, double* slope) {
  Hex& H = *c->hex;
  const int F = c->L - 1;
  const Level3& L = H.lv[F];
  double* ug = H.g[0];
  double* dug = H.g[2];
  if (int rc = h3_free_to_grid(c, F, u, ug, false)) return rc;
  if (int rc = h3_free_to_grid(c, F, du, dug, false)) return rc;
  const int ge = reduce_grid(c->m);
  k3_recon_elem<<<ge, kThreads, 0, c->stream>>>(c->m, L.ex, L.ey, L.nx, L.ny, ug, dug, dalpha, res_lo, res_up, a,
                                                 b_lo, b_up, dnu_lo, dnu_up, c->partials);
  VTS_LAUNCHED(c);
  k_dot<<<reduce_grid(c->n), kThreads, 0, c->stream>>>(c->n, res_u, du, c->partials + kMaxBlocks * 8,
                                                        c->counters + 1, c->dscal + 8, nullptr);
  VTS_LAUNCHED(c);
  if (slope) {
    std::vector<double> pe(2 * ge);
    VTS_CUDA(cudaMemcpyAsync(pe.data(), c->partials, sizeof(double) * 2 * ge, cudaMemcpyDeviceToHost, c->stream));
    if (int rc = sync_scalars(c, 9)) return rc;
    double s_lo = 0.0, s_up = 0.0;
    for (int b = 0; b < ge; ++b) {
      s_lo += pe[2 * b];
      s_up += pe[2 * b + 1];
    }
    *slope = ((c->hscal[8] + res_alpha * dalpha) + s_lo) + s_up;
  } else {
    VTS_CUDA(cudaStreamSynchronize(c->stream));
  }
  return 0;
}

static int h3_al_value(Ctx* c, const double* u, double alpha, const double* nu_lo, const double* nu_up,
                       const double* du, double dalpha, const double* dnu_lo, const double* dnu_up, double kappa,
                       const double* rho, const double* p, const double* mu_lo, const double* mu_up,
                       const double* q_lo, const double* q_up, const double* f, const double* lower,
                       const double* upper, double volume, double branch, double* value, unsigned* warn) {
  Hex& H = *c->hex;
  const int F = c->L - 1;
  const Level3& L = H.lv[F];
  double* ug = H.g[0];
  k_trial_grid<<<reduce_grid(L.ngrid), kThreads, 0, c->stream>>>(L.ngrid, L.g2f, u, du, kappa, f, ug,
                                                                  c->partials + kMaxBlocks * 8, c->counters + 2,
                                                                  c->dscal + 10);
  VTS_LAUNCHED(c);
  VTS_CUDA(cudaMemsetAsync(c->dflags, 0, sizeof(unsigned), c->stream));
  volatile double kd = kappa * dalpha;  // state.alpha + kappa * dalpha, two roundings (pbm.py:301)
  const double alpha_t = alpha + kd;
  Al3Args A{c->m, L.ex, L.ey, L.nx, L.ny, ug, alpha_t, kappa, branch, nu_lo, nu_up, dnu_lo, dnu_up, rho, p,
            mu_lo, mu_up, q_lo, q_up, lower, upper};
  const int ge = reduce_grid(c->m);
  k3_al_elem<<<ge, kThreads, 0, c->stream>>>(A, c->partials, c->dflags);
  VTS_LAUNCHED(c);
  k_al_finish<<<1, kThreads, 0, c->stream>>>(ge, c->partials, c->dscal + 10, alpha_t, volume, c->dscal);
  VTS_LAUNCHED(c);
  VTS_CUDA(cudaMemcpyAsync(c->hscal + 16, c->dflags, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
  if (int rc = sync_scalars(c, 1)) return rc;
  *value = c->hscal[0];
  if (warn) *warn = *reinterpret_cast<unsigned*>(c->hscal + 16) ? 1u : 0u;
  return 0;
}

// API-edge wrappers with the 2D entry points' conventions (free vectors, synchronous)
static int h3_newton_apply(Ctx* c, const double* x, double* y) {
  if (!c->system_bound) {
    set_error(VTS_E_ARGUMENT, "vts_newton_apply: no Newton system bound");
    return VTS_E_ARGUMENT;
  }
  Hex& H = *c->hex;
  const int F = c->L - 1;
  if (int rc = h3_free_to_grid(c, F, x, H.g[2], true)) return rc;
  if (int rc = h3_apply<false>(c, F, H.g[2], nullptr, H.g[3])) return rc;
  if (int rc = h3_grid_to_free(c, F, H.g[3], y, true)) return rc;
  VTS_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

static int h3_vcycle(Ctx* c, const double* b, double* z) {
  Hex& H = *c->hex;
  const int F = c->L - 1;
  if (int rc = h3_free_to_grid(c, F, b, H.g[2], true)) return rc;
  if (int rc = h3_vcycle_grid(c, H.g[2], H.g[3])) return rc;
  if (int rc = h3_grid_to_free(c, F, H.g[3], z, true)) return rc;
  VTS_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

static int h3_level_apply(Ctx* c, int k, const double* x, double* y) {
  if (k < 0 || k >= c->L || !c->mg_ready) {
    set_error(VTS_E_ARGUMENT, "vts_level_apply: bad level or multigrid not set up");
    return VTS_E_ARGUMENT;
  }
  const Level3& L = c->hex->lv[k];
  if (int rc = h3_free_to_grid(c, k, x, L.b, true)) return rc;
  if (int rc = h3_apply<false>(c, k, L.b, nullptr, L.r)) return rc;
  if (int rc = h3_grid_to_free(c, k, L.r, y, true)) return rc;
  VTS_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

}  // namespace vts
