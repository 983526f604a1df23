// Preconditioned MINRES on the bound Newton matrix (unity-built).
//
// minres_solve (linalg.py:128-242) with every vector on the device in the
// grid layout and every scalar of the Lanczos/Givens recurrence in a device
// struct (MinresDev).  One iteration is a fixed launch sequence
//   scale -> apply -> lanczos(+alfa) -> axpy -> V-cycle -> givens(beta) ->
//   update(w, x) -> [verify: apply -> residual norm]
// whose kernels return immediately once the device-side `stopped` flag is
// set, so the host only polls that flag and never re-derives a scalar.
// The vector kernels fuse the reference's updates with the dot products that
// follow them (fixed-order block trees, last-block finish).

namespace vts {

// VTS_MEMCPY_STATE=1 reads the MINRES state back with a copy-engine transfer (A/B)
static bool publish_kernel() {
  static const bool on = [] {
    const char* e = getenv("VTS_MEMCPY_STATE");
    return !(e && e[0] == '1');
  }();
  return on;
}

__global__ void k_mr_scale(int len, const double* __restrict__ y, double* __restrict__ v, const MinresDev* st) {
  pdl_enter();
  if (st->stopped) return;
  const double s = 1.0 / st->beta;  // linalg.py:193-194
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) v[i] = s * y[i];
}

// y = y - (beta/oldb) r1 (iteration >= 2), alfa = v.y   (linalg.py:196-198)
__global__ void k_mr_lanczos(int len, double* __restrict__ y, const double* __restrict__ r1,
                             const double* __restrict__ v, MinresDev* st, double* partials, unsigned* counter) {
  pdl_enter();
  if (st->stopped) return;
  __shared__ double scratch[kThreads / 32];
  const bool second = st->iters >= 1;  // st->iters counts completed iterations
  const double f = second ? st->beta / st->oldb : 0.0;
  double acc[1] = {0.0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) {
    double yi = y[i];
    if (second) yi = __dsub_rn(yi, __dmul_rn(f, r1[i]));
    y[i] = yi;
    acc[0] = fma(v[i], yi, acc[0]);
  }
  double tot[1];
  if (last_block_reduce<1>(acc, scratch, partials, counter, tot) && threadIdx.x == 0) st->alfa = tot[0];
}

// y = y - (alfa/beta) r2   (linalg.py:199)
__global__ void k_mr_axpy2(int len, double* __restrict__ y, const double* __restrict__ r2, const MinresDev* st) {
  pdl_enter();
  if (st->stopped) return;
  const double f = st->alfa / st->beta;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x)
    y[i] = __dsub_rn(y[i], __dmul_rn(f, r2[i]));
}

// beta = r2.y, then the Givens update of linalg.py:203-221 (last block)
__global__ void k_mr_givens(int len, const double* __restrict__ r2, const double* __restrict__ y, MinresDev* st,
                            double* partials, unsigned* counter) {
  pdl_enter();
  if (st->stopped) return;
  __shared__ double scratch[kThreads / 32];
  double acc[1] = {0.0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x)
    acc[0] = fma(r2[i], y[i], acc[0]);
  double tot[1];
  if (last_block_reduce<1>(acc, scratch, partials, counter, tot) && threadIdx.x == 0) {
    st->oldb = st->beta;
    double beta = tot[0];
    if (beta < 0.0) {
      st->status = kIndefinite;
      st->stopped = 1;
      st->no_verify = 1;
      return;
    }
    beta = sqrt(beta);
    st->beta = beta;
    const double oldeps = st->epsln;
    const double delta = st->cs * st->dbar + st->sn * st->alfa;
    const double gbar = st->sn * st->dbar - st->cs * st->alfa;
    st->epsln = st->sn * beta;
    st->dbar = -st->cs * beta;
    const double gamma = sqrt(gbar * gbar + beta * beta);
    st->oldeps = oldeps;
    st->delta = delta;
    st->gamma = gamma;
    if (!isfinite(gamma) || gamma == 0.0) {
      st->status = kBreakdown;
      st->stopped = 1;
      st->no_verify = 1;
      return;
    }
    st->cs = gbar / gamma;
    st->sn = beta / gamma;
    st->phi = st->cs * st->phibar;
    st->phibar = st->sn * st->phibar;
  }
}

// w_new = (v - oldeps w1 - delta w2)/gamma ; x_new = x + phi w_new  (linalg.py:223-229);
// then the next iteration's v = y / beta in place (k_mr_scale's product: beta is
// already the next one, linalg.py:193-194), saving that launch
__global__ void k_mr_update(int len, double* __restrict__ v, const double* __restrict__ w1,
                            const double* __restrict__ w2, double* __restrict__ wn, const double* __restrict__ x,
                            double* __restrict__ xn, const double* __restrict__ ynext, MinresDev* st, double* partials,
                            unsigned* counter) {
  pdl_enter();
  if (st->stopped) return;
  __shared__ double scratch[kThreads / 32];
  const double oldeps = st->oldeps, delta = st->delta, gamma = st->gamma, phi = st->phi;
  const double s = 1.0 / st->beta;
  double acc[1] = {0.0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) {
    const double w = __dsub_rn(__dsub_rn(v[i], __dmul_rn(oldeps, w1[i])), __dmul_rn(delta, w2[i])) / gamma;
    v[i] = s * ynext[i];
    wn[i] = w;
    const double xv = __dadd_rn(x[i], __dmul_rn(phi, w));
    xn[i] = xv;
    if (!isfinite(xv)) acc[0] = 1.0;
  }
  double tot[1];
  if (last_block_reduce<1>(acc, scratch, partials, counter, tot) && threadIdx.x == 0) {
    st->iters += 1;
    if (tot[0] != 0.0 || !isfinite(st->phibar)) {
      st->status = kNonfinite;
      st->stopped = 1;
      st->no_verify = 1;
      return;
    }
    const double est = st->phibar / st->beta1;
    st->est = est;
    st->no_verify = (est <= st->verify_at) ? 0 : 1;
    if (st->no_verify && st->iters >= st->max_iters) {
      st->status = kCap;
      st->stopped = 1;
    }
  }
}

// The iteration's state goes into the pinned host mirror (cudaMallocHost memory is
// device-accessible under unified addressing) from a kernel, so the next iteration's
// launches stay in the programmatic-launch chain, which a copy-engine transfer breaks.
// the iteration's state into the pinned host mirror, by one thread (k_mr_verify's tail)
VTS_DEVICE_INLINE void publish_state(const MinresDev* st, MinresDev* host) {
  constexpr int kWords = sizeof(MinresDev) / 8;
  for (int i = 0; i < kWords; ++i)
    reinterpret_cast<volatile unsigned long long*>(host)[i] = reinterpret_cast<const volatile unsigned long long*>(st)[i];
  __threadfence_system();
}

// true residual after a verify apply: relres = ||b - Ax|| / ||b||  (linalg.py:231-239); with
// `host`, the iteration's final state is then published to the pinned mirror (formerly a
// separate one-block kernel: one launch less per iteration): by block 0 when there is nothing to verify, else by
// the block that finishes the residual
__global__ void k_mr_verify(int len, const double* __restrict__ b, const double* __restrict__ ax, MinresDev* st,
                            double* partials, unsigned* counter, MinresDev* host = nullptr) {
  pdl_enter();
  if (st->no_verify) {
    if (host && blockIdx.x == 0 && threadIdx.x == 0) publish_state(st, host);
    return;
  }
  __shared__ double scratch[kThreads / 32];
  double acc[1] = {0.0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) {
    const double r = b[i] - ax[i];
    acc[0] = fma(r, r, acc[0]);
  }
  double tot[1];
  if (last_block_reduce<1>(acc, scratch, partials, counter, tot) && threadIdx.x == 0) {
    const double rel = sqrt(tot[0]) / st->bnorm;
    st->relres = rel;
    st->no_verify = 1;
    if (rel <= st->tol) {
      st->status = kConverged;
      st->stopped = 1;
    } else {
      st->verify_at = st->est * fmin(0.5, st->tol / rel);
      if (st->iters >= st->max_iters) {
        st->status = kCap;
        st->stopped = 1;
      }
    }
    if (host) publish_state(st, host);
  }
}

// history hook: ||b - A x|| / ||b|| after every iteration (tests only)
__global__ void k_mr_history(int len, const double* __restrict__ b, const double* __restrict__ ax,
                             const MinresDev* st, double* hist, double* partials, unsigned* counter) {
  pdl_enter();
  __shared__ double scratch[kThreads / 32];
  double acc[1] = {0.0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) {
    const double r = b[i] - ax[i];
    acc[0] = fma(r, r, acc[0]);
  }
  double tot[1];
  if (last_block_reduce<1>(acc, scratch, partials, counter, tot) && threadIdx.x == 0)
    hist[0] = sqrt(tot[0]) / st->bnorm;
}

__global__ void k_norm2(int len, const double* __restrict__ a, double* out, double* partials, unsigned* counter) {
  __shared__ double scratch[kThreads / 32];
  double acc[1] = {0.0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x)
    acc[0] = fma(a[i], a[i], acc[0]);
  double tot[1];
  if (last_block_reduce<1>(acc, scratch, partials, counter, tot) && threadIdx.x == 0) *out = tot[0];
}

__global__ void k_resnorm(int len, const double* __restrict__ b, const double* __restrict__ ax, double* out,
                          double* partials, unsigned* counter) {
  __shared__ double scratch[kThreads / 32];
  double acc[1] = {0.0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) {
    const double r = b[i] - ax[i];
    acc[0] = fma(r, r, acc[0]);
  }
  double tot[1];
  if (last_block_reduce<1>(acc, scratch, partials, counter, tot) && threadIdx.x == 0) *out = tot[0];
}

// r = b - ax and ||r||^2 (the warm start's initial residual, linalg.py:150-152)
__global__ void k_sub_norm(int len, const double* __restrict__ b, const double* __restrict__ ax,
                           double* __restrict__ r, double* out, double* partials, unsigned* counter) {
  __shared__ double scratch[kThreads / 32];
  double acc[1] = {0.0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) {
    const double ri = b[i] - ax[i];
    r[i] = ri;
    acc[0] = fma(ri, ri, acc[0]);
  }
  double tot[1];
  if (last_block_reduce<1>(acc, scratch, partials, counter, tot) && threadIdx.x == 0) *out = tot[0];
}

// Device-side start of a solve (device_init): the checks the host path makes on
// read-back scalars (||b|| = 0, beta1 <= 0, linalg.py:144-180) are made by these two
// one-thread kernels, which set the state so that the iteration loop's launches are
// no-ops and its first status poll reports the outcome.
__global__ void k_mr_init0(const double* __restrict__ bnorm2, MinresDev* st, double tol, int cap) {
  MinresDev h{};
  h.bnorm = sqrt(*bnorm2);
  h.tol = tol;
  h.max_iters = cap;
  h.verify_at = tol;
  h.relres = INFINITY;
  h.cs = -1.0;
  h.no_verify = 1;
  h.status = kRunning;
  if (h.bnorm == 0.0) {  // x = 0 is exact (linalg.py:141-142)
    h.stopped = 1;
    h.status = kConverged;
    h.relres = 0.0;
  }
  *st = h;
}
__global__ void k_mr_init1(const double* __restrict__ beta1_sq, const int* __restrict__ chol_status, MinresDev* st) {
  if (st->stopped) return;
  if (chol_status && *chol_status != 0) {  // the (shifted) coarse factor failed: mg_setup's error
    st->status = kCholFail;
    st->stopped = 1;
    return;
  }
  const double b1 = *beta1_sq;
  if (b1 < 0.0) {
    st->status = kIndefinite;
    st->stopped = 1;
    return;
  }
  if (b1 == 0.0) {  // the start iterate is the answer; relres = ||b - A 0|| / ||b||
    st->status = kConverged;
    st->stopped = 1;
    st->relres = 1.0;
    return;
  }
  const double beta1 = sqrt(b1);
  st->beta1 = beta1;
  st->beta = beta1;
  st->phibar = beta1;
}

int minres(Ctx* c, const double* b_free, double* x_free, double tol, int max_iters, double floor_tol,
           int precondition, int* iters_out, double* relres_out, int* conv_out, double* history,
           const double* x0_free, bool device_init) {
  if (device_init && (history || x0_free || !precondition)) {
    set_error(4, "minres: the device-side start needs a preconditioned cold start without history");
    return 4;
  }
  if (!c->system_bound || (precondition && !c->mg_ready)) {
    set_error(4, "minres: bind the Newton system (and set up the multigrid) first");
    return 4;
  }
  const int F = c->L - 1;
  const int len = c->lv[F].d.ngrid + 1;
  const int grid = (int)std::min<long long>(div_up(len, kThreads), kReduceGridCap);
  double* B = c->fvec[4];
  double* pool[8] = {c->fvec[5], c->fvec[6], c->fvec[7], c->fvec[8], c->fvec[9], c->fvec[10], c->fvec[11], c->fvec[13]};
  double* W[3] = {c->fvec[1], c->fvec[2], c->fvec[3]};
  double* X[2] = {c->fvec[0], c->fvec[12]};
  double* T = c->lv[F].r;  // verify / history apply target
  if (int rc = free_to_grid(c, F, b_free, B, true)) return rc;
  k_norm2<<<grid, kThreads, 0, c->stream>>>(len, B, c->dscal + 30, c->partials, c->counters + 7);
  VTS_LAUNCHED(c);
  const int n = c->n;
  const int napi = c->unbordered ? n : n + 1;  // entries of the caller's vectors
  const int cap = max_iters > 0 ? max_iters : 3 * napi;
  double bnorm = 0.0;
  if (device_init) {
    k_mr_init0<<<1, 1, 0, c->stream>>>(c->dscal + 30, c->mst, tol, cap);
    VTS_LAUNCHED(c);
  } else {
    VTS_CUDA(cudaMemcpyAsync(c->hscal + 30, c->dscal + 30, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    VTS_CUDA(cudaStreamSynchronize(c->stream));
    bnorm = sqrt(c->hscal[30]);
  }
  if (!device_init && bnorm == 0.0) {
    VTS_CUDA(cudaMemsetAsync(x_free, 0, sizeof(double) * napi, c->stream));
    VTS_CUDA(cudaStreamSynchronize(c->stream));
    *iters_out = 0;
    *relres_out = 0.0;
    *conv_out = 1;
    return 0;
  }
  // x = x0 or 0; r1 = b - A x0 or b (linalg.py:144-152); y = M r1
  double* r1 = pool[0];
  double* y = pool[1];
  double rel0 = 1.0;  // ||b - A x|| / ||b|| at the start
  if (x0_free) {
    if (int rc = free_to_grid(c, F, x0_free, X[0], true)) return rc;
    if (int rc = newton_apply_grid(c, X[0], T, nullptr)) return rc;
    k_sub_norm<<<grid, kThreads, 0, c->stream>>>(len, B, T, r1, c->dscal + 31, c->partials, c->counters + 7);
    VTS_LAUNCHED(c);
    VTS_CUDA(cudaMemcpyAsync(c->hscal + 31, c->dscal + 31, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    VTS_CUDA(cudaStreamSynchronize(c->stream));
    rel0 = sqrt(c->hscal[31]) / bnorm;
    if (rel0 <= floor_tol) {  // the warm start already meets the floor (linalg.py:153-154)
      if (int rc = grid_to_free(c, F, X[0], x_free, true)) return rc;
      VTS_CUDA(cudaStreamSynchronize(c->stream));
      *iters_out = 0;
      *relres_out = rel0;
      *conv_out = 1;
      return 0;
    }
  } else {
    VTS_CUDA(cudaMemcpyAsync(r1, B, sizeof(double) * len, cudaMemcpyDeviceToDevice, c->stream));
    VTS_CUDA(cudaMemsetAsync(X[0], 0, sizeof(double) * len, c->stream));
  }
  if (precondition) {
    if (int rc = vcycle_grid(c, r1, y, device_init ? &c->mst->stopped : nullptr)) return rc;
  } else {
    VTS_CUDA(cudaMemcpyAsync(y, r1, sizeof(double) * len, cudaMemcpyDeviceToDevice, c->stream));
  }
  if (device_init) {
    k_dot<<<grid, kThreads, 0, c->stream>>>(len, r1, y, c->partials, c->counters + 0, c->dscal + 31,
                                            &c->mst->stopped);
    VTS_LAUNCHED(c);
    k_mr_init1<<<1, 1, 0, c->stream>>>(c->dscal + 31, c->chol_status, c->mst);
    VTS_LAUNCHED(c);
  } else {
    // beta1 = r1 . y
    k_dot<<<grid, kThreads, 0, c->stream>>>(len, r1, y, c->partials, c->counters + 0, c->dscal + 31, nullptr);
    VTS_LAUNCHED(c);
    VTS_CUDA(cudaMemcpyAsync(c->hscal + 31, c->dscal + 31, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    VTS_CUDA(cudaStreamSynchronize(c->stream));
  }
  double beta1 = device_init ? 1.0 : c->hscal[31];
  if (beta1 < 0.0 || beta1 == 0.0) {  // the start iterate is the answer (or the last sound one)
    if (int rc = grid_to_free(c, F, X[0], x_free, true)) return rc;
    VTS_CUDA(cudaStreamSynchronize(c->stream));
  }
  if (beta1 < 0.0) {
    set_error(1, "preconditioner is indefinite: <M r, r> < 0");
    return 1;
  }
  if (beta1 == 0.0) {
    *iters_out = 0;
    *relres_out = rel0;  // ||b - A x|| / ||b||
    *conv_out = 1;
    return 0;
  }
  if (!device_init) {
    beta1 = sqrt(beta1);
    MinresDev h{};
    h.beta1 = beta1;
    h.beta = beta1;
    h.oldb = 0.0;
    h.dbar = 0.0;
    h.epsln = 0.0;
    h.phibar = beta1;
    h.cs = -1.0;
    h.sn = 0.0;
    h.verify_at = tol;
    h.relres = INFINITY;
    h.tol = tol;
    h.bnorm = bnorm;
    h.iters = 0;
    h.max_iters = cap;
    h.stopped = 0;
    h.status = kRunning;
    h.no_verify = 1;
    *c->hmst = h;
    VTS_CUDA(cudaMemcpyAsync(c->mst, c->hmst, sizeof(MinresDev), cudaMemcpyHostToDevice, c->stream));
  }
  VTS_CUDA(cudaMemsetAsync(W[0], 0, sizeof(double) * len, c->stream));
  VTS_CUDA(cudaMemsetAsync(W[1], 0, sizeof(double) * len, c->stream));
  // buffers: r1 and r2 alias at the start (linalg.py:189)
  double* r2 = r1;
  double* v = pool[2];
  double* w = W[0];   // current w
  double* w2 = W[1];  // current w2
  double* wfree = W[2];
  double* x = X[0];
  double* xalt = X[1];
  std::vector<double*> freeb = {pool[3], pool[4], pool[5], pool[6], pool[7]};
  const int* stopped = &c->mst->stopped;
  const int* nover = &c->mst->no_verify;
  double* dhist = c->dscal + 32;  // latest history entry, read back every iteration
  // one iteration's launches; its update reads x_in and writes x_out
  double* x_in[2] = {nullptr, nullptr};
  double* x_out[2] = {nullptr, nullptr};
  auto enqueue = [&](int it) -> int {
    if (it == 0) {  // later iterations' v comes from the previous update
      VTS_CUDA(launch_pdl(k_mr_scale, dim3(grid), dim3(kThreads), 0, c->stream, len, y, v, c->mst));
      VTS_LAUNCHED(c);
    }
    if (int rc = newton_apply_grid(c, v, y, stopped)) return rc;
    VTS_CUDA(launch_pdl(k_mr_lanczos, dim3(grid), dim3(kThreads), 0, c->stream, len, y, r1, v, c->mst, c->partials, c->counters + 8));
    VTS_LAUNCHED(c);
    VTS_CUDA(launch_pdl(k_mr_axpy2, dim3(grid), dim3(kThreads), 0, c->stream, len, y, r2, c->mst));
    VTS_LAUNCHED(c);
    // r1 = r2 ; r2 = y ; new y buffer
    double* dead = (r1 == r2) ? nullptr : r1;
    r1 = r2;
    r2 = y;
    if (dead) freeb.push_back(dead);
    y = freeb.back();
    freeb.pop_back();
    if (precondition) {
      if (int rc = vcycle_grid(c, r2, y, stopped)) return rc;
    } else {
      VTS_CUDA(cudaMemcpyAsync(y, r2, sizeof(double) * len, cudaMemcpyDeviceToDevice, c->stream));
    }
    VTS_CUDA(launch_pdl(k_mr_givens, dim3(grid), dim3(kThreads), 0, c->stream, len, r2, y, c->mst, c->partials, c->counters + 9));
    VTS_LAUNCHED(c);
    // w1 = w2 ; w2 = w ; w = new (into the dead w1 buffer)
    double* w1 = w2;
    w2 = w;
    double* wn = wfree;
    VTS_CUDA(launch_pdl(k_mr_update, dim3(grid), dim3(kThreads), 0, c->stream, len, v, w1, w2, wn, x, xalt,
                        (const double*)y, c->mst, c->partials, c->counters + 10));
    VTS_LAUNCHED(c);
    wfree = w1;
    w = wn;
    if (history) {
      if (int rc = newton_apply_grid(c, xalt, T, nullptr)) return rc;
      VTS_CUDA(launch_pdl(k_mr_history, dim3(grid), dim3(kThreads), 0, c->stream, len, B, T, c->mst, dhist, c->partials, c->counters + 11));
      VTS_LAUNCHED(c);
    }
    if (int rc = newton_apply_grid(c, xalt, T, nover)) return rc;
    VTS_CUDA(launch_pdl(k_mr_verify, dim3(grid), dim3(kThreads), 0, c->stream, len, B, T, c->mst, c->partials, c->counters + 12,
                        publish_kernel() ? c->hmst + (it & 1) : (MinresDev*)nullptr));
    VTS_LAUNCHED(c);
    // assume the update succeeds (the next iteration reads x_out); a failed or
    // stopped iteration makes every later launch a no-op on the device
    x_in[it & 1] = x;
    x_out[it & 1] = xalt;
    std::swap(x, xalt);
    if (publish_kernel()) {
      // k_mr_verify published the state
    } else {
      VTS_CUDA(cudaMemcpyAsync(c->hmst + (it & 1), c->mst, sizeof(MinresDev), cudaMemcpyDeviceToHost, c->stream));
    }
    VTS_CUDA(cudaEventRecord(c->mr_ev[it & 1], c->stream));
    return 0;
  };
  if (!c->mr_ev[0]) {
    VTS_CUDA(cudaEventCreateWithFlags(&c->mr_ev[0], cudaEventDisableTiming));
    VTS_CUDA(cudaEventCreateWithFlags(&c->mr_ev[1], cudaEventDisableTiming));
  }
  // Iteration it+1 is enqueued before iteration it's state is read back, so the
  // host's launch latency hides behind the device's work (the history hook
  // reads back every iteration and stays synchronous).
  int status = kRunning;
  double* xfinal = x;
  int last = -1;
  if (cap > 0)
    if (int rc = enqueue(0)) return rc;
  for (int it = 0; it < cap; ++it) {
    if (!history && it + 1 < cap)
      if (int rc = enqueue(it + 1)) return rc;
    VTS_CUDA(cudaEventSynchronize(c->mr_ev[it & 1]));
    const MinresDev s = c->hmst[it & 1];
    last = it;
    if (s.status == kIndefinite || s.status == kBreakdown || s.status == kNonfinite || s.status == kCholFail) {
      status = s.status;
      xfinal = x_in[it & 1];  // the last sound iterate
      break;
    }
    xfinal = x_out[it & 1];
    if (history) {
      double hv;
      VTS_CUDA(cudaMemcpy(&hv, dhist, sizeof(double), cudaMemcpyDeviceToHost));
      history[s.iters - 1] = hv;
    }
    if (s.stopped) {
      status = s.status;
      break;
    }
    if (history && it + 1 < cap)
      if (int rc = enqueue(it + 1)) return rc;
  }
  // a look-ahead iteration behind the one that stopped ran as device no-ops
  VTS_CUDA(cudaStreamSynchronize(c->stream));
  // stopped by the device-side start (||b|| = 0 or beta1 <= 0): no update ran, the answer is x = 0
  if (device_init && last >= 0 && c->hmst[last & 1].iters == 0) xfinal = x_in[0];
  x = xfinal;
  if (last >= 0) *c->hmst = c->hmst[last & 1];
  if (status == kRunning) status = kCap;
  const MinresDev& s = *c->hmst;
  double relres = s.relres;
  if (status == kCap) {
    if (int rc = newton_apply_grid(c, x, T, nullptr)) return rc;
    k_resnorm<<<grid, kThreads, 0, c->stream>>>(len, B, T, c->dscal + 31, c->partials, c->counters + 7);
    VTS_LAUNCHED(c);
    VTS_CUDA(cudaMemcpyAsync(c->hscal + 31, c->dscal + 31, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    VTS_CUDA(cudaStreamSynchronize(c->stream));
    relres = sqrt(c->hscal[31]) / (device_init ? s.bnorm : bnorm);
  }
  if (int rc = grid_to_free(c, F, x, x_free, true)) return rc;
  *iters_out = s.iters;
  *relres_out = relres;
  *conv_out = (status == kConverged) || (status == kCap && relres <= tol);
  if (status == kIndefinite) {
    set_error(1, "preconditioner is indefinite: <M r, r> < 0");
    return 1;
  }
  if (status == kBreakdown) {
    set_error(2, "MINRES recurrence broke down");
    return 2;
  }
  if (status == kNonfinite) {
    set_error(3, "NaN/inf encountered in MINRES recurrences");
    return 3;
  }
  if (status == kCholFail) {
    set_error(6, "coarse Cholesky failed even with the shift");
    return 6;
  }
  return 0;
}

}  // namespace vts

namespace vts {

// ---------------------------------------------------------------------------
// minres_solve for an arbitrary operator / preconditioner (linalg.py:118-242):
// `a` and `precond` are host callbacks that apply the operator to a device
// vector (a CSR matrix, a dense matrix or a user callable on the reference's
// side, _as_matvec linalg.py:118-125).  The recurrences are the same device
// kernels as the bound-system solver, on plain vectors of length `len`; every
// callback runs with the context stream drained and must leave its output
// complete on return.  One state read-back per iteration (no look-ahead: the
// callbacks synchronise anyway).
// ---------------------------------------------------------------------------
int minres_generic(Ctx* c, long long len_ll, const double* b, double* x_out, const double* x0, double tol,
                   int max_iters, double floor_tol, vts_apply_fn op, vts_apply_fn prec, void* user,
                   int* iters_out, double* relres_out, int* conv_out, double* history, bool native) {
  if (!op || len_ll < 1 || len_ll > INT32_MAX) {
    set_error(4, "minres: bad operator or length");
    return 4;
  }
  const int len = (int)len_ll;
  const int grid = (int)std::min<long long>(div_up(len, kThreads), kReduceGridCap);
  double* base = nullptr;
  constexpr int kVecs = 12;
  VTS_CUDA(cudaMalloc(&base, sizeof(double) * (size_t)len * kVecs + sizeof(MinresDev) + 256));
  struct Guard {
    double* p;
    ~Guard() { cudaFree(p); }
  } guard{base};
  double* vec[kVecs];
  for (int i = 0; i < kVecs; ++i) vec[i] = base + (size_t)i * len;
  MinresDev* st = reinterpret_cast<MinresDev*>(base + (size_t)kVecs * len);
  double* r1 = vec[0];
  double* r2 = vec[1];
  double* y = vec[2];
  double* v = vec[3];
  double* w1 = vec[4];
  double* w2 = vec[5];
  double* wn = vec[6];
  double* x = vec[7];
  double* xn = vec[8];
  double* T = vec[9];
  double* spare = vec[10];
  // foreign (Python) callbacks run on other streams: drain around them; native
  // ones (the 3D operators) enqueue on the context stream, in order
  auto call = [&](vts_apply_fn fn, const double* in, double* out) -> int {
    if (!native) VTS_CUDA(cudaStreamSynchronize(c->stream));
    if (int rc = fn(user, in, out)) {
      if (!native) set_error(4, "minres: operator callback failed");
      return rc;
    }
    if (!native) VTS_CUDA(cudaDeviceSynchronize());
    return 0;
  };
  auto scalar = [&](const double* dptr) -> double {
    double h = 0.0;
    cudaMemcpyAsync(&h, dptr, sizeof(double), cudaMemcpyDeviceToHost, c->stream);
    cudaStreamSynchronize(c->stream);
    return h;
  };
  auto finish_x = [&](const double* src) -> int {
    VTS_CUDA(cudaMemcpyAsync(x_out, src, sizeof(double) * len, cudaMemcpyDeviceToDevice, c->stream));
    VTS_CUDA(cudaStreamSynchronize(c->stream));
    return 0;
  };
  k_norm2<<<grid, kThreads, 0, c->stream>>>(len, b, c->dscal + 30, c->partials, c->counters + 7);
  VTS_LAUNCHED(c);
  const double bnorm = sqrt(scalar(c->dscal + 30));
  const int cap = max_iters > 0 ? max_iters : 3 * len;
  *iters_out = 0;
  if (bnorm == 0.0) {
    VTS_CUDA(cudaMemsetAsync(x_out, 0, sizeof(double) * len, c->stream));
    VTS_CUDA(cudaStreamSynchronize(c->stream));
    *relres_out = 0.0;
    *conv_out = 1;
    return 0;
  }
  double rel0 = 1.0;
  if (x0) {
    VTS_CUDA(cudaMemcpyAsync(x, x0, sizeof(double) * len, cudaMemcpyDeviceToDevice, c->stream));
    if (int rc = call(op, x, T)) return rc;
    k_sub_norm<<<grid, kThreads, 0, c->stream>>>(len, b, T, r1, c->dscal + 31, c->partials, c->counters + 7);
    VTS_LAUNCHED(c);
    rel0 = sqrt(scalar(c->dscal + 31)) / bnorm;
    if (rel0 <= floor_tol) {
      *relres_out = rel0;
      *conv_out = 1;
      return finish_x(x);
    }
  } else {
    VTS_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * len, c->stream));
    VTS_CUDA(cudaMemcpyAsync(r1, b, sizeof(double) * len, cudaMemcpyDeviceToDevice, c->stream));
  }
  if (prec) {
    if (int rc = call(prec, r1, y)) return rc;
  } else {
    VTS_CUDA(cudaMemcpyAsync(y, r1, sizeof(double) * len, cudaMemcpyDeviceToDevice, c->stream));
  }
  k_dot<<<grid, kThreads, 0, c->stream>>>(len, r1, y, c->partials, c->counters + 0, c->dscal + 31, nullptr);
  VTS_LAUNCHED(c);
  double beta1 = scalar(c->dscal + 31);
  if (beta1 < 0.0 || beta1 == 0.0) {
    if (int rc = finish_x(x)) return rc;
  }
  if (beta1 < 0.0) {
    set_error(1, "preconditioner is indefinite: <M r, r> < 0");
    return 1;
  }
  if (beta1 == 0.0) {
    *relres_out = rel0;
    *conv_out = 1;
    return 0;
  }
  beta1 = sqrt(beta1);
  MinresDev h{};
  h.beta1 = beta1;
  h.beta = beta1;
  h.phibar = beta1;
  h.cs = -1.0;
  h.verify_at = tol;
  h.relres = INFINITY;
  h.tol = tol;
  h.bnorm = bnorm;
  h.max_iters = cap;
  h.status = kRunning;
  h.no_verify = 1;
  VTS_CUDA(cudaMemcpyAsync(st, &h, sizeof(MinresDev), cudaMemcpyHostToDevice, c->stream));
  VTS_CUDA(cudaMemsetAsync(w1, 0, sizeof(double) * len, c->stream));
  VTS_CUDA(cudaMemsetAsync(w2, 0, sizeof(double) * len, c->stream));
  VTS_CUDA(cudaStreamSynchronize(c->stream));
  // r2 aliases r1 at the start (linalg.py:189); buffers rotate like minres()
  r2 = r1;
  double* freeb[3] = {vec[1], spare, vec[11]};
  int nfree = 3;
  double* w = w2;     // current w (zero)
  double* wcur2 = w1; // current w2 (zero)
  double* wfree = wn;
  double* x_sound = x;
  MinresDev s{};
  int status = kRunning;
  for (int it = 0; it < cap; ++it) {
    if (it == 0) {  // later iterations' v comes from the previous update (k_mr_update)
      k_mr_scale<<<grid, kThreads, 0, c->stream>>>(len, y, v, st);
      VTS_LAUNCHED(c);
    }
    if (int rc = call(op, v, y)) return rc;
    k_mr_lanczos<<<grid, kThreads, 0, c->stream>>>(len, y, r1, v, st, c->partials, c->counters + 8);
    VTS_LAUNCHED(c);
    k_mr_axpy2<<<grid, kThreads, 0, c->stream>>>(len, y, r2, st);
    VTS_LAUNCHED(c);
    double* dead = (r1 == r2) ? nullptr : r1;
    r1 = r2;
    r2 = y;
    if (dead) freeb[nfree++] = dead;
    y = freeb[--nfree];
    if (prec) {
      if (int rc = call(prec, r2, y)) return rc;
    } else {
      VTS_CUDA(cudaMemcpyAsync(y, r2, sizeof(double) * len, cudaMemcpyDeviceToDevice, c->stream));
    }
    k_mr_givens<<<grid, kThreads, 0, c->stream>>>(len, r2, y, st, c->partials, c->counters + 9);
    VTS_LAUNCHED(c);
    double* wold1 = wcur2;
    wcur2 = w;
    // k_mr_update also writes the next iteration's v = y / beta
    k_mr_update<<<grid, kThreads, 0, c->stream>>>(len, v, wold1, wcur2, wfree, x, xn, (const double*)y, st,
                                                 c->partials, c->counters + 10);
    VTS_LAUNCHED(c);
    w = wfree;
    wfree = wold1;
    VTS_CUDA(cudaMemcpyAsync(&s, st, sizeof(MinresDev), cudaMemcpyDeviceToHost, c->stream));
    VTS_CUDA(cudaStreamSynchronize(c->stream));
    if (s.status == kIndefinite || s.status == kBreakdown || s.status == kNonfinite) {
      status = s.status;
      break;
    }
    std::swap(x, xn);
    x_sound = x;
    if (history || !s.no_verify) {
      if (int rc = call(op, x, T)) return rc;
    }
    if (history) {
      k_mr_history<<<grid, kThreads, 0, c->stream>>>(len, b, T, st, c->dscal + 32, c->partials, c->counters + 11);
      VTS_LAUNCHED(c);
      history[s.iters - 1] = scalar(c->dscal + 32);
    }
    if (!s.no_verify) {
      k_mr_verify<<<grid, kThreads, 0, c->stream>>>(len, b, T, st, c->partials, c->counters + 12);
      VTS_LAUNCHED(c);
      VTS_CUDA(cudaMemcpyAsync(&s, st, sizeof(MinresDev), cudaMemcpyDeviceToHost, c->stream));
      VTS_CUDA(cudaStreamSynchronize(c->stream));
    }
    if (s.stopped) {
      status = s.status;
      break;
    }
  }
  if (status == kRunning) status = kCap;
  double relres = s.relres;
  if (status == kCap) {
    if (int rc = call(op, x_sound, T)) return rc;
    k_resnorm<<<grid, kThreads, 0, c->stream>>>(len, b, T, c->dscal + 31, c->partials, c->counters + 7);
    VTS_LAUNCHED(c);
    relres = sqrt(scalar(c->dscal + 31)) / bnorm;
  }
  if (int rc = finish_x(x_sound)) return rc;
  *iters_out = s.iters;
  *relres_out = relres;
  *conv_out = (status == kConverged) || (status == kCap && relres <= tol);
  if (status == kIndefinite) {
    set_error(1, "preconditioner is indefinite: <M r, r> < 0");
    return 1;
  }
  if (status == kBreakdown) {
    set_error(2, "MINRES recurrence broke down");
    return 2;
  }
  if (status == kNonfinite) {
    set_error(3, "NaN/inf encountered in MINRES recurrences");
    return 3;
  }
  return 0;
}

}  // namespace vts
