// DOC reuse: the damped optimality-criteria method of
// the reference (doc.py:111-208) on the Newton step's device machinery.
//
//  * bind_stiffness  K(rho) = sum_e rho_e K_e (fem.py:211-219) bound as the
//                    bordered system [[K, 0], [0, 1]] (zero border, unit corner),
//                    so the matrix-free apply, the Galerkin hierarchy, the V-cycle
//                    and MINRES run unchanged; the border slot of every vector
//                    stays exactly zero, so the core iterates are those of the
//                    unbordered solve (multigrid.py:82-90 with border None)
//  * element_energy  w_e = u_e K_e, q_e = u_e . w_e / 2 (fem.py:175-180)
//  * doc_bisect      the clamped multiplicative update and the volume bisection
//                    (doc.py:63-108) in ONE cooperative launch: every bisection
//                    step is a grid-wide sum (block partials, grid barrier, every
//                    block folds the partials in the same fixed order, so all
//                    blocks take the same branch with no broadcast)
//  * doc_measure     max |rho+ - rho|, f.u and the closed-form best-alpha gap
//                    (doc.py:150-155, model.py:69-98; the kink scan sorts the
//                    element energies with CUB's radix sort)

#include <cooperative_groups.h>
#include <cub/cub.cuh>

namespace vts {

namespace cg = cooperative_groups;

__global__ void k_bind_stiffness(int m, const double* __restrict__ rho, double* __restrict__ rho_hat,
                                 double* __restrict__ chat, double* d_corner, unsigned* flags) {
  unsigned neg = 0;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    const double r = rho[e];
    rho_hat[e] = r;
    chat[e] = 0.0;
    neg |= (r < 0.0) ? 1u : 0u;
  }
  if (neg) atomicOr(flags, 1u);
  if (blockIdx.x == 0 && threadIdx.x == 0) *d_corner = 1.0;
}

int bind_stiffness(Ctx* c, const double* rho, unsigned* warn) {
  const int F = c->L - 1;
  const LevelBuf& L = c->lv[F];
  VTS_CUDA(cudaMemsetAsync(c->u_grid, 0, sizeof(double) * (L.d.ngrid + 1), c->stream));
  VTS_CUDA(cudaMemsetAsync(L.d.border, 0, sizeof(double) * (L.d.ngrid + 1), c->stream));
  VTS_CUDA(cudaMemsetAsync(c->dflags, 0, sizeof(unsigned), c->stream));
  k_bind_stiffness<<<div_up(c->m, kThreads), kThreads, 0, c->stream>>>(c->m, rho, c->rho_hat, c->chat,
                                                                       c->d_corner, c->dflags);
  VTS_LAUNCHED(c);
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

// w_e = u_e K_e and q_e = 1/2 u_e . w_e, in k_phi_elem's order (fem.py:175-180)
__global__ void k_elem_energy(int m, int ex, int nx, const double* __restrict__ ug, double* __restrict__ w_out,
                              double* __restrict__ q) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    int nd[4];
    elem_nodes(e, ex, nx, nd);
    double ue[8], w[8];
    gather8(ug, nd, ue);
    ke_times(ue, w);
    double qq = w[0] * ue[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) qq = fma(w[i], ue[i], qq);
    q[e] = 0.5 * qq;
    if (w_out) {
#pragma unroll
      for (int j = 0; j < 8; j += 2)
        *reinterpret_cast<double2*>(w_out + 8 * (size_t)e + j) = make_double2(w[j], w[j + 1]);
    }
  }
}

int element_energy(Ctx* c, const double* u, double* w, double* q) {
  const int F = c->L - 1;
  const LevelDev& d = c->lv[F].d;
  double* ug = c->fvec[10];
  if (int rc = free_to_grid(c, F, u, ug, false)) return rc;
  k_elem_energy<<<div_up(c->m, kThreads), kThreads, 0, c->stream>>>(c->m, d.ex, d.nx, ug, w, q);
  VTS_LAUNCHED(c);
  return 0;
}

// doc_update (doc.py:63-75): clip(rho_e * z_e^q / alpha, lower_e, upper_e); z_e is the
// input times zscale (2 when the input is q_e and z = 2 q, doc.py:149 -- exact either
// way); numpy's z**0.5 is a square root, z**1 the identity
VTS_DEVICE_INLINE double doc_value(double rho, double zin, double zscale, double lo, double up, double alpha,
                                   double expo) {
  const double z = zscale * zin;
  const double zq = expo == 0.5 ? sqrt(z) : (expo == 1.0 ? z : pow(z, expo));
  double v = (rho * zq) / alpha;
  v = (v < lo) ? lo : v;  // np.maximum then np.minimum; NaN propagates
  v = (v > up) ? up : v;
  return v;
}

struct DocBisectArgs {
  int m;
  const double *rho, *q, *lower, *upper;
  double zscale, volume, expo, alpha_hi, tol;
  int cap;
  double* partials;  // [2 * gridDim.x]
  double* out;       // alpha, status, steps, total at alpha
};

// grid-wide sum of doc_value(alpha): block partials -> grid barrier -> every
// block folds the partials in block order (identical result everywhere)
__device__ double doc_total(const DocBisectArgs& A, double alpha, int buf, double* scratch, cg::grid_group& g) {
  double acc[1] = {0.0};
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < A.m; e += gridDim.x * blockDim.x)
    acc[0] += doc_value(A.rho[e], A.q[e], A.zscale, A.lower[e], A.upper[e], alpha, A.expo);
  block_sum<1>(acc, scratch);
  double* part = A.partials + (size_t)buf * gridDim.x;
  if (threadIdx.x == 0) part[blockIdx.x] = acc[0];
  g.sync();
  double t[1] = {0.0};
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) t[0] += __ldcg(part + b);
  block_sum<1>(t, scratch);
  __shared__ double s_total;
  if (threadIdx.x == 0) s_total = t[0];
  __syncthreads();
  return s_total;
}

// bisect_volume (doc.py:78-108); status 0 ok, 1 bracket invalid, 2 not closed in cap steps
__global__ void __launch_bounds__(kThreads) k_doc_bisect(DocBisectArgs A) {
  cg::grid_group g = cg::this_grid();
  __shared__ double scratch[kThreads / 32];
  double hi = A.alpha_hi, lo = 0.0;
  int buf = 0;
  const double total_hi = doc_total(A, hi, buf, scratch, g);
  buf ^= 1;
  if (total_hi > A.volume) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      A.out[0] = hi;
      A.out[1] = 1.0;
      A.out[2] = 0.0;
      A.out[3] = total_hi;
    }
    return;
  }
  double alpha = hi, last_total = total_hi;
  int steps = 0, closed = 0;
  for (int it = 0; it < A.cap; ++it) {
    if ((hi - lo) / (hi + lo) <= A.tol) {
      closed = 1;
      break;
    }
    alpha = 0.5 * (hi + lo);
    last_total = doc_total(A, alpha, buf, scratch, g);
    buf ^= 1;
    ++steps;
    if (last_total > A.volume) lo = alpha;
    else hi = alpha;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    A.out[0] = alpha;  // the last alpha tried: its update is the returned design
    A.out[1] = closed ? 0.0 : 2.0;
    A.out[2] = (double)steps;
    A.out[3] = last_total;
  }
}

// the update at one multiplier: `alpha_dev` (device, the bisection's result) or `alpha`
__global__ void k_doc_apply(int m, const double* __restrict__ rho, const double* __restrict__ z, double zscale,
                            const double* __restrict__ lower, const double* __restrict__ upper,
                            const double* __restrict__ alpha_dev, double alpha, double expo,
                            double* __restrict__ rho_new) {
  const double al = alpha_dev ? alpha_dev[0] : alpha;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x)
    rho_new[e] = doc_value(rho[e], z[e], zscale, lower[e], upper[e], al, expo);
}

int doc_update(Ctx* c, const double* rho, const double* z, double zscale, double alpha, double exponent,
               const double* lower, const double* upper, double* rho_new) {
  k_doc_apply<<<div_up(c->m, kThreads), kThreads, 0, c->stream>>>(c->m, rho, z, zscale, lower, upper, nullptr, alpha,
                                                                   exponent, rho_new);
  VTS_LAUNCHED(c);
  return 0;
}

int doc_bisect(Ctx* c, const double* rho, const double* q, double zscale, const double* lower,
               const double* upper, double volume, double exponent, double alpha_hi, double tol, int cap,
               double* rho_new, double* alpha_out, int* status) {
  static int max_blocks = 0;
  if (!max_blocks) {
    int per_sm = 0, dev = 0, sms = 0;
    VTS_CUDA(cudaGetDevice(&dev));
    VTS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    VTS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_doc_bisect, kThreads, 0));
    max_blocks = std::max(1, per_sm * sms);
  }
  const int grid = std::max(1, std::min(max_blocks, std::min(div_up(c->m, kThreads), kMaxBlocks / 2)));
  DocBisectArgs A{c->m, rho, q, lower, upper, zscale, volume, exponent, alpha_hi, tol, cap, c->partials,
                  c->dscal + 40};
  void* args[] = {&A};
  VTS_CUDA(cudaLaunchCooperativeKernel((const void*)k_doc_bisect, dim3(grid), dim3(kThreads), args, 0, c->stream));
  VTS_LAUNCHED(c);
  k_doc_apply<<<div_up(c->m, kThreads), kThreads, 0, c->stream>>>(c->m, rho, q, zscale, lower, upper, c->dscal + 40,
                                                                   0.0, exponent, rho_new);
  VTS_LAUNCHED(c);
  VTS_CUDA(cudaMemcpyAsync(c->hscal + 40, c->dscal + 40, sizeof(double) * 4, cudaMemcpyDeviceToHost, c->stream));
  VTS_CUDA(cudaStreamSynchronize(c->stream));
  *alpha_out = c->hscal[40];
  *status = (int)c->hscal[41];
  return 0;
}

// ---------------------------------------------------------------------------
// doc_measure: step size, f.u and best_alpha_gap (doc.py:150-155, model.py:69-98)
// ---------------------------------------------------------------------------
// max |rho+ - rho| (doc.py:150), f.u and sum(rho+).  The max of non-negative doubles is the
// max of their bit patterns as integers (NaN sorts above inf, so it propagates
// like np.max): one atomicMax per block, order-free; f.u is the usual fixed tree.
__global__ void k_doc_step_fu(int m, int n, const double* __restrict__ rho_new, const double* __restrict__ rho,
                              const double* __restrict__ f, const double* __restrict__ u, double* partials,
                              unsigned* counter, unsigned long long* step_bits, double* sums) {
  __shared__ double scratch[2 * kThreads / 32];
  __shared__ unsigned long long smax;
  if (threadIdx.x == 0) smax = 0ull;
  __syncthreads();
  unsigned long long mx = 0ull;
  double acc[2] = {0.0, 0.0};  // f.u, sum(rho_new)
  const int len = max(m, n);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) {
    if (i < m) {
      const unsigned long long b = __double_as_longlong(fabs(rho_new[i] - rho[i]));
      mx = b > mx ? b : mx;
      acc[1] += rho_new[i];
    }
    if (i < n) acc[0] = fma(f[i], u[i], acc[0]);
  }
  atomicMax(&smax, mx);
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(step_bits, smax);
  double tot[2];
  if (last_block_reduce<2>(acc, scratch, partials, counter, tot) && threadIdx.x == 0) {
    sums[0] = tot[0];
    sums[1] = tot[1];
  }
}

__global__ void k_iota(int m, int* __restrict__ idx, int* first, unsigned long long* step_bits) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *first = INT32_MAX;
    *step_bits = 0ull;
  }
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) idx[e] = e;
}

__global__ void k_gather2(int m, const int* __restrict__ order, const double* __restrict__ lo,
                          const double* __restrict__ up, double* __restrict__ lo_s, double* __restrict__ up_s) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
    const int e = order[j];
    lo_s[j] = lo[e];
    up_s[j] = up[e];
  }
}

// first kink j with volume - (cumsum(lo)_j + (sum(up) - cumsum(up)_j)) >= 0 (argmax of
// the boolean; 0 when none), model.py:89-97
__global__ void k_first_kink(int m, double volume, const double* __restrict__ clo, const double* __restrict__ cup,
                             int* first) {
  const double upsum = cup[m - 1];
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
    const double deriv = volume - (clo[j] + (upsum - cup[j]));
    if (deriv >= 0.0) atomicMin(first, j);
  }
}

// duality_gap(alpha, q, fu) (model.py:69-79) with alpha = q_sorted[j*]
__global__ void k_doc_gap(int m, const double* __restrict__ q, const double* __restrict__ q_sorted,
                          const int* __restrict__ first, const double* __restrict__ lo,
                          const double* __restrict__ up, const double* __restrict__ fu_ptr, double volume,
                          double* partials, unsigned* counter, double* out) {
  __shared__ double scratch[kThreads / 32];
  const int j = (*first < m) ? *first : 0;
  const double alpha = q_sorted[j];
  double acc[1] = {0.0};
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    const double slack = alpha - q[e];
    acc[0] += fmin(lo[e] * slack, up[e] * slack);
  }
  double tot[1];
  if (last_block_reduce<1>(acc, scratch, partials, counter, tot) && threadIdx.x == 0) {
    out[0] = (-0.5 * fu_ptr[0] + alpha * volume) - tot[0];
    out[1] = alpha;
  }
}

int doc_measure(Ctx* c, const double* rho_new, const double* rho, const double* q, const double* u,
                const double* f, const double* lower, const double* upper, double volume, double* out5) {
  const int m = c->m;
  if (!c->doc_ws) {
    size_t tmp_sort = 0, tmp_scan = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_sort, (const double*)nullptr, (double*)nullptr,
                                    (const int*)nullptr, (int*)nullptr, m);
    cub::DeviceScan::InclusiveSum(nullptr, tmp_scan, (const double*)nullptr, (double*)nullptr, m);
    c->doc_tmp_bytes = std::max(tmp_sort, tmp_scan);
    const size_t bytes = (size_t)m * (3 * sizeof(double) + 2 * sizeof(double) + 2 * sizeof(int)) +
                         c->doc_tmp_bytes + 1024;
    VTS_CUDA(cudaMalloc(&c->doc_ws, bytes));
  }
  char* p = static_cast<char*>(c->doc_ws);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) & ~size_t(255);
    return r;
  };
  double* q_s = reinterpret_cast<double*>(take(sizeof(double) * m));
  double* lo_s = reinterpret_cast<double*>(take(sizeof(double) * m));
  double* up_s = reinterpret_cast<double*>(take(sizeof(double) * m));
  double* clo = reinterpret_cast<double*>(take(sizeof(double) * m));
  double* cup = reinterpret_cast<double*>(take(sizeof(double) * m));
  int* idx = reinterpret_cast<int*>(take(sizeof(int) * m));
  int* order = reinterpret_cast<int*>(take(sizeof(int) * m));
  int* first = reinterpret_cast<int*>(take(sizeof(int)));
  void* tmp = take(c->doc_tmp_bytes);
  const int n = c->n;
  unsigned long long* step_bits = reinterpret_cast<unsigned long long*>(c->dscal + 44);
  k_iota<<<div_up(m, kThreads), kThreads, 0, c->stream>>>(m, idx, first, step_bits);
  VTS_LAUNCHED(c);
  k_doc_step_fu<<<reduce_grid(std::max(m, n)), kThreads, 0, c->stream>>>(m, n, rho_new, rho, f, u, c->partials,
                                                                          c->counters + 13, step_bits, c->dscal + 45);
  VTS_LAUNCHED(c);
  size_t tb = c->doc_tmp_bytes;
  VTS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, q, q_s, idx, order, m, 0, 64, c->stream));
  k_gather2<<<div_up(m, kThreads), kThreads, 0, c->stream>>>(m, order, lower, upper, lo_s, up_s);
  VTS_LAUNCHED(c);
  tb = c->doc_tmp_bytes;
  VTS_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, lo_s, clo, m, c->stream));
  tb = c->doc_tmp_bytes;
  VTS_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, up_s, cup, m, c->stream));
  k_first_kink<<<div_up(m, kThreads), kThreads, 0, c->stream>>>(m, volume, clo, cup, first);
  VTS_LAUNCHED(c);
  k_doc_gap<<<reduce_grid(m), kThreads, 0, c->stream>>>(m, q, q_s, first, lower, upper, c->dscal + 45, volume,
                                                        c->partials, c->counters + 14, c->dscal + 47);
  VTS_LAUNCHED(c);
  VTS_CUDA(cudaMemcpyAsync(c->hscal + 44, c->dscal + 44, sizeof(double) * 5, cudaMemcpyDeviceToHost, c->stream));
  VTS_CUDA(cudaStreamSynchronize(c->stream));
  out5[0] = c->hscal[44];  // max |rho+ - rho|
  out5[1] = c->hscal[45];  // f.u
  out5[2] = c->hscal[47];  // best-alpha duality gap
  out5[3] = c->hscal[48];  // its alpha
  out5[4] = c->hscal[46];  // sum(rho+)
  return 0;
}

}  // namespace vts
