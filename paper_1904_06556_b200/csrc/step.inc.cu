// Device-resident Newton step of newton_inner (pbm.py:273-325), unity-built into
// vts_b200.cu.
//
// The host-orchestrated step (paper_1904_06556_b200/pbm.py) reads a scalar back
// after nearly every call: the corner of the Schur system, the coarse factor's
// status, ||b|| and beta1 at the start of MINRES, the slope, every Armijo trial
// value, and the evaluation at the new point -- eight or more stream
// synchronisations per step, each one leaving the GPU idle while the host turns
// around.  Here every decision those read-backs fed is taken on the device:
//
//   * the scalars the kernels consume (alpha, res_alpha, dalpha, kappa) live in a
//     device struct (StepDev) and are read through pointers;
//   * the coarse factor's shifted retry is enqueued behind a device flag
//     (mg_setup's device_gate);
//   * MINRES starts without read-backs (minres' device_init); its loop still polls
//     one pinned status block per iteration, which never stalls the stream;
//   * slope, sufficient-decrease test and step halving are one-thread kernels; the
//     trial evaluations after the decision and the state update / evaluation before
//     it are skipped through device flags.
//
// The host synchronises once after the MINRES loop (twice when the line search
// needs more than kTrialsPerPass trials).  The two flag-free phases -- Newton
// system + Galerkin hierarchy + coarse factor, and reconstruction + slope +
// trials + update + evaluation -- are captured as CUDA graphs and replayed while
// the caller's buffers stay the same.  (The V-cycle inside MINRES is not: its
// overlap flags carry host-counted epochs, which a replayed graph would repeat.)
// Every kernel is the host path's, so both paths compute the same bits
// (tests/test_gpu_step.py).

namespace vts {

struct StepDev {
  double alpha, value, res_alpha;  // state alpha; the evaluation the step starts from
  double dalpha, slope, kappa, trial;
  double c1, shrink;               // PbmConfig.armijo_c1 / armijo_shrink
  int max_halvings;                // PbmConfig.armijo_max_halvings
  int ntrials;                     // trial values evaluated
  int search_done;                 // accepted, exhausted or no descent: trials are skipped
  int no_update;                   // the state update and the new evaluation are skipped
  int status;                      // 0 step taken, 1 non-descent direction, 2 line search exhausted
  int pad;
};

struct StepHost {  // pinned; written by k_step_publish, read after the synchronisation
  StepDev sd;
  double scalars[8];  // eval_lagrangian's scalars at the new point
  unsigned flags;     // saturation during the step
  int retry;          // the coarse factor needed the shift
};

struct GraphSlot {
  cudaGraphExec_t exec = nullptr;
  std::vector<uintptr_t> key;
  long long launches = 0;  // kernels one replay launches
};

struct StepState {
  StepDev* dev = nullptr;
  StepHost* host = nullptr;  // pinned
  cudaStream_t cap = nullptr;  // capture stream (the context stream may be the legacy stream)
  GraphSlot setup, post;
  ~StepState() {
    if (setup.exec) cudaGraphExecDestroy(setup.exec);
    if (post.exec) cudaGraphExecDestroy(post.exec);
    if (cap) cudaStreamDestroy(cap);
    if (host) cudaFreeHost(host);
    if (dev) cudaFree(dev);
  }
};

constexpr int kTrialsPerPass = 2;  // trial values enqueued before the host looks (kappa = 1 is the rule)

__global__ void k_step_dalpha(const double* __restrict__ du, int n, StepDev* sd) { sd->dalpha = du[n]; }

// slope = res_u.du + res_alpha dalpha + res_lo.dnu_lo + res_up.dnu_up (pbm.py:290-295),
// summed exactly as reconstruct_nu's host side does (element partials in block order)
__global__ void k_step_slope(int nb, const double* __restrict__ pe, const double* __restrict__ dot, StepDev* sd) {
  double s_lo = 0.0, s_up = 0.0;
  for (int b = 0; b < nb; ++b) {
    s_lo = __dadd_rn(s_lo, pe[2 * b]);
    s_up = __dadd_rn(s_up, pe[2 * b + 1]);
  }
  const double slope = __dadd_rn(__dadd_rn(__dadd_rn(*dot, __dmul_rn(sd->res_alpha, sd->dalpha)), s_lo), s_up);
  sd->slope = slope;
  sd->kappa = 1.0;
  sd->ntrials = 0;
  sd->no_update = 1;
  if (slope >= 0.0) {  // pbm.py:296-297
    sd->status = 1;
    sd->search_done = 1;
  } else {
    sd->status = 0;
    sd->search_done = 0;
  }
}

// one sufficient-decrease test and halving (pbm.py:299-318), in Python's operation order
__global__ void k_step_armijo(const double* __restrict__ trial, StepDev* sd) {
  if (sd->search_done) return;
  const double t = *trial;
  sd->trial = t;
  sd->ntrials += 1;
  if (t <= __dadd_rn(sd->value, __dmul_rn(__dmul_rn(sd->c1, sd->kappa), sd->slope))) {
    sd->search_done = 1;
    sd->no_update = 0;
    return;
  }
  sd->kappa = __dmul_rn(sd->kappa, sd->shrink);
  if (sd->ntrials >= sd->max_halvings + 1) {
    sd->status = 2;
    sd->search_done = 1;
  }
}

// state.alpha + kappa * dalpha (pbm.py:321)
__global__ void k_step_alpha(StepDev* sd) {
  if (sd->no_update) return;
  sd->alpha = __dadd_rn(sd->alpha, __dmul_rn(sd->kappa, sd->dalpha));
}

__global__ void k_step_publish(const StepDev* __restrict__ sd, const double* __restrict__ scal,
                               const unsigned* __restrict__ flags, const int* __restrict__ retry, StepHost* host) {
  volatile StepHost* h = host;
  if (threadIdx.x == 0) {
    const unsigned long long* s = reinterpret_cast<const unsigned long long*>(sd);
    volatile unsigned long long* d = reinterpret_cast<volatile unsigned long long*>(&host->sd);
    static_assert(sizeof(StepDev) % 8 == 0, "copied in 8-byte words");
    for (int i = 0; i < (int)(sizeof(StepDev) / 8); ++i) d[i] = s[i];
    for (int i = 0; i < 8; ++i) h->scalars[i] = scal[i];
    h->flags = *flags;
    h->retry = *retry;
  }
  __threadfence_system();
}

static bool step_graphs_enabled() {
  static const bool on = [] {
    const char* e = getenv("VTS_NO_GRAPH");
    return !(e && e[0] == '1');
  }();
  return on;
}

// Runs `enqueue` on the context stream through a CUDA graph captured the first time
// (and whenever `key` -- every pointer and scalar baked into the launches -- changes).
template <class F>
static int run_graph(Ctx* c, GraphSlot& g, const std::vector<uintptr_t>& key, int* graphs, F&& enqueue) {
  if (!step_graphs_enabled()) return enqueue();
  StepState& S = *c->step;
  if (!g.exec || g.key != key) {
    if (g.exec) {
      VTS_CUDA(cudaGraphExecDestroy(g.exec));
      g.exec = nullptr;
    }
    if (!S.cap) VTS_CUDA(cudaStreamCreateWithFlags(&S.cap, cudaStreamNonBlocking));
    cudaStream_t saved = c->stream;
    const long long l0 = c->launches;
    c->stream = S.cap;
    VTS_CUDA(cudaStreamBeginCapture(S.cap, cudaStreamCaptureModeThreadLocal));
    const int rc = enqueue();
    cudaGraph_t graph = nullptr;
    const cudaError_t e = cudaStreamEndCapture(S.cap, &graph);
    c->stream = saved;
    g.launches = c->launches - l0;
    c->launches = l0;
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    VTS_CUDA(e);
    const cudaError_t ei = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    VTS_CUDA(ei);
    g.key = key;
  }
  VTS_CUDA(cudaGraphLaunch(g.exec, c->stream));
  c->launches += g.launches;
  ++*graphs;
  return 0;
}

static uintptr_t as_key(const void* p) { return reinterpret_cast<uintptr_t>(p); }
static uintptr_t as_key(double v) {
  uintptr_t u;
  std::memcpy(&u, &v, sizeof(u));
  return u;
}

int newton_step(Ctx* c, const vts_newton_step_args* a, vts_newton_step_result* r) {
  if (c->dim != 2) {
    set_error(4, "vts_newton_step: the device-resident step is built for the 2D context");
    return 4;
  }
  if (!a->u || !a->nu_lo || !a->nu_up || !a->rho || !a->p || !a->mu_lo || !a->mu_up || !a->q_lo || !a->q_up ||
      !a->f || !a->lower || !a->upper || !a->res_u || !a->res_lo || !a->res_up || !a->q || !a->mu_hat_lo ||
      !a->mu_hat_up || !a->a || !a->b_lo || !a->b_up || !a->rho_hat || !a->chat || !a->rhs || !a->border ||
      !a->du || !a->dnu_lo || !a->dnu_up || !r) {
    set_error(4, "vts_newton_step: NULL argument");
    return 4;
  }
  if (!(a->minres_tol > 0.0 && a->minres_tol < 1.0) || a->minres_cap < 0 || a->armijo_max_halvings < 0) {
    set_error(4, "vts_newton_step: bad controls");
    return 4;
  }
  if (!c->step) {
    c->step = new StepState();
    VTS_CUDA(cudaMalloc(&c->step->dev, sizeof(StepDev)));
    VTS_CUDA(cudaMallocHost(&c->step->host, sizeof(StepHost)));
  }
  StepState& S = *c->step;
  std::memset(r, 0, sizeof(*r));
  const int F = c->L - 1;
  const LevelDev& d = c->lv[F].d;
  StepDev* sd = S.dev;

  // the step's inputs: the caller's alpha and the evaluation it starts from
  {
    StepDev h{};
    h.alpha = a->alpha;
    h.value = a->value;
    h.res_alpha = a->res_alpha;
    h.c1 = a->armijo_c1;
    h.shrink = a->armijo_shrink;
    h.max_halvings = a->armijo_max_halvings;
    h.search_done = 1;
    h.no_update = 1;
    S.host->sd = h;
    VTS_CUDA(cudaMemcpyAsync(sd, &S.host->sd, sizeof(StepDev), cudaMemcpyHostToDevice, c->stream));
    VTS_CUDA(cudaMemsetAsync(c->dflags, 0, sizeof(unsigned), c->stream));
  }

  // 1. schur_system + MgPreconditioner.__init__ (pbm.py:280-281)
  const std::vector<uintptr_t> key1 = {as_key(a->u), as_key(a->res_u), as_key(a->res_lo), as_key(a->res_up),
                                       as_key(a->a), as_key(a->b_lo), as_key(a->b_up), as_key(a->rho_hat),
                                       as_key(a->chat), as_key(a->rhs), as_key(a->border), as_key(a->shift_scale)};
  if (int rc = run_graph(c, S.setup, key1, &r->graphs, [&]() -> int {
        if (int rc2 = schur_system(c, a->u, a->res_u, 0.0, a->res_lo, a->res_up, a->a, a->b_lo, a->b_up,
                                   a->rho_hat, a->chat, a->rhs, a->border, nullptr, &sd->res_alpha))
          return rc2;
        return mg_setup(c, a->shift_scale, true);
      }))
    return rc;
  c->system_bound = true;
  c->border_flip = false;
  c->unbordered = false;
  c->mg_ready = true;

  // 2. minres_solve (pbm.py:283-286): device-side start, status polled per iteration
  int iters = 0, conv = 0;
  double relres = 0.0;
  const int mrc = minres(c, a->rhs, a->du, a->minres_tol, a->minres_cap, a->minres_floor, 1, &iters, &relres,
                         &conv, nullptr, nullptr, true);
  r->minres_iterations = iters;
  r->minres_relres = relres;
  r->minres_converged = conv;
  if (mrc) return mrc;  // MINRES error (the last sound iterate is in du) or the coarse factor failed

  // 3. reconstruct_nu + slope, the Armijo trials, the update and the new evaluation (pbm.py:287-325)
  const int ge = reduce_grid(c->m);
  auto trials = [&]() -> int {
    double* ug = c->fvec[0];
    for (int t = 0; t < kTrialsPerPass; ++t) {
      k_trial_grid<<<reduce_grid(d.ngrid), kThreads, 0, c->stream>>>(
          d.ngrid, c->lv[F].grid2free, a->u, a->du, 0.0, a->f, ug, c->partials + kMaxBlocks * 8, c->counters + 2,
          c->dscal + 10, &sd->kappa, &sd->search_done);
      VTS_LAUNCHED(c);
      AlElemArgs A{c->m, d.ex, d.nx, ug, 0.0, 0.0, a->branch, a->nu_lo, a->nu_up, a->dnu_lo, a->dnu_up, a->rho,
                   a->p, a->mu_lo, a->mu_up, a->q_lo, a->q_up, a->lower, a->upper, &sd->alpha, &sd->kappa,
                   &sd->dalpha, &sd->search_done};
      k_al_elem<<<ge, kThreads, 0, c->stream>>>(A, c->partials, c->dflags);
      VTS_LAUNCHED(c);
      k_al_finish<<<1, kThreads, 0, c->stream>>>(ge, c->partials, c->dscal + 10, 0.0, a->volume, c->dscal + 24,
                                                  &sd->alpha, &sd->kappa, &sd->dalpha, &sd->search_done);
      VTS_LAUNCHED(c);
      k_step_armijo<<<1, 1, 0, c->stream>>>(c->dscal + 24, sd);
      VTS_LAUNCHED(c);
    }
    return 0;
  };
  auto update_and_eval = [&]() -> int {
    const int* skip = &sd->no_update;
    k_axpy<<<reduce_grid(c->n), kThreads, 0, c->stream>>>(c->n, 0.0, a->du, a->u, &sd->kappa, skip);
    VTS_LAUNCHED(c);
    k_step_alpha<<<1, 1, 0, c->stream>>>(sd);
    VTS_LAUNCHED(c);
    k_axpy<<<reduce_grid(c->m), kThreads, 0, c->stream>>>(c->m, 0.0, a->dnu_lo, a->nu_lo, &sd->kappa, skip);
    VTS_LAUNCHED(c);
    k_axpy<<<reduce_grid(c->m), kThreads, 0, c->stream>>>(c->m, 0.0, a->dnu_up, a->nu_up, &sd->kappa, skip);
    VTS_LAUNCHED(c);
    double scal[8];
    if (int rc = eval_lagrangian(c, a->u, 0.0, a->nu_lo, a->nu_up, a->rho, a->mu_lo, a->mu_up, a->p, a->q_lo,
                                 a->q_up, a->f, a->lower, a->upper, a->volume, a->norm_f, a->norm_bounds, a->branch,
                                 a->res_u, a->res_lo, a->res_up, a->q, a->mu_hat_lo, a->mu_hat_up, a->a, a->b_lo,
                                 a->b_up, a->rho_hat, nullptr, scal, nullptr, &sd->alpha, skip))
      return rc;
    k_step_publish<<<1, 32, 0, c->stream>>>(sd, c->dscal, c->dflags, c->chol_retry, S.host);
    VTS_LAUNCHED(c);
    return 0;
  };
  const std::vector<uintptr_t> key2 = {
      as_key(a->u), as_key(a->nu_lo), as_key(a->nu_up), as_key(a->rho), as_key(a->p), as_key(a->mu_lo),
      as_key(a->mu_up), as_key(a->q_lo), as_key(a->q_up), as_key(a->f), as_key(a->lower), as_key(a->upper),
      as_key(a->volume), as_key(a->norm_f), as_key(a->norm_bounds), as_key(a->branch), as_key(a->res_u),
      as_key(a->res_lo), as_key(a->res_up), as_key(a->q), as_key(a->mu_hat_lo), as_key(a->mu_hat_up),
      as_key(a->a), as_key(a->b_lo), as_key(a->b_up), as_key(a->rho_hat), as_key(a->du), as_key(a->dnu_lo),
      as_key(a->dnu_up)};
  if (int rc = run_graph(c, S.post, key2, &r->graphs, [&]() -> int {
        k_step_dalpha<<<1, 1, 0, c->stream>>>(a->du, c->n, sd);
        VTS_LAUNCHED(c);
        double* ug = c->fvec[0];
        double* dug = c->fvec[2];
        if (int rc2 = free_to_grid(c, F, a->u, ug, false)) return rc2;
        if (int rc2 = free_to_grid(c, F, a->du, dug, false)) return rc2;
        k_recon_elem<<<ge, kThreads, 0, c->stream>>>(c->m, d.ex, d.nx, ug, dug, 0.0, a->res_lo, a->res_up, a->a,
                                                      a->b_lo, a->b_up, a->dnu_lo, a->dnu_up, c->partials,
                                                      &sd->dalpha);
        VTS_LAUNCHED(c);
        k_dot<<<reduce_grid(c->n), kThreads, 0, c->stream>>>(c->n, a->res_u, a->du, c->partials + kMaxBlocks * 8,
                                                              c->counters + 1, c->dscal + 8, nullptr);
        VTS_LAUNCHED(c);
        k_step_slope<<<1, 1, 0, c->stream>>>(ge, c->partials, c->dscal + 8, sd);
        VTS_LAUNCHED(c);
        if (int rc2 = trials()) return rc2;
        return update_and_eval();
      }))
    return rc;
  VTS_CUDA(cudaStreamSynchronize(c->stream));
  r->host_syncs = 1;
  // a search that needs more trials: the next ones (skipped once decided), then the
  // update and evaluation again (skipped unless this pass accepts)
  while (!S.host->sd.search_done) {
    if (int rc = trials()) return rc;
    if (int rc = update_and_eval()) return rc;
    VTS_CUDA(cudaStreamSynchronize(c->stream));
    r->host_syncs += 1;
  }
  const StepHost& H = *S.host;
  r->status = H.sd.status;
  r->kappa = H.sd.kappa;
  r->slope = H.sd.slope;
  r->dalpha = H.sd.dalpha;
  r->alpha = H.sd.alpha;
  r->trials = H.sd.ntrials;
  for (int i = 0; i < 8; ++i) r->scalars[i] = H.scalars[i];
  c->shifted = H.retry;
  r->warnings = (H.flags ? VTS_W_SATURATED : 0u) | (H.retry ? VTS_W_SHIFTED : 0u);
  return 0;
}

}  // namespace vts
