// Host-side context of the B200 PBM Newton step: mesh hierarchy, device
// workspace, the bound Newton matrix and the multigrid hierarchy built from it.
#pragma once

#include <cstdio>
#include <string>
#include <utility>
#include <vector>

#include "vts_common.cuh"

struct VtsError {
  int code;
  std::string msg;
};

namespace vts {

struct LevelBuf {
  LevelDev d{};
  int32_t* grid2free = nullptr;  // [ngrid] free index or -1
  double* b = nullptr;           // [ngrid + 1] V-cycle right-hand side
  double* x = nullptr;           // [ngrid + 1] V-cycle iterate
  double* r = nullptr;           // [ngrid + 1] residual / scratch
  // GS wavefront progress flags, 3 x gs_groups, all tagged and never reset:
  // [0, G) sweep B's stored windows ((pair epoch << 32) | windows; overlap only),
  // [G, 2G) unused, [2G, 3G) sweep A's stored windows
  unsigned long long* gs_flags = nullptr;
  int gs_groups = 0;
  unsigned long long pair_epoch = 0;   // launches of the pipelined sweep pair on this level
  unsigned long long ready_epoch = 0;  // launches of k_prolong_rows into this level
  // descent overlap, [gs_groups x kSeg] (row band x column segment), tagged:
  unsigned long long* ovl_bready = nullptr;  // b restricted into this level (bready_epoch)
  unsigned long long* ovl_rdone = nullptr;   // residual of this level computed (rdone_epoch)
  // ascent overlap, [gs_groups x kChunk column chunks]: x_old prolongated (ready_epoch)
  unsigned long long* ovl_xready = nullptr;
  // descent overlap: the residual/restriction items of this level in the order they become
  // ready (k_residual_restrict_rows takes them by ticket), and the ticket counter
  int32_t* rr_order = nullptr;
  unsigned* rr_ticket = nullptr;
  int rr_items = 0;
  // ascent overlap: k_prolong_rows' items (band x column chunk) in diagonal order, ticket and exit counters
  int32_t* pr_order = nullptr;
  unsigned* pr_ticket = nullptr;  // grows by pr_items + blocks per launch (pr_base: the next launch's first ticket)
  unsigned pr_base = 0;
  int pr_items = 0;
  unsigned long long bready_epoch = 0;
  unsigned long long rdone_epoch = 0;
  double* x1 = nullptr;               // [ngrid + 1] sweep A's result inside a pair
  // cross-cluster band handoff rows, 2 x gs_groups x nx nodes (sweep A / single
  // sweeps, sweep B): each value is its own ready flag (kXferEmpty until the
  // producing band writes it; the consuming band resets it after reading)
  double* gs_xfer = nullptr;
  size_t pad_nodes = 0;  // zero nodes before/after stL, stU and every vector of this level
};

// MINRES device scalars (linalg.py:128-242 recurrences), one struct per solve
struct MinresDev {
  double beta1, beta, oldb, alfa, dbar, epsln, oldeps, phibar, cs, sn, phi, delta, gamma;
  double verify_at, relres, tol, bnorm, est;
  int iters, max_iters, stopped, status, no_verify, pad;
};

enum MinresStatus { kRunning = 0, kConverged = 1, kCap = 2, kIndefinite = -1, kBreakdown = -2, kNonfinite = -3,
                    kCholFail = -4 };

struct Hex;  // 3D hexahedral data (hex3d.inc.cu)

struct Ctx {
  int dim = 2;                  // 2: Q1 plane stress (this file's levels); 3: trilinear hexahedra (hex)
  Hex* hex = nullptr;
  int L = 0;                    // number of levels (index 0 = coarsest)
  std::vector<LevelBuf> lv;
  cudaStream_t stream = nullptr;
  int n = 0, m = 0;             // finest free dofs, elements
  double ke[64];
  double modal[8];         // K_e in the corner-mode basis / 16 (c_modal); valid when modal_ok
  bool modal_ok = false;   // K_e has the rectangular-Q1 mode structure: modal Newton apply

  // bound Newton matrix (finest level)
  double* u_grid = nullptr;     // [ngrid]
  double* rho_hat = nullptr;    // [m]
  double* chat = nullptr;       // [m]
  double corner = 0.0;
  double* d_corner = nullptr;   // device copy of corner
  bool system_bound = false;
  bool border_flip = false;    // the bound system is E S+ E (an IP system, ip.inc.cu): flip x_alpha at the API edge
  // the bound system is the plain stiffness K(rho) (fem.py:211-219, doc.inc.cu): held as
  // [[K, 0], [0, 1]] so every bordered kernel runs unchanged; API vectors have n entries
  // and the grid's border slot is zero on input (then stays exactly zero)
  bool unbordered = false;
  bool mg_ready = false;
  int shifted = 0;

  // coarsest dense Cholesky (free order + border)
  int N0 = 0;
  double* chol = nullptr;       // [N0 * N0] lower factor (row-major)
  double* chol_rdiag = nullptr; // [N0] correctly rounded reciprocals of its diagonal
  int* chol_status = nullptr;   // device status
  int* chol_retry = nullptr;    // device: the plain factor failed, the shifted one was built (device-gated setup)

  double* rap_tmp = nullptr;    // unsymmetrised coarse stencil of the largest coarse level

  // finest-level grid work vectors (ngrid + 1 each)
  std::vector<double*> fvec;

  // reductions
  double* partials = nullptr;   // [kMaxBlocks * kMaxPartials]
  unsigned int* counters = nullptr;  // last-block counters
  // descent overlap: x_alpha residual rows per level (k_residual_restrict_rows),
  // partials [16 levels x kReduceGridCap], last-block counters [16], and flags [16]:
  // b_alpha of the level is restricted (tagged like the level's bready_epoch)
  double* ovl_part = nullptr;
  unsigned* ovl_cnt = nullptr;
  unsigned long long* ovl_aflag = nullptr;
  double* dscal = nullptr;      // device scalars [64]
  double* hscal = nullptr;      // pinned host scalars [64]
  unsigned* dflags = nullptr;   // device warning flags
  MinresDev* mst = nullptr;     // device MINRES state
  MinresDev* hmst = nullptr;    // pinned host mirror, [2]: the two iterations in flight
  cudaEvent_t mr_ev[2] = {nullptr, nullptr};  // their state copies have landed

  // device-resident Newton step (step.inc.cu), allocated on first use
  struct StepState* step = nullptr;

  // DOC workspace (doc.inc.cu: sorted energies, scans, CUB scratch), allocated on first use
  void* doc_ws = nullptr;
  size_t doc_tmp_bytes = 0;

  long long launches = 0;
  std::vector<void*> allocs;  // the device arena holding every array of the context
  std::vector<size_t> alloc_bytes;  // sizes of `allocs` (returned to the device pool)

  // optional per-launch timing of the wavefront kernel (vts_profile_begin/end)
  bool prof = false;
  struct ProfEv {
    cudaEvent_t a, b;
    int level;
    int pair;  // 0: k_gs_tri, 1: k_gs_pair descent (zero guess + forward), 2: k_gs_pair ascent
  };
  std::vector<ProfEv> prof_ev;
  size_t prof_used = 0;  // padded device arrays owned by the context
};

constexpr int kMaxBlocks = 8192;
constexpr int kMaxPartials = 16;
constexpr int kNumFineVecs = 14;

// ---- error plumbing (capi.cu) ----
void set_error(int code, const std::string& msg);
int cuda_check(cudaError_t e, const char* what);
#define VTS_CUDA(call)                                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return cuda_check(_e, #call); \
  } while (0)
#define VTS_LAUNCHED(ctx)                                     \
  do {                                                        \
    (ctx)->launches++;                                        \
    cudaError_t _e = cudaGetLastError();                      \
    if (_e != cudaSuccess) return cuda_check(_e, "launch");   \
  } while (0)

// Programmatic dependent launch.  Kernels of the V-cycle / MINRES chain are
// launched with the programmatic stream-serialization attribute, so the next
// launch's CTAs are scheduled and run their prologue while the previous kernel
// drains; every such kernel starts with pdl_enter(): wait until the previous
// grid has completed and its memory is visible, then allow the next launch.
// (A kernel launched without the attribute passes both instructions at once.)
// VTS_NO_PDL=1 launches everything plainly (A/B checks).
// Kernel timeline probe (tools/probe/tl_probe, -DVTS_TIMELINE): first block start /
// last block end per (kernel kind, level) in globaltimer ns; level from nx = 4 * 2^k + 1
#ifdef VTS_TIMELINE
__device__ unsigned long long g_tl[160][2];
__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int tl_slot(int kind, int nx) {
  const int k = 31 - __clz(max(nx - 1, 4)) - 2;
  return kind * 16 + min(max(k, 0), 15);
}
__device__ unsigned long long g_items[1024][4];  // finest residual/restriction items: flag wait start, work start, end, block
#define VTS_TL_BEGIN(kind, nx) \
  do { if (threadIdx.x == 0) atomicMin(&g_tl[tl_slot(kind, nx)][0], tl_now()); } while (0)
#define VTS_TL_END(kind, nx) \
  do { __syncthreads(); if (threadIdx.x == 0) atomicMax(&g_tl[tl_slot(kind, nx)][1], tl_now()); } while (0)
#else
#define VTS_TL_BEGIN(kind, nx) do {} while (0)
#define VTS_TL_END(kind, nx) do {} while (0)
#endif

__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("VTS_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

inline int div_up(long long a, long long b) { return (int)((a + b - 1) / b); }

// ---- element / nodal passes (elem_kernels.cu) ----
int free_to_grid(Ctx* c, int level, const double* src, double* dst, bool bordered, const int* skip = nullptr);
int grid_to_free(Ctx* c, int level, const double* src, double* dst, bool bordered);
int eval_lagrangian(Ctx* c, const double* u, double alpha, const double* nu_lo, const double* nu_up,
                    const double* rho, const double* mu_lo, const double* mu_up, const double* p,
                    const double* q_lo, const double* q_up, const double* f, const double* lower,
                    const double* upper, double volume, double norm_f, double norm_bounds,
                    double branch, double* res_u, double* res_lo, double* res_up, double* q,
                    double* mu_hat_lo, double* mu_hat_up, double* a, double* b_lo, double* b_up,
                    double* rho_hat, double* w_out, double* scalars, unsigned* warn,
                    const double* alpha_dev = nullptr, const int* skip = nullptr);
int schur_system(Ctx* c, const double* u, const double* res_u, double res_alpha,
                 const double* res_lo, const double* res_up, const double* a, const double* b_lo,
                 const double* b_up, const double* rho_hat, double* chat, double* rhs,
                 double* border, double* corner, const double* res_alpha_dev = nullptr);
int reconstruct_nu(Ctx* c, const double* u, const double* du, double dalpha, const double* res_u,
                   double res_alpha, const double* res_lo, const double* res_up, const double* a,
                   const double* b_lo, const double* b_up, double* dnu_lo, double* dnu_up,
                   double* slope);
int al_value(Ctx* c, const double* u, double alpha, const double* nu_lo, const double* nu_up,
             const double* du, double dalpha, const double* dnu_lo, const double* dnu_up,
             double kappa, const double* rho, const double* p, const double* mu_lo,
             const double* mu_up, const double* q_lo, const double* q_up, const double* f,
             const double* lower, const double* upper, double volume, double branch,
             double* value, unsigned* warn);
int axpy(Ctx* c, long long len, double kappa, const double* dx, double* x);
int penalty_eval(Ctx* c, long long n, const double* tau, double branch, double* v, double* d1, double* d2,
                 unsigned* warn);
int outer_update(Ctx* c, double beta, double gamma, double floor_p, const double* rho_hat,
                 const double* mu_hat_lo, const double* mu_hat_up, double* rho, double* mu_lo,
                 double* mu_up, double* p, double* q_lo, double* q_up, int update_penalties);
int gap(Ctx* c, const double* u, double alpha, const double* q, const double* f,
        const double* nu_lo, const double* nu_up, const double* lower, const double* upper,
        double volume, const double* rho, double* d_val, double* gap, double* fu,
        double* rho_sum);

// ---- operators (apply.cu) ----
// y = S x on grid-layout bordered vectors of the finest level (matrix free)
int newton_apply_grid(Ctx* c, const double* x, double* y, const int* skip);
// y = A_k x on grid-layout bordered vectors of level k (stencil)
int level_apply_grid(Ctx* c, int k, const double* x, double* y, const int* skip);
int level_residual_grid(Ctx* c, int k, const double* x, const double* b, double* r, const int* skip);

// ---- multigrid (mg.cu) ----
// device_gate: the coarse factor's shifted retry (multigrid.py:92-103) is enqueued
// behind device flags instead of a host read-back of the factor status (no sync)
int mg_setup(Ctx* c, double shift_scale, bool device_gate = false);
int vcycle_grid(Ctx* c, const double* b, double* z, const int* skip);
int debug_smooth(Ctx* c, int k, bool forward, bool zero_first, const double* b_free, double* x_free);
int profile_begin(Ctx* c);
int profile_end(Ctx* c, double* out);

// ---- MINRES (minres.cu) ----
int minres(Ctx* c, const double* b_free, double* x_free, double tol, int max_iters,
           double floor_tol, int precondition, int* iters, double* relres, int* converged,
           double* history, const double* x0_free = nullptr, bool device_init = false);

// ---- generic reductions (elem_kernels.cu) ----
// dot of two grid vectors (free dofs only are nonzero) incl. the border slot
// when `bordered`; result written to dst (device) ; deterministic.
int dot_grid(Ctx* c, int level, const double* a, const double* b, bool bordered, double* dst,
             const int* skip);

int minres_generic(Ctx* c, long long len, const double* b, double* x_out, const double* x0, double tol,
                   int max_iters, double floor_tol, vts_apply_fn op, vts_apply_fn prec, void* user,
                   int* iters_out, double* relres_out, int* conv_out, double* history, bool native = false);

// ---- device-resident Newton step (step.inc.cu) ----
int newton_step(Ctx* c, const vts_newton_step_args* a, vts_newton_step_result* r);

// ---- DOC reuse (doc.inc.cu) ----
int bind_stiffness(Ctx* c, const double* rho, unsigned* warn);
int element_energy(Ctx* c, const double* u, double* w, double* q);
int doc_bisect(Ctx* c, const double* rho, const double* q, double zscale, const double* lower,
               const double* upper, double volume, double exponent, double alpha_hi, double tol, int cap,
               double* rho_new, double* alpha_out, int* status);
int doc_update(Ctx* c, const double* rho, const double* z, double zscale, double alpha, double exponent,
               const double* lower, const double* upper, double* rho_new);
int doc_measure(Ctx* c, const double* rho_new, const double* rho, const double* q, const double* u,
                const double* f, const double* lower, const double* upper, double volume, double* out5);

}  // namespace vts
