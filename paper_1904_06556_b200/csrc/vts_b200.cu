// libvts_b200 — B200-native PBM inner Newton step behind a C ABI.
//
// Unity build: every kernel file is included here so the element stiffness
// can live in one __constant__ symbol without relocatable device code.
// See include/vts_b200.h for the entry points and the reference interfaces
// they replace, DESIGN.md for the data layout and the kernels' rooflines.

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "../../include/vts_b200.h"
#include "context.cuh"
#include "tma.cuh"

#include "elem_kernels.inc.cu"
#include "apply.inc.cu"
#include "mg.inc.cu"
#include "minres.inc.cu"
#include "ip.inc.cu"
#include "doc.inc.cu"
#include "step.inc.cu"
#include "hex3d.inc.cu"

namespace vts {

static thread_local std::string g_last_error;
static std::mutex g_ke_mutex;
static const Ctx* g_ke_owner = nullptr;

void set_error(int code, const std::string& msg) {
  (void)code;
  g_last_error = msg;
}

int cuda_check(cudaError_t e, const char* what) {
  set_error(VTS_E_CUDA, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
  return VTS_E_CUDA;
}

// The element stiffness is a module-wide __constant__ (uniform operands in every
// element kernel).  Contexts whose K_e equals the loaded one share it with no
// ordering at all.  A context with a different K_e takes the constant over in
// stream order: its stream first waits for everything enqueued so far on every
// stream that used the loaded constant (one event per stream), then uploads.
// Calls of a context with the old K_e hand it back the same way, so no kernel
// ever reads a constant that is not its context's, whatever streams they use.
static double g_ke_loaded[64 + 8];
static bool g_ke_valid = false;
static std::vector<cudaStream_t> g_ke_users;  // streams that used the loaded constant
static std::map<cudaStream_t, int> g_stream_refs;  // live contexts per stream
static cudaEvent_t g_ke_event = nullptr;

static double g_ke3_loaded[576];
static bool g_ke3_valid = false;
static std::vector<cudaStream_t> g_ke3_users;

// the 3D path's K_e (c_ke3, 24 x 24) under the same ownership rule
static int ensure_ke3(Ctx* c) {
  if (g_ke3_valid && std::memcmp(c->hex->ke, g_ke3_loaded, sizeof(g_ke3_loaded)) == 0) {
    if (std::find(g_ke3_users.begin(), g_ke3_users.end(), c->stream) == g_ke3_users.end())
      g_ke3_users.push_back(c->stream);
    return 0;
  }
  if (!g_ke_event) VTS_CUDA(cudaEventCreateWithFlags(&g_ke_event, cudaEventDisableTiming));
  for (cudaStream_t s : g_ke3_users) {
    if (s == c->stream) continue;
    VTS_CUDA(cudaEventRecord(g_ke_event, s));
    VTS_CUDA(cudaStreamWaitEvent(c->stream, g_ke_event, 0));
  }
  VTS_CUDA(cudaMemcpyToSymbolAsync(c_ke3, c->hex->ke, sizeof(double) * 576, 0, cudaMemcpyHostToDevice, c->stream));
  std::memcpy(g_ke3_loaded, c->hex->ke, sizeof(g_ke3_loaded));
  g_ke3_valid = true;
  g_ke3_users.assign(1, c->stream);
  return 0;
}

static int ensure_ke(Ctx* c) {
  std::lock_guard<std::mutex> lock(g_ke_mutex);
  if (c->dim == 3) return ensure_ke3(c);
  if (g_ke_owner == c) return 0;
  double want[64 + 8];
  std::memcpy(want, c->ke, sizeof(double) * 64);
  std::memcpy(want + 64, c->modal, sizeof(double) * 8);
  if (g_ke_valid && std::memcmp(want, g_ke_loaded, sizeof(want)) == 0) {
    if (std::find(g_ke_users.begin(), g_ke_users.end(), c->stream) == g_ke_users.end())
      g_ke_users.push_back(c->stream);
    g_ke_owner = c;
    return 0;
  }
  if (!g_ke_event) VTS_CUDA(cudaEventCreateWithFlags(&g_ke_event, cudaEventDisableTiming));
  for (cudaStream_t s : g_ke_users) {
    if (s == c->stream) continue;
    VTS_CUDA(cudaEventRecord(g_ke_event, s));
    VTS_CUDA(cudaStreamWaitEvent(c->stream, g_ke_event, 0));
  }
  VTS_CUDA(cudaMemcpyToSymbolAsync(c_ke, c->ke, sizeof(double) * 64, 0, cudaMemcpyHostToDevice, c->stream));
  VTS_CUDA(cudaMemcpyToSymbolAsync(c_modal, c->modal, sizeof(double) * 8, 0, cudaMemcpyHostToDevice, c->stream));
  std::memcpy(g_ke_loaded, want, sizeof(want));
  g_ke_valid = true;
  g_ke_users.assign(1, c->stream);
  g_ke_owner = c;
  return 0;
}

// Every device array of a context lives in ONE allocation (cudaMalloc and
// cudaFree cost tens to hundreds of microseconds each, and a context has ~130
// arrays).  Creation records requests, then `Arena::commit` allocates, zeroes
// the whole block once and hands out 256-byte aligned pointers.
// Pinned host scalars ([64] doubles, then the MINRES state mirror) come from a
// process-wide pool: cudaMallocHost costs milliseconds, and solvers create a
// context per problem.  free_ctx releases a block only after a device
// synchronisation, so no copy into it can still be in flight.
constexpr size_t kPinnedBytes = ((64 * sizeof(double) + 2 * sizeof(MinresDev)) + 255) & ~size_t(255);
static std::mutex g_pinned_mutex;
static std::vector<void*> g_pinned_free;

// Device arenas are recycled the same way: a context's single allocation goes
// back to a small process-wide pool (at most kDevPool blocks) and the next
// context of a similar size takes it, so a solver that creates one context per
// problem pays cudaMalloc once (tens of milliseconds for a 0.5 GB arena).
constexpr size_t kDevPool = 2;
static std::mutex g_dev_mutex;
static std::vector<std::pair<void*, size_t>> g_dev_free;

static cudaError_t device_acquire(void** p, size_t* bytes) {
  {
    std::lock_guard<std::mutex> lock(g_dev_mutex);
    for (size_t i = 0; i < g_dev_free.size(); ++i) {
      const size_t have = g_dev_free[i].second;
      if (have >= *bytes && have <= 2 * *bytes) {
        *p = g_dev_free[i].first;
        *bytes = have;
        g_dev_free.erase(g_dev_free.begin() + (ptrdiff_t)i);
        return cudaSuccess;
      }
    }
  }
  return cudaMalloc(p, *bytes);
}

static void device_release(void* p, size_t bytes) {
  void* evict = nullptr;
  {
    std::lock_guard<std::mutex> lock(g_dev_mutex);
    g_dev_free.emplace_back(p, bytes);
    if (g_dev_free.size() > kDevPool) {
      evict = g_dev_free.front().first;
      g_dev_free.erase(g_dev_free.begin());
    }
  }
  if (evict) cudaFree(evict);
}

static void* pinned_acquire() {
  {
    std::lock_guard<std::mutex> lock(g_pinned_mutex);
    if (!g_pinned_free.empty()) {
      void* p = g_pinned_free.back();
      g_pinned_free.pop_back();
      return p;
    }
  }
  void* p = nullptr;
  return cudaMallocHost(&p, kPinnedBytes) == cudaSuccess ? p : nullptr;
}

static void pinned_release(void* p) {
  std::lock_guard<std::mutex> lock(g_pinned_mutex);
  g_pinned_free.push_back(p);
}

#ifndef VTS_CREATE_MARK
#define VTS_CREATE_MARK(s)
#endif

struct Arena {
  struct Req {
    void** slot;
    size_t offset;  // bytes from the arena base to the handed-out pointer
  };
  std::vector<Req> reqs;
  size_t used = 0;

  size_t take(void** slot, size_t bytes, size_t pad_bytes) {
    const size_t start = (used + 255) & ~size_t(255);
    used = start + std::max<size_t>(bytes + 2 * pad_bytes, 1);
    reqs.push_back({slot, start + pad_bytes});
    return start + pad_bytes;
  }
  int commit(Ctx* c) {
    char* base = nullptr;
    size_t bytes = std::max<size_t>(used, 256);
    VTS_CUDA(device_acquire(reinterpret_cast<void**>(&base), &bytes));
    c->allocs.push_back(base);
    c->alloc_bytes.push_back(bytes);
    VTS_CUDA(cudaMemset(base, 0, used));
    for (const Req& r : reqs) *r.slot = base + r.offset;
    return 0;
  }
};

template <typename T>
static size_t dalloc(Arena& a, T** p, size_t count) {
  return a.take(reinterpret_cast<void**>(p), count * sizeof(T), 0);
}

// zeroed array of `count` doubles with `pad` zero doubles before and after
// (the skewed TMA boxes of the Gauss-Seidel wavefront read into the padding)
static void dalloc_pad(Arena& a, double** p, size_t count, size_t pad) {
  a.take(reinterpret_cast<void**>(p), count * sizeof(double), pad * sizeof(double));
}

static void free_ctx(Ctx* c) {
  cudaDeviceSynchronize();  // nothing may still write into the blocks handed back below
  for (size_t i = 0; i < c->allocs.size(); ++i) device_release(c->allocs[i], c->alloc_bytes[i]);
  for (cudaEvent_t e : c->mr_ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->prof_ev) {
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  if (c->hscal) pinned_release(c->hscal);
  if (c->doc_ws) cudaFree(c->doc_ws);
  delete c->step;
  {
    // after the synchronisation above nothing of this context is in flight; its
    // stream may be destroyed by its owner, so it leaves the user list unless a
    // live context still runs on it
    std::lock_guard<std::mutex> lock(g_ke_mutex);
    if (g_ke_owner == c) g_ke_owner = nullptr;
    if (--g_stream_refs[c->stream] == 0) {
      g_stream_refs.erase(c->stream);
      g_ke_users.erase(std::remove(g_ke_users.begin(), g_ke_users.end(), c->stream), g_ke_users.end());
      g_ke3_users.erase(std::remove(g_ke3_users.begin(), g_ke3_users.end(), c->stream), g_ke3_users.end());
    }
  }
  delete c->hex;
  delete c;
}

// K_e in the basis of corner modes.  Per displacement component the four nodal
// values (corners (0,0) (1,0) (1,1) (0,1)) map to the modes 1 = (1 1 1 1),
// xi = (-1 1 1 -1), eta = (-1 -1 1 1) and h = (1 -1 1 -1); T (8 x 8) holds them
// as columns and T^T T = 4 I, so K u = T (T^T K T / 16) (T^T u).  For the
// bilinear rectangle (any E, nu, aspect) T^T K T vanishes on the translations
// and couples only {xi_x, eta_y} (normal strains), {xi_y, eta_x} (shear) and
// each hourglass mode with itself: 8 numbers instead of 64, and the Newton
// apply does ~80 instead of ~150 fp64 operations per element.  Any other K_e
// keeps the dense apply (modal_ok = false).
static void modal_form(Ctx* c) {
  static const double e[4][4] = {{1, 1, 1, 1}, {-1, 1, 1, -1}, {-1, -1, 1, 1}, {1, -1, 1, -1}};
  double t[8][8] = {};  // column 2k + comp: mode k of component comp
  for (int k = 0; k < 4; ++k)
    for (int a = 0; a < 4; ++a)
      for (int comp = 0; comp < 2; ++comp) t[2 * a + comp][2 * k + comp] = e[k][a];
  double km[8][8];
  double kmax = 0.0;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      double sum = 0.0;
      for (int p = 0; p < 8; ++p)
        for (int q = 0; q < 8; ++q) sum += t[p][i] * c->ke[8 * p + q] * t[q][j];
      km[i][j] = sum / 16.0;
      kmax = std::max(kmax, std::fabs(km[i][j]));
    }
  // modes: 0 1x, 1 1y, 2 xi_x, 3 xi_y, 4 eta_x, 5 eta_y, 6 h_x, 7 h_y
  const int keep[8][2] = {{2, 2}, {5, 5}, {2, 5}, {3, 3}, {4, 4}, {3, 4}, {6, 6}, {7, 7}};
  bool ok = kmax > 0.0;
  for (int i = 0; i < 8 && ok; ++i)
    for (int j = 0; j < 8 && ok; ++j) {
      bool kept = false;
      for (const auto& kv : keep) kept |= (kv[0] == i && kv[1] == j) || (kv[0] == j && kv[1] == i);
      if (!kept && std::fabs(km[i][j]) > 1e-13 * kmax) ok = false;
      if (std::fabs(km[i][j] - km[j][i]) > 1e-13 * kmax) ok = false;
    }
  for (int i = 0; i < 8; ++i) c->modal[i] = km[keep[i][0]][keep[i][1]];
  c->modal_ok = ok;
}

static int create(Ctx** out, int levels, const int32_t* ex, const int32_t* ey, const int64_t* const* dof_maps,
                  const double* ke, int64_t stream) {
  if (levels < 1 || !ex || !ey || !dof_maps || !ke || !out) {
    set_error(VTS_E_ARGUMENT, "vts_ctx_create: bad arguments");
    return VTS_E_ARGUMENT;
  }
  for (int k = 0; k < levels; ++k) {
    if (ex[k] < 1 || ey[k] < 1) {
      set_error(VTS_E_ARGUMENT, "vts_ctx_create: element counts must be positive");
      return VTS_E_ARGUMENT;
    }
    if (k > 0 && (ex[k] != 2 * ex[k - 1] || ey[k] != 2 * ey[k - 1])) {
      set_error(VTS_E_ARGUMENT, "vts_ctx_create: each level must refine the previous one by 2 per axis");
      return VTS_E_ARGUMENT;
    }
  }
  Ctx* c = new Ctx();
  c->L = levels;
  c->stream = reinterpret_cast<cudaStream_t>(stream);
  {
    std::lock_guard<std::mutex> lock(g_ke_mutex);
    ++g_stream_refs[c->stream];
  }
  std::memcpy(c->ke, ke, sizeof(double) * 64);
  modal_form(c);
  c->lv.resize(levels);
  auto fail = [&](int rc) {
    free_ctx(c);
    return rc;
  };
  Arena arena;
  // the per-level index maps (free mask, free->grid, grid->free) are placed
  // first in the arena; they are written into one host image and uploaded
  // with one copy after the allocation (free->grid is sized by ng, an upper
  // bound of the free count)
  std::vector<size_t> map_off(3 * levels);
  for (int k = 0; k < levels; ++k) {
    LevelBuf& L = c->lv[k];
    L.d.ex = ex[k];
    L.d.ey = ey[k];
    L.d.nx = ex[k] + 1;
    L.d.ny = ey[k] + 1;
    L.d.nnodes = L.d.nx * L.d.ny;
    L.d.ngrid = 2 * L.d.nnodes;
    const size_t ng = L.d.ngrid;
    map_off[3 * k] = dalloc(arena, const_cast<uint8_t**>(&L.d.free_mask), ng);
    map_off[3 * k + 1] = dalloc(arena, const_cast<int32_t**>(&L.d.free2grid), ng);
    map_off[3 * k + 2] = dalloc(arena, &L.grid2free, ng);
  }
  std::vector<char> image(arena.used);
  for (int k = 0; k < levels; ++k) {
    LevelBuf& L = c->lv[k];
    const int ng = L.d.ngrid;
    uint8_t* mask = reinterpret_cast<uint8_t*>(image.data() + map_off[3 * k]);
    int32_t* f2g = reinterpret_cast<int32_t*>(image.data() + map_off[3 * k + 1]);
    int32_t* g2f = reinterpret_cast<int32_t*>(image.data() + map_off[3 * k + 2]);
    const int64_t* dm = dof_maps[k];
    int nfree = 0;
    for (int i = 0; i < ng; ++i) {
      const int64_t d = dm[i];
      if (d >= 0) {
        if (d != nfree) {
          set_error(VTS_E_ARGUMENT, "vts_ctx_create: dof map must number free dofs node-major in order");
          return fail(VTS_E_ARGUMENT);
        }
        mask[i] = 1;
        g2f[i] = nfree;
        f2g[nfree++] = i;
      } else {
        mask[i] = 0;
        g2f[i] = -1;
      }
    }
    if (nfree == 0) {
      set_error(VTS_E_ARGUMENT, "vts_ctx_create: a level has no free dofs");
      return fail(VTS_E_ARGUMENT);
    }
    L.d.nfree = nfree;
  }
  VTS_CREATE_MARK("maps");
  const size_t upload_end = arena.used;
  for (int k = 0; k < levels; ++k) {
    LevelBuf& L = c->lv[k];
    const size_t ng = L.d.ngrid;
    L.pad_nodes = (size_t)kPadRows * L.d.nx;
    if (const char* e = getenv("VTS_ARENA_PAD")) {  // placement diagnostic (see below): n x 256 bytes before each level
      static char* unused[64];
      dalloc(arena, &unused[k & 63], (size_t)std::max(1, atoi(e)) * 256);
    }
    dalloc_pad(arena, &L.d.stL, (size_t)L.d.nnodes * kHalf, L.pad_nodes * kHalf);
    dalloc_pad(arena, &L.d.stU, (size_t)L.d.nnodes * kHalf, L.pad_nodes * kHalf);
    dalloc_pad(arena, &L.d.border, ng + 1, 2 * L.pad_nodes);
    dalloc_pad(arena, &L.b, ng + 1, 2 * L.pad_nodes);
    dalloc_pad(arena, &L.x, ng + 1, 2 * L.pad_nodes);
    dalloc_pad(arena, &L.r, ng + 1, 2 * L.pad_nodes);
    dalloc_pad(arena, &L.x1, ng + 1, 2 * L.pad_nodes);
    L.gs_groups = div_up(L.d.ny, 8);  // >= bands of any GS row-band height used
    dalloc(arena, &L.gs_flags, 3 * (size_t)L.gs_groups);
    dalloc(arena, &L.ovl_bready, (size_t)kSeg * L.gs_groups);
    dalloc(arena, &L.ovl_rdone, (size_t)kSeg * L.gs_groups);
    dalloc(arena, &L.ovl_xready, (size_t)div_up(L.d.nx, kChunk) * L.gs_groups);
    dalloc(arena, &L.gs_xfer, 2 * 2 * (size_t)L.gs_groups * L.d.nx);
  }
  const LevelBuf& F = c->lv[levels - 1];
  c->n = F.d.nfree;
  c->m = F.d.ex * F.d.ey;
  const int len = F.d.ngrid + 1;
  c->fvec.assign(kNumFineVecs, nullptr);
  for (int i = 0; i < kNumFineVecs; ++i) dalloc_pad(arena, &c->fvec[i], std::max(len, c->m + 1), 2 * F.pad_nodes);
  dalloc(arena, &c->u_grid, len);
  dalloc(arena, &c->rho_hat, c->m);
  dalloc(arena, &c->chat, c->m);
  dalloc(arena, &c->d_corner, 1);
  c->N0 = c->lv[0].d.nfree + 1;
  dalloc(arena, &c->chol, (size_t)c->N0 * c->N0);
  dalloc(arena, &c->chol_rdiag, (size_t)c->N0);
  dalloc(arena, &c->chol_status, 1);
  dalloc(arena, &c->chol_retry, 1);
  const size_t rap = levels > 1 ? (size_t)c->lv[levels - 2].d.nnodes * kStencilStride : 1;
  dalloc(arena, &c->rap_tmp, rap);
  dalloc(arena, &c->partials, (size_t)kMaxBlocks * kMaxPartials);
  dalloc(arena, &c->ovl_part, (size_t)16 * kReduceGridCap);
  dalloc(arena, &c->ovl_cnt, 16);
  dalloc(arena, &c->ovl_aflag, 16);
  dalloc(arena, &c->counters, 64);
  dalloc(arena, &c->dscal, 64);
  dalloc(arena, &c->dflags, 4);
  dalloc(arena, &c->mst, 1);
  // (after everything else.  The placement of the level arrays matters: shifting each level's
  // block by a few hundred bytes to a few KB moves the V-cycle between two repeatable states
  // 3.7 % apart -- 945 vs 911 MINRES it/s on C3 with 256 n bytes of padding per level, n = 0 1
  // 2 7 1024 fast, 3 4 8 16 64 slow (tools/runs/r02_s5_layout.sh) -- so new per-level arrays
  // go here, behind the arrays the sweeps stream.)
  for (int k = 0; k < levels; ++k) {
    LevelBuf& L = c->lv[k];
    L.rr_items = k >= 1 ? div_up(c->lv[k - 1].d.ny, kBandRows) * 3 * kSeg : 0;
    dalloc(arena, &L.rr_order, (size_t)std::max(L.rr_items, 1));
    dalloc(arena, &L.rr_ticket, 1);
    L.pr_items = div_up(L.d.ny, kBandRows) * div_up(L.d.nx, kChunk);
    dalloc(arena, &L.pr_order, (size_t)L.pr_items);
    dalloc(arena, &L.pr_ticket, 1);
  }
  VTS_CREATE_MARK("plan");
  if (arena.commit(c)) return fail(VTS_E_CUDA);
  VTS_CREATE_MARK("commit");
  {
    char* base = static_cast<char*>(c->allocs.back());
    if (cudaMemcpy(base, image.data(), upload_end, cudaMemcpyHostToDevice) != cudaSuccess) {
      set_error(VTS_E_CUDA, "vts_ctx_create: device upload failed");
      return fail(VTS_E_CUDA);
    }
  }
  for (int k = 0; k < levels; ++k) {  // handoff rows start empty (kXferEmpty: all bits set)
    const LevelBuf& L = c->lv[k];
    if (cudaMemset(L.gs_xfer, 0xFF, 2 * 2 * (size_t)L.gs_groups * L.d.nx * sizeof(double)) != cudaSuccess) {
      set_error(VTS_E_CUDA, "vts_ctx_create: device memset failed");
      return fail(VTS_E_CUDA);
    }
    {
      const std::vector<int32_t> order = pr_item_order(L.d.nx, L.d.ny);
      if (cudaMemcpy(L.pr_order, order.data(), order.size() * sizeof(int32_t), cudaMemcpyHostToDevice) != cudaSuccess) {
        set_error(VTS_E_CUDA, "vts_ctx_create: device upload failed");
        return fail(VTS_E_CUDA);
      }
    }
    if (k >= 1) {
      const std::vector<int32_t> order = rr_item_order(L.d.nx, L.d.ny, c->lv[k - 1].d.nx, c->lv[k - 1].d.ny);
      if (cudaMemcpy(L.rr_order, order.data(), order.size() * sizeof(int32_t), cudaMemcpyHostToDevice) != cudaSuccess) {
        set_error(VTS_E_CUDA, "vts_ctx_create: device upload failed");
        return fail(VTS_E_CUDA);
      }
    }
  }
  VTS_CREATE_MARK("upload");
  if (!(c->hscal = static_cast<double*>(pinned_acquire()))) {
    set_error(VTS_E_CUDA, "vts_ctx_create: pinned allocation failed");
    return fail(VTS_E_CUDA);
  }
  c->hmst = reinterpret_cast<MinresDev*>(c->hscal + 64);
  VTS_CREATE_MARK("pinned");
  if (cudaDeviceSynchronize() != cudaSuccess) {
    set_error(VTS_E_CUDA, "vts_ctx_create: device synchronisation failed");
    return fail(VTS_E_CUDA);
  }
  *out = c;
  return 0;
}

}  // namespace vts

#include "hex3d_host.inc.cu"

using vts::Ctx;
using vts::cuda_check;

struct vts_ctx {
  Ctx impl;
};

static Ctx* C(vts_ctx* p) { return reinterpret_cast<Ctx*>(p); }
static const Ctx* C(const vts_ctx* p) { return reinterpret_cast<const Ctx*>(p); }

#define VTS_REQUIRE_CTX(ctx)                                 \
  do {                                                       \
    if (!(ctx)) {                                            \
      vts::set_error(VTS_E_ARGUMENT, "null context");       \
      return VTS_E_ARGUMENT;                                 \
    }                                                        \
    if (int _rc = vts::ensure_ke(C(ctx))) return _rc;        \
  } while (0)

// entry points of the 2D path only (benchmark probes, the interior-point blocks)
#define VTS_REQUIRE_2D(ctx)                                                   \
  do {                                                                        \
    if (C(ctx)->dim != 2) {                                                   \
      vts::set_error(VTS_E_ARGUMENT, "this entry point exists for 2D contexts only"); \
      return VTS_E_ARGUMENT;                                                  \
    }                                                                         \
  } while (0)

extern "C" {

const char* vts_last_error(void) { return vts::g_last_error.c_str(); }

int vts_version(void) { return 1; }

int vts_ctx_create(vts_ctx** out, int32_t levels, const int32_t* ex, const int32_t* ey,
                   const int64_t* const* dof_maps, const double* ke, int64_t stream) {
  Ctx* c = nullptr;
  const int rc = vts::create(&c, levels, ex, ey, dof_maps, ke, stream);
  if (rc) return rc;
  *out = reinterpret_cast<vts_ctx*>(c);
  return 0;
}

int vts_ctx_create3(vts_ctx** out, int32_t levels, const int32_t* ex, const int32_t* ey, const int32_t* ez,
                    const int64_t* const* dof_maps, const double* ke, int64_t stream) {
  Ctx* c = nullptr;
  const int rc = vts::h3_create(&c, levels, ex, ey, ez, dof_maps, ke, stream);
  if (rc) return rc;
  *out = reinterpret_cast<vts_ctx*>(c);
  return 0;
}

int vts_ctx_dim(const vts_ctx* ctx) { return ctx ? C(ctx)->dim : 0; }

int vts_ctx_destroy(vts_ctx* ctx) {
  if (ctx) vts::free_ctx(C(ctx));
  return 0;
}

int vts_ctx_sizes(const vts_ctx* ctx, int64_t* n, int64_t* m) {
  if (!ctx) return VTS_E_ARGUMENT;
  if (n) *n = C(ctx)->n;
  if (m) *m = C(ctx)->m;
  return 0;
}

int vts_level_size(const vts_ctx* ctx, int32_t level, int64_t* n) {
  if (!ctx || level < 0 || level >= C(ctx)->L) return VTS_E_ARGUMENT;
  *n = C(ctx)->dim == 3 ? C(ctx)->hex->lv[level].nfree : C(ctx)->lv[level].d.nfree;
  return 0;
}

int vts_eval_lagrangian(vts_ctx* ctx, const double* u, double alpha, const double* nu_lo, const double* nu_up,
                        const double* rho, const double* mu_lo, const double* mu_up, const double* p,
                        const double* q_lo, const double* q_up, const double* f, const double* lower,
                        const double* upper, double volume, double norm_f, double norm_bounds, double branch,
                        double* res_u, double* res_lo, double* res_up, double* q, double* mu_hat_lo,
                        double* mu_hat_up, double* a, double* b_lo, double* b_up, double* rho_hat, double* w_out,
                        double* scalars, uint32_t* warn_flags) {
  VTS_REQUIRE_CTX(ctx);
  unsigned warn = 0;
  const int rc = C(ctx)->dim == 3
                     ? vts::h3_eval_lagrangian(C(ctx), u, alpha, nu_lo, nu_up, rho, mu_lo, mu_up, p, q_lo, q_up, f,
                                               lower, upper, volume, norm_f, norm_bounds, branch, res_u, res_lo,
                                               res_up, q, mu_hat_lo, mu_hat_up, a, b_lo, b_up, rho_hat, w_out,
                                               scalars, &warn)
                     : vts::eval_lagrangian(C(ctx), u, alpha, nu_lo, nu_up, rho, mu_lo, mu_up, p, q_lo, q_up, f,
                                            lower, upper, volume, norm_f, norm_bounds, branch, res_u, res_lo, res_up,
                                            q, mu_hat_lo, mu_hat_up, a, b_lo, b_up, rho_hat, w_out, scalars, &warn);
  if (warn_flags) *warn_flags = warn ? VTS_W_SATURATED : 0u;
  return rc;
}

int vts_schur_system(vts_ctx* ctx, const double* u, const double* res_u, double res_alpha, const double* res_lo,
                     const double* res_up, const double* a, const double* b_lo, const double* b_up,
                     const double* rho_hat, double* chat, double* rhs, double* border, double* corner) {
  VTS_REQUIRE_CTX(ctx);
  if (C(ctx)->dim == 3)
    return vts::h3_schur_system(C(ctx), u, res_u, res_alpha, res_lo, res_up, a, b_lo, b_up, rho_hat, chat, rhs,
                                border, corner);
  return vts::schur_system(C(ctx), u, res_u, res_alpha, res_lo, res_up, a, b_lo, b_up, rho_hat, chat, rhs, border,
                           corner);
}

int vts_newton_apply(vts_ctx* ctx, const double* x, double* y) {
  VTS_REQUIRE_CTX(ctx);
  Ctx* c = C(ctx);
  if (c->dim == 3) return vts::h3_newton_apply(c, x, y);
  if (!c->system_bound) {
    vts::set_error(VTS_E_ARGUMENT, "vts_newton_apply: no Newton system bound");
    return VTS_E_ARGUMENT;
  }
  const int F = c->L - 1;
  if (int rc = vts::free_to_grid(c, F, x, c->fvec[10], true)) return rc;
  if (int rc = vts::newton_apply_grid(c, c->fvec[10], c->fvec[11], nullptr)) return rc;
  if (int rc = vts::grid_to_free(c, F, c->fvec[11], y, true)) return rc;
  VTS_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

int vts_mg_setup(vts_ctx* ctx, double shift_scale, int32_t* shifted) {
  VTS_REQUIRE_CTX(ctx);
  const int rc = C(ctx)->dim == 3 ? vts::h3_mg_setup(C(ctx), shift_scale) : vts::mg_setup(C(ctx), shift_scale);
  if (shifted) *shifted = C(ctx)->shifted;
  return rc;
}

int vts_vcycle(vts_ctx* ctx, const double* b, double* z) {
  VTS_REQUIRE_CTX(ctx);
  Ctx* c = C(ctx);
  if (c->dim == 3) return vts::h3_vcycle(c, b, z);
  if (!c->mg_ready) {
    vts::set_error(VTS_E_ARGUMENT, "vts_vcycle: multigrid not set up");
    return VTS_E_ARGUMENT;
  }
  const int F = c->L - 1;
  if (int rc = vts::free_to_grid(c, F, b, c->fvec[10], true)) return rc;
  if (int rc = vts::vcycle_grid(c, c->fvec[10], c->fvec[11], nullptr)) return rc;
  if (int rc = vts::grid_to_free(c, F, c->fvec[11], z, true)) return rc;
  VTS_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

int vts_level_apply(vts_ctx* ctx, int32_t level, const double* x, double* y) {
  VTS_REQUIRE_CTX(ctx);
  Ctx* c = C(ctx);
  if (c->dim == 3) return vts::h3_level_apply(c, level, x, y);
  if (level < 0 || level >= c->L || !c->mg_ready) {
    vts::set_error(VTS_E_ARGUMENT, "vts_level_apply: bad level or multigrid not set up");
    return VTS_E_ARGUMENT;
  }
  if (int rc = vts::free_to_grid(c, level, x, c->fvec[10], true)) return rc;
  if (int rc = vts::level_apply_grid(c, level, c->fvec[10], c->fvec[11], nullptr)) return rc;
  if (int rc = vts::grid_to_free(c, level, c->fvec[11], y, true)) return rc;
  VTS_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

int vts_minres(vts_ctx* ctx, const double* b, double* x, double tol, int32_t max_iters, double floor_tol,
               int32_t precondition, int32_t* iterations, double* relres, int32_t* converged, double* history) {
  VTS_REQUIRE_CTX(ctx);
  int it = 0, conv = 0;
  double rr = 0.0;
  const int rc = C(ctx)->dim == 3
                     ? vts::h3_minres(C(ctx), b, x, nullptr, tol, max_iters, floor_tol, precondition, &it, &rr, &conv,
                                      history)
                     : vts::minres(C(ctx), b, x, tol, max_iters, floor_tol, precondition, &it, &rr, &conv, history);
  if (iterations) *iterations = it;
  if (relres) *relres = rr;
  if (converged) *converged = conv;
  return rc;
}

int vts_debug_smooth(vts_ctx* ctx, int32_t level, int32_t forward, int32_t zero_first, const double* b,
                     double* x) {
  VTS_REQUIRE_CTX(ctx);
  VTS_REQUIRE_2D(ctx);
  return vts::debug_smooth(C(ctx), level, forward != 0, zero_first != 0, b, x);
}

int vts_minres_warm(vts_ctx* ctx, const double* b, double* x, const double* x0, double tol, int32_t max_iters,
                    double floor_tol, int32_t precondition, int32_t* iterations, double* relres, int32_t* converged,
                    double* history) {
  VTS_REQUIRE_CTX(ctx);
  int it = 0, conv = 0;
  double rr = 0.0;
  const int rc = C(ctx)->dim == 3
                     ? vts::h3_minres(C(ctx), b, x, x0, tol, max_iters, floor_tol, precondition, &it, &rr, &conv,
                                      history)
                     : vts::minres(C(ctx), b, x, tol, max_iters, floor_tol, precondition, &it, &rr, &conv, history, x0);
  if (iterations) *iterations = it;
  if (relres) *relres = rr;
  if (converged) *converged = conv;
  return rc;
}

int vts_minres_generic(vts_ctx* ctx, int64_t len, const double* b, double* x, const double* x0, double tol,
                       int32_t max_iters, double floor_tol, vts_apply_fn op, vts_apply_fn precond, void* user,
                       int32_t* iterations, double* relres, int32_t* converged, double* history) {
  VTS_REQUIRE_CTX(ctx);
  if (!b || !x) {
    vts::set_error(VTS_E_ARGUMENT, "vts_minres_generic: NULL vector");
    return VTS_E_ARGUMENT;
  }
  int it = 0, conv = 0;
  double rr = 0.0;
  const int rc = vts::minres_generic(C(ctx), len, b, x, x0, tol, max_iters, floor_tol, op, precond, user, &it, &rr,
                                     &conv, history);
  if (iterations) *iterations = it;
  if (relres) *relres = rr;
  if (converged) *converged = conv;
  return rc;
}

int vts_bind_stiffness(vts_ctx* ctx, const double* rho, uint32_t* warn_flags) {
  VTS_REQUIRE_CTX(ctx);
  if (!rho) {
    vts::set_error(VTS_E_ARGUMENT, "vts_bind_stiffness: NULL rho");
    return VTS_E_ARGUMENT;
  }
  unsigned warn = 0;
  const int rc = C(ctx)->dim == 3 ? vts::h3_bind_stiffness(C(ctx), rho, &warn) : vts::bind_stiffness(C(ctx), rho, &warn);
  if (warn_flags) *warn_flags = warn;
  return rc;
}

int vts_element_products(vts_ctx* ctx, const double* u, double* w, double* q) {
  VTS_REQUIRE_CTX(ctx);
  if (!u || !q) {
    vts::set_error(VTS_E_ARGUMENT, "vts_element_products: NULL argument");
    return VTS_E_ARGUMENT;
  }
  return C(ctx)->dim == 3 ? vts::h3_element_products(C(ctx), u, w, q) : vts::element_energy(C(ctx), u, w, q);
}

int vts_doc_bisect(vts_ctx* ctx, const double* rho, const double* z, double z_scale, const double* lower,
                   const double* upper, double volume, double exponent, double alpha_hi, double tol, int32_t cap,
                   double* rho_new, double* alpha, int32_t* status) {
  VTS_REQUIRE_CTX(ctx);
  if (!rho || !z || !lower || !upper || !rho_new || !alpha || !status || cap < 0 || !(alpha_hi > 0.0)) {
    vts::set_error(VTS_E_ARGUMENT, "vts_doc_bisect: bad arguments");
    return VTS_E_ARGUMENT;
  }
  int st = 0;
  const int rc = vts::doc_bisect(C(ctx), rho, z, z_scale, lower, upper, volume, exponent, alpha_hi, tol, cap,
                                 rho_new, alpha, &st);
  *status = st;
  return rc;
}

int vts_doc_update(vts_ctx* ctx, const double* rho, const double* z, double z_scale, double alpha, double exponent,
                   const double* lower, const double* upper, double* rho_new) {
  VTS_REQUIRE_CTX(ctx);
  if (!rho || !z || !lower || !upper || !rho_new) {
    vts::set_error(VTS_E_ARGUMENT, "vts_doc_update: NULL argument");
    return VTS_E_ARGUMENT;
  }
  if (!(alpha > 0.0)) {
    vts::set_error(VTS_E_ARGUMENT, "volume multiplier must be positive");
    return VTS_E_ARGUMENT;
  }
  return vts::doc_update(C(ctx), rho, z, z_scale, alpha, exponent, lower, upper, rho_new);
}

int vts_doc_measure(vts_ctx* ctx, const double* rho_new, const double* rho, const double* q, const double* u,
                    const double* f, const double* lower, const double* upper, double volume, double* out) {
  VTS_REQUIRE_CTX(ctx);
  if (!rho_new || !rho || !q || !u || !f || !lower || !upper || !out) {
    vts::set_error(VTS_E_ARGUMENT, "vts_doc_measure: NULL argument");
    return VTS_E_ARGUMENT;
  }
  return vts::doc_measure(C(ctx), rho_new, rho, q, u, f, lower, upper, volume, out);
}

int vts_reconstruct_nu(vts_ctx* ctx, const double* u, const double* du, double dalpha, const double* res_u,
                       double res_alpha, const double* res_lo, const double* res_up, const double* a,
                       const double* b_lo, const double* b_up, double* dnu_lo, double* dnu_up, double* slope) {
  VTS_REQUIRE_CTX(ctx);
  if (C(ctx)->dim == 3)
    return vts::h3_reconstruct_nu(C(ctx), u, du, dalpha, res_u, res_alpha, res_lo, res_up, a, b_lo, b_up, dnu_lo,
                                  dnu_up, slope);
  const int rc = vts::reconstruct_nu(C(ctx), u, du, dalpha, res_u, res_alpha, res_lo, res_up, a, b_lo, b_up,
                                     dnu_lo, dnu_up, slope);
  if (rc) return rc;
  if (!slope) VTS_CUDA(cudaStreamSynchronize(C(ctx)->stream));
  return 0;
}

int vts_al_value(vts_ctx* ctx, const double* u, double alpha, const double* nu_lo, const double* nu_up,
                 const double* du, double dalpha, const double* dnu_lo, const double* dnu_up, double kappa,
                 const double* rho, const double* p, const double* mu_lo, const double* mu_up, const double* q_lo,
                 const double* q_up, const double* f, const double* lower, const double* upper, double volume,
                 double branch, double* value, uint32_t* warn_flags) {
  VTS_REQUIRE_CTX(ctx);
  unsigned warn = 0;
  auto* fn = C(ctx)->dim == 3 ? vts::h3_al_value : vts::al_value;
  const int rc = fn(C(ctx), u, alpha, nu_lo, nu_up, du, dalpha, dnu_lo, dnu_up, kappa, rho, p, mu_lo,
                               mu_up, q_lo, q_up, f, lower, upper, volume, branch, value, &warn);
  if (warn_flags) *warn_flags = warn ? VTS_W_SATURATED : 0u;
  return rc;
}

int vts_axpy(vts_ctx* ctx, int64_t len, double kappa, const double* dx, double* x) {
  VTS_REQUIRE_CTX(ctx);
  return vts::axpy(C(ctx), len, kappa, dx, x);
}

int vts_outer_update(vts_ctx* ctx, double beta, double gamma, double floor_p, const double* rho_hat,
                     const double* mu_hat_lo, const double* mu_hat_up, double* rho, double* mu_lo, double* mu_up,
                     double* p, double* q_lo, double* q_up, int32_t update_penalties) {
  VTS_REQUIRE_CTX(ctx);
  return vts::outer_update(C(ctx), beta, gamma, floor_p, rho_hat, mu_hat_lo, mu_hat_up, rho, mu_lo, mu_up, p, q_lo,
                           q_up, update_penalties);
}

int vts_gap(vts_ctx* ctx, const double* u, double alpha, const double* q, const double* f, const double* nu_lo,
            const double* nu_up, const double* lower, const double* upper, double volume, const double* rho,
            double* d_val, double* gap, double* fu, double* rho_sum) {
  VTS_REQUIRE_CTX(ctx);
  return vts::gap(C(ctx), u, alpha, q, f, nu_lo, nu_up, lower, upper, volume, rho, d_val, gap, fu, rho_sum);
}

int vts_penalty_eval(vts_ctx* ctx, int64_t n, const double* tau, double branch, double* value, double* d1,
                     double* d2, uint32_t* warn_flags) {
  VTS_REQUIRE_CTX(ctx);
  unsigned warn = 0;
  const int rc = vts::penalty_eval(C(ctx), n, tau, branch, value, d1, d2, &warn);
  if (warn_flags) *warn_flags = warn ? VTS_W_SATURATED : 0u;
  return rc;
}

int vts_newton_step(vts_ctx* ctx, const vts_newton_step_args* args, vts_newton_step_result* result) {
  VTS_REQUIRE_CTX(ctx);
  VTS_REQUIRE_2D(ctx);
  if (!args || !result) {
    vts::set_error(VTS_E_ARGUMENT, "vts_newton_step: NULL argument");
    return VTS_E_ARGUMENT;
  }
  return vts::newton_step(C(ctx), args, result);
}

int vts_time_kernels(vts_ctx* ctx, int32_t reps, double* ms) {
  VTS_REQUIRE_CTX(ctx);
  VTS_REQUIRE_2D(ctx);
  return vts::time_kernels(C(ctx), reps, ms);
}

int vts_time_cold(vts_ctx* ctx, int32_t reps, void* flush, int64_t flush_bytes, double* ms) {
  VTS_REQUIRE_CTX(ctx);
  VTS_REQUIRE_2D(ctx);
  if (reps < 1 || !flush || flush_bytes <= 0 || !ms) {
    vts::set_error(4, "vts_time_cold: bad arguments");
    return 4;
  }
  return vts::time_cold(C(ctx), reps, flush, (size_t)flush_bytes, ms);
}

int vts_ip_residual(vts_ctx* ctx, const double* u, double alpha, const double* rho, const double* nu_lo,
                    const double* nu_up, double r, double s, const double* lower, const double* upper, double volume,
                    const double* f, double norm_f, double* q, double* res_c, double* res_lo, double* res_up,
                    double* res_u, double* scalars) {
  VTS_REQUIRE_CTX(ctx);
  VTS_REQUIRE_2D(ctx);
  if (!u || !rho || !nu_lo || !nu_up || !lower || !upper || !f || !q || !res_c || !res_lo || !res_up || !res_u ||
      !scalars) {
    vts::set_error(VTS_E_ARGUMENT, "vts_ip_residual: NULL argument");
    return VTS_E_ARGUMENT;
  }
  return vts::ip_residual(C(ctx), u, alpha, rho, nu_lo, nu_up, r, s, lower, upper, volume, f, norm_f, q, res_c,
                          res_lo, res_up, res_u, scalars);
}

int vts_ip_schur_system(vts_ctx* ctx, const double* u, const double* rho, const double* nu_lo, const double* nu_up,
                        const double* lower, const double* upper, const double* res_c, const double* res_lo,
                        const double* res_up, const double* res_u, double res_alpha, double* dcoef, double* g,
                        double* rhs, double* corner) {
  VTS_REQUIRE_CTX(ctx);
  VTS_REQUIRE_2D(ctx);
  if (!u || !rho || !nu_lo || !nu_up || !lower || !upper || !res_c || !res_lo || !res_up || !res_u || !dcoef || !g ||
      !rhs) {
    vts::set_error(VTS_E_ARGUMENT, "vts_ip_schur_system: NULL argument");
    return VTS_E_ARGUMENT;
  }
  return vts::ip_schur_system(C(ctx), u, rho, nu_lo, nu_up, lower, upper, res_c, res_lo, res_up, res_u, res_alpha,
                              dcoef, g, rhs, corner);
}

int vts_ip_reconstruct(vts_ctx* ctx, const double* u, const double* du, double dalpha, const double* dcoef,
                       const double* g, const double* res_c, const double* res_lo, const double* res_up,
                       const double* rho, const double* nu_lo, const double* nu_up, const double* lower,
                       const double* upper, double* drho, double* dnu_up, double* dnu_lo) {
  VTS_REQUIRE_CTX(ctx);
  VTS_REQUIRE_2D(ctx);
  if (!u || !du || !dcoef || !g || !res_c || !res_lo || !res_up || !rho || !nu_lo || !nu_up || !lower || !upper ||
      !drho || !dnu_up || !dnu_lo) {
    vts::set_error(VTS_E_ARGUMENT, "vts_ip_reconstruct: NULL argument");
    return VTS_E_ARGUMENT;
  }
  return vts::ip_reconstruct(C(ctx), u, du, dalpha, dcoef, g, res_c, res_lo, res_up, rho, nu_lo, nu_up, lower, upper,
                             drho, dnu_up, dnu_lo);
}

int vts_ip_step_bounds(vts_ctx* ctx, const double* rho, const double* drho, const double* nu_lo,
                       const double* dnu_lo, const double* nu_up, const double* dnu_up, const double* lower,
                       const double* upper, double* mins) {
  VTS_REQUIRE_CTX(ctx);
  VTS_REQUIRE_2D(ctx);
  if (!rho || !drho || !nu_lo || !dnu_lo || !nu_up || !dnu_up || !lower || !upper || !mins) {
    vts::set_error(VTS_E_ARGUMENT, "vts_ip_step_bounds: NULL argument");
    return VTS_E_ARGUMENT;
  }
  return vts::ip_step_bounds(C(ctx), rho, drho, nu_lo, dnu_lo, nu_up, dnu_up, lower, upper, mins);
}

int64_t vts_kernel_launches(const vts_ctx* ctx) { return ctx ? C(ctx)->launches : 0; }

int vts_profile_begin(vts_ctx* ctx) {
  VTS_REQUIRE_CTX(ctx);
  VTS_REQUIRE_2D(ctx);
  return vts::profile_begin(C(ctx));
}

int vts_profile_end(vts_ctx* ctx, double* out) {
  VTS_REQUIRE_CTX(ctx);
  if (!out) {
    vts::set_error(4, "vts_profile_end: out is NULL");
    return 4;
  }
  return vts::profile_end(C(ctx), out);
}

}  // extern "C"
