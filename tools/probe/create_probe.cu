// Times vts_ctx_create / vts_ctx_destroy on the 1024x512 cantilever hierarchy
// (9 levels) to see what context construction costs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o create_probe create_probe.cu -lcuda
#include <chrono>
#include <cstdio>
static double g_t0;
static double tnow() { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
#define VTS_CREATE_MARK(s) fprintf(stderr, "  %-10s %.2f ms\n", s, tnow() - g_t0)
#include "../../paper_1904_06556_b200/csrc/vts_b200.cu"
#include <chrono>
#include <cstdio>
#include <vector>

static double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
  const int levels = argc > 1 ? atoi(argv[1]) : 9;
  std::vector<int32_t> ex(levels), ey(levels);
  std::vector<std::vector<int64_t>> dofs(levels);
  std::vector<const int64_t*> ptrs(levels);
  for (int k = 0; k < levels; ++k) {
    ex[k] = 4 << k;
    ey[k] = 2 << k;
    const int nx = ex[k] + 1, ny = ey[k] + 1;
    dofs[k].assign(2 * nx * ny, -1);
    int64_t n = 0;
    for (int iy = 0; iy < ny; ++iy)
      for (int ix = 0; ix < nx; ++ix)
        for (int c = 0; c < 2; ++c)
          if (ix > 0) dofs[k][2 * (iy * nx + ix) + c] = n++;
    ptrs[k] = dofs[k].data();
  }
  double ke[64] = {};
  for (int i = 0; i < 8; ++i) ke[9 * i] = 1.0;
  cudaFree(nullptr);
  for (int rep = 0; rep < 4; ++rep) {
    vts_ctx* h = nullptr;
    double t0 = now_ms();
    g_t0 = tnow();
    int rc = vts_ctx_create(&h, levels, ex.data(), ey.data(), ptrs.data(), ke, 0);
    double t1 = now_ms();
    vts_ctx_destroy(h);
    double t2 = now_ms();
    printf("create %.2f ms (rc %d), destroy %.2f ms\n", t1 - t0, rc, t2 - t1);
  }
  return 0;
}
