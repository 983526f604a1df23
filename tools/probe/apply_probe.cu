// Standalone probe of the Newton apply through the library internals: builds a
// cantilever hierarchy, a synthetic Newton system, the multigrid, then times
// single sweeps per level and the V-cycle.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o gs_probe gs_probe.cu
#include "../../paper_1904_06556_b200/csrc/vts_b200.cu"
#include <cstdio>
#include <random>
#include <vector>

int main(int argc, char** argv) {
  const int levels = argc > 1 ? atoi(argv[1]) : 3;
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
  double ke[64];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) ke[8 * i + j] = (i == j ? 0.5 : -0.5 / 7.0);
  vts_ctx* h = nullptr;
  if (vts_ctx_create(&h, levels, ex.data(), ey.data(), ptrs.data(), ke, 0)) {
    printf("create failed: %s\n", vts_last_error());
    return 1;
  }
  vts::Ctx* c = reinterpret_cast<vts::Ctx*>(h);
  vts::ensure_ke(c);
  std::mt19937_64 g(1);
  std::uniform_real_distribution<double> u(-0.01, 0.01), pos(0.5, 2.0);
  std::vector<double> ug(c->lv[levels - 1].d.ngrid), rh(c->m), ch(c->m);
  for (auto& v : ug) v = u(g);
  for (auto& v : rh) v = pos(g);
  for (auto& v : ch) v = 1e-3 * pos(g);
  cudaMemcpy(c->u_grid, ug.data(), ug.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(c->rho_hat, rh.data(), rh.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(c->chat, ch.data(), ch.size() * 8, cudaMemcpyHostToDevice);
  double corner = 1.0;
  cudaMemcpy(c->d_corner, &corner, 8, cudaMemcpyHostToDevice);
  c->system_bound = true;
  if (vts::mg_setup(c, 1e-12)) {
    printf("mg_setup failed: %s\n", vts_last_error());
    return 1;
  }
  fprintf(stderr, "setup done\n");
  double* xin = c->fvec[10];
  double* yout = c->fvec[11];
  cudaMemset(xin, 0, (c->lv[levels - 1].d.ngrid + 1) * 8);
  fprintf(stderr, "memset done\n");
  int rc = vts::newton_apply_grid(c, xin, yout, nullptr);
  fprintf(stderr, "launched\n");
  cudaError_t err = cudaDeviceSynchronize();
  fprintf(stderr, "sync: %s\n", cudaGetErrorString(err));
  fprintf(stderr, "rc %d\n", rc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 20; ++r) vts::newton_apply_grid(c, xin, yout, nullptr);
  cudaEventRecord(e1);
  err = cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("apply: %.2f us (%s)\n", ms * 1e3 / 20, cudaGetErrorString(err));
  vts_ctx_destroy(h);
  return 0;
}
