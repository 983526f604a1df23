// Standalone probe of the GS wavefront through the library internals: builds a
// cantilever hierarchy, a synthetic Newton system, the multigrid, then times
// single sweeps per level and the V-cycle.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o gs_probe gs_probe.cu
#include "../../paper_1904_06556_b200/csrc/vts_b200.cu"
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

int main(int argc, char** argv) {
  const int levels = argc > 1 ? atoi(argv[1]) : 9;
  const int base = argc > 2 ? atoi(argv[2]) : 4;  // coarsest elements in x (y = base / 2)
  std::vector<int32_t> ex(levels), ey(levels);
  std::vector<std::vector<int64_t>> dofs(levels);
  std::vector<const int64_t*> ptrs(levels);
  for (int k = 0; k < levels; ++k) {
    ex[k] = base << k;
    ey[k] = (base / 2) << k;
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
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int k = levels - 1; k >= std::max(0, levels - 4); --k) {
    vts::LevelBuf& L = c->lv[k];
    for (int variant = 0; variant < 3; ++variant) {
      const bool fwd = variant < 2, zero = variant == 0;
      vts::gs_sweep(c, k, L.b, L.x, fwd, zero, nullptr);
      cudaEventRecord(e0);
      const int reps = 5;
      for (int r = 0; r < reps; ++r) vts::gs_sweep(c, k, L.b, L.x, fwd, zero, nullptr);
      cudaEventRecord(e1);
      cudaError_t err = cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= reps;
      const int steps = L.d.nx + 2 * L.d.ny;
      printf("level %d (%d x %d) %s%s sweep: %8.1f us  (%s) ~%.0f cycles/step\n", k, L.d.nx, L.d.ny,
             fwd ? "fwd" : "bwd", zero ? "-zero" : "     ", ms * 1e3, cudaGetErrorString(err), ms * 1.965e6 / steps);
    }
  }
#ifdef VTS_GS_PROBE
  {
    vts::LevelBuf& L = c->lv[levels - 1];
    vts::gs_sweep(c, levels - 1, L.b, L.x, true, false, nullptr);
    cudaDeviceSynchronize();
    std::vector<long long> pr(4 * 256);
    cudaMemcpyFromSymbol(pr.data(), vts::g_gs_probe, pr.size() * 8);
    const int bands = (L.d.ny + vts::gs::R - 1) / vts::gs::R;
    std::vector<long long> p2(2 * 256), p3(2 * 256);
    cudaMemcpyFromSymbol(p2.data(), vts::g_gs_probe2, p2.size() * 8);
    cudaMemcpyFromSymbol(p3.data(), vts::g_gs_probe3, p3.size() * 8);
    long long t0 = pr[0];
    const int nwin = (L.d.nx + vts::gs::SKEW * (vts::gs::R - 1) + vts::gs::W - 1) / vts::gs::W;
    printf("W %d, %d windows per band\n", vts::gs::W, nwin);
    for (int b = 0; b < bands; ++b)
      printf("band %2d: start %7.1f us  first-window %7.1f  end %7.1f  (dur %6.1f, above %6.1f, in %5.1f, out %5.1f, "
             "loops %6.1f = %4.0f ns/step, end-of-window %5.1f us)\n", b,
             (pr[4 * b] - t0) / 1e3, (pr[4 * b + 1] - t0) / 1e3, (pr[4 * b + 2] - t0) / 1e3,
             (pr[4 * b + 2] - pr[4 * b + 1]) / 1e3, pr[4 * b + 3] / 1e3, p2[2 * b] / 1e3, p2[2 * b + 1] / 1e3,
             p3[2 * b] / 1e3, p3[2 * b] / double(nwin * vts::gs::W), p3[2 * b + 1] / 1e3);
  }
  {  // pair timeline: sweep A bands (probe slots 0..) and sweep B bands (128..)
    vts::LevelBuf& L = c->lv[levels - 1];
    vts::gs_two_sweeps(c, levels - 1, L.b, L.x, false, false, nullptr);
    cudaDeviceSynchronize();
    std::vector<long long> pr(4 * 256);
    cudaMemcpyFromSymbol(pr.data(), vts::g_gs_probe, pr.size() * 8);
    std::vector<long long> pr2(2 * 256);
    cudaMemcpyFromSymbol(pr2.data(), vts::g_gs_probe2, pr2.size() * 8);
    std::vector<long long> pr3(2 * 256);
    cudaMemcpyFromSymbol(pr3.data(), vts::g_gs_probe3, pr3.size() * 8);
    const int bands = (L.d.ny + vts::gs::R - 1) / vts::gs::R;
    long long t0 = pr[0];
    printf("pair timeline (bwd pair, finest):\n");
    for (int b : {0, 1, 2, 10, 11, 16, 22, 32}) {
      if (b >= bands) continue;
      for (int role = 0; role < 2; ++role) {
        const int i = b + 128 * role;
        printf("  %s band %2d: start %7.1f  first-window %7.1f  end %7.1f  (dur %6.1f, waiting-above %6.1f, in %6.1f, out %6.1f, "
               "loops %6.1f, end-of-window %5.1f)\n",
               role ? "B" : "A", b, (pr[4 * i] - t0) / 1e3, (pr[4 * i + 1] - t0) / 1e3, (pr[4 * i + 2] - t0) / 1e3,
               (pr[4 * i + 2] - pr[4 * i + 1]) / 1e3, pr[4 * i + 3] / 1e3, pr2[2 * i] / 1e3, pr2[2 * i + 1] / 1e3,
               pr3[2 * i] / 1e3, pr3[2 * i + 1] / 1e3);
      }
    }
  }
#endif
  double* xin = c->fvec[10];
  double* yout = c->fvec[11];
  vts::vcycle_grid(c, xin, yout, nullptr);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) vts::vcycle_grid(c, xin, yout, nullptr);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("V-cycle: %.1f us (%s)\n", ms * 1e3 / 5, cudaGetErrorString(err));
#ifdef VTS_TIMELINE
  for (int rep = 0; rep < 2; ++rep) {  // kernel timeline of one V-cycle (first block start, last block end)
    std::vector<unsigned long long> tl(160 * 2);
    for (int i = 0; i < 160; ++i) {
      tl[2 * i] = ~0ull;
      tl[2 * i + 1] = 0;
    }
    cudaMemcpyToSymbol(vts::g_tl, tl.data(), tl.size() * 8);
    cudaDeviceSynchronize();
    vts::vcycle_grid(c, xin, yout, nullptr);
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(tl.data(), vts::g_tl, tl.size() * 8);
    unsigned long long t0 = ~0ull, t1 = 0;
    for (int i = 0; i < 160; ++i)
      if (tl[2 * i] != ~0ull) t0 = std::min(t0, tl[2 * i]), t1 = std::max(t1, tl[2 * i + 1]);
    static const char* names[10] = {"desc pair", "asc pair", "resid+restrict rows", "prolong rows", "bottom",
                                     "alpha residual", "residual", "restrict", "prolong_add", "level apply"};
    printf("timeline rep %d: %.1f us first start -> last end\n", rep, (t1 - t0) / 1e3);
    std::vector<std::pair<unsigned long long, int>> order;
    for (int i = 0; i < 160; ++i)
      if (tl[2 * i] != ~0ull) order.push_back({tl[2 * i], i});
    std::sort(order.begin(), order.end());
    for (auto& o : order) {
      const int i = o.second;
      printf("  %-20s L%-2d start %7.1f  end %7.1f  (%6.1f us)\n", names[i / 16], i % 16, (tl[2 * i] - t0) / 1e3,
             tl[2 * i + 1] ? (tl[2 * i + 1] - t0) / 1e3 : -1.0, tl[2 * i + 1] ? (tl[2 * i + 1] - tl[2 * i]) / 1e3 : 0.0);
    }
    if (rep == 1) {  // the finest level's residual/restriction items: wait and work times
      std::vector<unsigned long long> it(1024 * 4);
      cudaMemcpyFromSymbol(it.data(), vts::g_items, it.size() * 8);
      const int R = vts::gs::R, cb = (c->lv[levels - 2].d.ny + R - 1) / R, items = cb * 3 * vts::kSeg;
      double work_sum = 0.0, wait_sum = 0.0;
      std::vector<std::pair<double, int>> ends;
      for (int i = 0; i < items && i < 1024; ++i) {
        if (!it[4 * i + 2]) continue;
        work_sum += (it[4 * i + 2] - it[4 * i + 1]) / 1e3;
        wait_sum += (it[4 * i + 1] - it[4 * i]) / 1e3;
        ends.push_back({(it[4 * i + 2] - t0) / 1e3, i});
      }
      std::sort(ends.begin(), ends.end());
      printf("  finest resid/restrict items: %d, mean work %.2f us, mean wait %.2f us; last 12:\n", (int)ends.size(),
             work_sum / std::max<size_t>(1, ends.size()), wait_sum / std::max<size_t>(1, ends.size()));
      for (size_t k = ends.size() > 12 ? ends.size() - 12 : 0; k < ends.size(); ++k) {
        const int i = ends[k].second;
        printf("    item %3d (block %2llu, q %2d): wait from %7.1f, work %7.1f -> %7.1f (%.1f us)\n", i, it[4 * i + 3],
               i % (3 * vts::kSeg), (it[4 * i] - t0) / 1e3, (it[4 * i + 1] - t0) / 1e3, (it[4 * i + 2] - t0) / 1e3,
               (it[4 * i + 2] - it[4 * i + 1]) / 1e3);
      }
    }
#ifdef VTS_GS_PROBE
    if (rep == 1) {  // bands of the ascent pair of the level VTS_PROBE_LEVEL (default: finest) inside the V-cycle
      const int plev = getenv("VTS_PROBE_LEVEL") ? atoi(getenv("VTS_PROBE_LEVEL")) : levels - 1;
      const int pnx = c->lv[plev].d.nx;
      cudaMemcpyToSymbol(vts::g_gs_probe_nx, &pnx, 4);
      vts::vcycle_grid(c, xin, yout, nullptr);
      cudaDeviceSynchronize();
      std::vector<long long> pr(4 * 256), p2(2 * 256), p3(2 * 256);
      cudaMemcpyFromSymbol(pr.data(), vts::g_gs_probe, pr.size() * 8);
      cudaMemcpyFromSymbol(p2.data(), vts::g_gs_probe2, p2.size() * 8);
      cudaMemcpyFromSymbol(p3.data(), vts::g_gs_probe3, p3.size() * 8);
      const int zero = 0;
      cudaMemcpyToSymbol(vts::g_gs_probe_nx, &zero, 4);
      const int bands = (c->lv[plev].d.ny + vts::gs::R - 1) / vts::gs::R;
      long long b0 = pr[0];
      printf("  level %d asc pair bands (us from A band 0's start; wait-above / wait-in / wait-out / loops):\n", plev);
      for (int b = 0; b < bands; ++b)
        for (int h = 0; h < 2; ++h) {
          const int i = b + 128 * h;
          printf("   %c band %2d: start %7.1f first %7.1f end %7.1f | above %6.1f in %6.1f out %6.1f loops %6.1f\n", h ? 'B' : 'A', b,
                 (pr[4 * i] - b0) / 1e3, (pr[4 * i + 1] - b0) / 1e3, (pr[4 * i + 2] - b0) / 1e3, pr[4 * i + 3] / 1e3,
                 p2[2 * i] / 1e3, p2[2 * i + 1] / 1e3, p3[2 * i] / 1e3);
        }
    }
#endif
  }
#endif
#ifdef VTS_BOT_PROBE
  {  // marks of the fused bottom in the last of several back-to-back V-cycles
    for (int r = 0; r < 6; ++r) vts::vcycle_grid(c, xin, yout, nullptr);
    cudaDeviceSynchronize();
    int n = 0;
    long long pr[64];
    cudaMemcpyFromSymbol(&n, vts::g_bot_n, 4);
    cudaMemcpyFromSymbol(pr, vts::g_bot_probe, 64 * 8);
    for (int i = 1; i < n; ++i) printf("bottom mark %2d: +%6.2f us  (at %7.2f)\n", i, (pr[i] - pr[i - 1]) / 1e3, (pr[i] - pr[0]) / 1e3);
    printf("bottom total (first to last mark): %.1f us\n", (pr[n - 1] - pr[0]) / 1e3);
  }
#endif
  {  // determinism: the V-cycle on fixed input, bitwise, many times
    const size_t n = c->lv[levels - 1].d.ngrid + 1;
    std::vector<double> r0(n), r1(n);
    vts::vcycle_grid(c, xin, yout, nullptr);
    cudaMemcpy(r0.data(), yout, n * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    const int nrep = getenv("VTS_DET_REPS") ? atoi(getenv("VTS_DET_REPS")) : 200;
    for (int r = 0; r < nrep; ++r) {
      vts::vcycle_grid(c, xin, yout, nullptr);
      cudaMemcpy(r1.data(), yout, n * 8, cudaMemcpyDeviceToHost);
      if (memcmp(r0.data(), r1.data(), n * 8) != 0) {
        ++bad;
        size_t first = 0;
        while (first < n && r0[first] == r1[first]) ++first;
        if (bad <= 3) printf("determinism: rep %d differs first at %zu (%.17g vs %.17g)\n", r, first, r0[first], r1[first]);
      }
    }
    printf("determinism: %d of %d V-cycles differ\n", bad, nrep);
  }
  vts_ctx_destroy(h);
  return 0;
}
