// Isolated wavefront compute loop: cycles per step for variants (no helpers, data preloaded in smem).
#include <cstdio>
#include <cstdint>
constexpr int CH = 8, NS = 6, R = 16, HALF = 20, SKEW = 2;
struct Slot { double st[CH * HALF]; double2 p[CH]; double2 q[CH]; };
struct RowRing { Slot in[NS]; double2 out[NS][CH]; double2 pad; };

template <int VAR>
__global__ void k(int nx, double* sink, long long* cyc) {
  extern __shared__ __align__(128) unsigned char raw[];
  RowRing* rows = reinterpret_cast<RowRing*>(raw);
  const int l = threadIdx.x;
  for (int i = threadIdx.x; i < (int)(R * sizeof(RowRing) / 8); i += blockDim.x) reinterpret_cast<double*>(raw)[i] = 1e-3 * (i % 7);
  __syncthreads();
  const bool act = l < R;
  double2 win[SKEW + 1];
  for (int i = 0; i <= SKEW; ++i) win[i] = make_double2(0, 0);
  double2 wprev = make_double2(0, 0);
  const int T = nx + SKEW * (R - 1);
  long long t0 = clock64();
  for (int t = 0; t < T; ++t) {
    const int j = t - SKEW * l;
    double2 nv = make_double2(0, 0);
    const bool on = act && j >= 0 && j < nx;
    if (VAR == 3 ? act : on) {
      const int kk = j / CH;
      Slot& sl = rows[l].in[kk % NS];
      const int pos = j % CH;
      const double2* a2 = reinterpret_cast<const double2*>(sl.st + pos * HALF);
      double a[HALF];
      if (VAR == 5) { for (int i = 0; i < HALF; ++i) a[i] = 1e-3 * (i + 1); }
      else { for (int i = 0; i < HALF / 2; ++i) { const double2 v = a2[i]; a[2 * i] = v.x; a[2 * i + 1] = v.y; } }
      const double2 pp = (VAR == 5 || VAR == 6) ? make_double2(0.1, 0.2) : sl.p[pos];
      const double2 xm = win[0], xz = win[1], xp = win[2];
      double s0 = pp.x, s1 = pp.y;
      s0 = fma(-a[0], xm.x, s0); s0 = fma(-a[1], xm.y, s0); s0 = fma(-a[4], xz.x, s0); s0 = fma(-a[5], xz.y, s0);
      s0 = fma(-a[12], wprev.x, s0); s0 = fma(-a[13], wprev.y, s0); s0 = fma(-a[8], xp.x, s0); s0 = fma(-a[9], xp.y, s0);
      const double n0 = s0 * a[17];
      s1 = fma(-a[2], xm.x, s1); s1 = fma(-a[3], xm.y, s1); s1 = fma(-a[6], xz.x, s1); s1 = fma(-a[7], xz.y, s1);
      s1 = fma(-a[14], wprev.x, s1); s1 = fma(-a[15], wprev.y, s1); s1 = fma(-a[10], xp.x, s1); s1 = fma(-a[11], xp.y, s1);
      s1 = fma(-a[16], n0, s1);
      const double n1 = s1 * a[18];
      nv = make_double2(n0, n1);
      if (VAR != 4) rows[l].out[kk % NS][pos] = nv;
      wprev = nv;
    }
    double r0, r1;
    if (VAR == 1) { r0 = nv.x * 0.5; r1 = nv.y * 0.5; }
    else { r0 = __shfl_up_sync(0xffffffffu, nv.x, 1); r1 = __shfl_up_sync(0xffffffffu, nv.y, 1); }
    if (l == 0) { r0 = 0; r1 = 0; }
    for (int i = 0; i < SKEW; ++i) win[i] = win[i + 1];
    win[SKEW] = make_double2(r0, r1);
  }
  long long t1 = clock64();
  if (l == 0) cyc[0] = t1 - t0;
  sink[l] = wprev.x + wprev.y + win[0].x;
}

template <int VAR>
void run(const char* name) {
  double* sink; long long* cyc; cudaMalloc(&sink, 1024); cudaMalloc(&cyc, 8);
  const int smem = R * sizeof(RowRing);
  cudaFuncSetAttribute(k<VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int nx = 1025;
  k<VAR><<<1, 32, smem>>>(nx, sink, cyc); cudaDeviceSynchronize();
  k<VAR><<<1, 32, smem>>>(nx, sink, cyc);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-40s %6.1f cycles/step (%s)\n", name, (double)c / (nx + SKEW * (R - 1)), cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<0>("baseline (shfl, STS, predicated on)");
  run<1>("no shuffle");
  run<3>("no j-range predicate (act only)");
  run<4>("no STS");
  run<5>("no LDS at all (coefficients in regs)");
  run<6>("no P load");
  return 0;
}
