// Single-warp fp64 issue rate: cycles per warp-DFMA with 8 independent chains,
// all 32 lanes vs 16 active lanes, and DFMA vs LDS.128 mix.
#include <cstdio>
__global__ void k(double* out, long long* cyc, int active, int iters) {
  const int l = threadIdx.x;
  double a0 = l, a1 = l + 1, a2 = l + 2, a3 = l + 3, a4 = l + 4, a5 = l + 5, a6 = l + 6, a7 = l + 7;
  const double m = 0.999999, c = 1e-9;
  long long t0 = clock64();
  if (l < active) {
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
        a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
      }
    }
  }
  __syncwarp();
  long long t1 = clock64();
  out[l] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (l == 0) *cyc = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024); cudaMalloc(&c, 8);
  for (int act : {32, 16, 8, 1}) {
    const int iters = 1000;
    k<<<1, 32>>>(o, c, act, iters);
    cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("active lanes %2d: %.2f cycles per warp-DFMA (8 independent chains)\n", act, (double)h / (iters * 64.0));
  }
  return 0;
}
