#include <cstdio>
__global__ void k(double* out, int n, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < n; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void k16(double* out, int n, double a, double b) {  // half the lanes active
  if ((threadIdx.x & 31) >= 16) return;
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < n; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  double* out; cudaMalloc(&out, 148 * 8 * 256 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int n = 20000;
  for (int blocks : {148 * 8, 1, 4}) {
    for (int threads : {256, 32}) {
      k<<<blocks, threads>>>(out, n, 0.999, 1e-3);
      cudaEventRecord(e0); k<<<blocks, threads>>>(out, n, 0.999, 1e-3); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 8 * n * (double)blocks * threads;
      printf("blocks %5d threads %4d: %8.3f ms  %8.2f TFLOP/s  (%.2f cycles per warp-DFMA per warp)\n", blocks, threads, ms,
             fl / ms / 1e9, ms * 1e-3 * 1.965e9 / (8.0 * n));
      k16<<<blocks, threads>>>(out, n, 0.999, 1e-3);
      cudaEventRecord(e0); k16<<<blocks, threads>>>(out, n, 0.999, 1e-3); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("   16-lane variant: %8.3f ms (%.2f cycles per warp-DFMA)\n", ms, ms * 1e-3 * 1.965e9 / (8.0 * n));
    }
  }
  return 0;
}
