// Microbenchmarks that size the wavefront Gauss-Seidel design on B200:
// fp64 dependent-op latency, shuffle latency, cross-SM flag hand-off latency
// through L2, DSMEM hand-off inside a cluster, single-SM streaming bandwidth.
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint64_t clk() { uint64_t c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)); return c; }

__global__ void k_dfma(double* out, long long* cyc, int n, double a, double b) {
  double x = out[threadIdx.x];
  uint64_t t0 = clk();
  for (int i = 0; i < n; ++i) { x = fma(x, a, b); }
  uint64_t t1 = clk();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = (long long)(t1 - t0);
}
__global__ void k_dmul(double* out, long long* cyc, int n, double a) {
  double x = out[threadIdx.x];
  uint64_t t0 = clk();
  for (int i = 0; i < n; ++i) { x = x * a; }
  uint64_t t1 = clk();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = (long long)(t1 - t0);
}
__global__ void k_ddiv(double* out, long long* cyc, int n, double a) {
  double x = out[threadIdx.x];
  uint64_t t0 = clk();
  for (int i = 0; i < n; ++i) { x = a / x; }
  uint64_t t1 = clk();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = (long long)(t1 - t0);
}
__global__ void k_shfl(double* out, long long* cyc, int n) {
  double x = out[threadIdx.x];
  uint64_t t0 = clk();
  for (int i = 0; i < n; ++i) { x = __shfl_up_sync(0xffffffffu, x, 1) + 1.0; }
  uint64_t t1 = clk();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = (long long)(t1 - t0);
}
__global__ void k_smem_pingpong(long long* cyc, int n) {
  // warp 0 lane 0 and warp 1 lane 0 ping-pong through a shared flag
  __shared__ volatile int flag;
  if (threadIdx.x == 0) flag = 0;
  __syncthreads();
  int w = threadIdx.x / 32;
  if ((threadIdx.x & 31) == 0 && w < 2) {
    uint64_t t0 = clk();
    for (int i = 0; i < n; ++i) {
      if (w == 0) { while (flag != 2 * i) {} flag = 2 * i + 1; }
      else { while (flag != 2 * i + 1) {} flag = 2 * i + 2; }
    }
    uint64_t t1 = clk();
    if (w == 0) cyc[0] = (long long)(t1 - t0);
  }
}
__global__ void k_gmem_pingpong(int* flag, long long* cyc, int n) {
  // block 0 and block 1 (different SMs) ping-pong through a global flag
  if (threadIdx.x != 0) return;
  int b = blockIdx.x;
  uint64_t t0 = clk();
  for (int i = 0; i < n; ++i) {
    if (b == 0) {
      int v; do { asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag)); } while (v != 2 * i);
      asm volatile("st.release.gpu.global.b32 [%0], %1;" :: "l"(flag), "r"(2 * i + 1));
    } else {
      int v; do { asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag)); } while (v != 2 * i + 1);
      asm volatile("st.release.gpu.global.b32 [%0], %1;" :: "l"(flag), "r"(2 * i + 2));
    }
  }
  uint64_t t1 = clk();
  if (b == 0) cyc[0] = (long long)(t1 - t0);
}
__global__ void k_gmem_pingpong_relaxed(int* flag, long long* cyc, int n) {
  if (threadIdx.x != 0) return;
  int b = blockIdx.x;
  volatile int* f = flag;
  uint64_t t0 = clk();
  for (int i = 0; i < n; ++i) {
    if (b == 0) { while (f[0] != 2 * i) {} __threadfence(); f[0] = 2 * i + 1; }
    else { while (f[0] != 2 * i + 1) {} __threadfence(); f[0] = 2 * i + 2; }
  }
  uint64_t t1 = clk();
  if (b == 0) cyc[0] = (long long)(t1 - t0);
}
__global__ void __cluster_dims__(2, 1, 1) k_dsmem_pingpong(long long* cyc, int n) {
  __shared__ int flag;
  cg::cluster_group cl = cg::this_cluster();
  if (threadIdx.x == 0) flag = 0;
  cl.sync();
  int r = cl.block_rank();
  int* peer = cl.map_shared_rank(&flag, 0);  // both use block 0's flag
  if (threadIdx.x == 0) {
    volatile int* f = peer;
    uint64_t t0 = clk();
    for (int i = 0; i < n; ++i) {
      if (r == 0) { while (f[0] != 2 * i) {} f[0] = 2 * i + 1; }
      else { while (f[0] != 2 * i + 1) {} f[0] = 2 * i + 2; }
    }
    uint64_t t1 = clk();
    if (r == 0) cyc[0] = (long long)(t1 - t0);
  }
  cl.sync();
}
__global__ void k_stream(const double2* __restrict__ in, double* out, long long per_block) {
  // each block streams its own contiguous chunk with plain 16B loads
  const double2* p = in + blockIdx.x * per_block;
  double s = 0;
  for (long long i = threadIdx.x; i < per_block; i += blockDim.x * 4) {
    double2 a = p[i];
    double2 b = (i + blockDim.x < per_block) ? p[i + blockDim.x] : make_double2(0, 0);
    double2 c = (i + 2 * blockDim.x < per_block) ? p[i + 2 * blockDim.x] : make_double2(0, 0);
    double2 d = (i + 3 * blockDim.x < per_block) ? p[i + 3 * blockDim.x] : make_double2(0, 0);
    s += a.x + a.y + b.x + b.y + c.x + c.y + d.x + d.y;
  }
  if (s == 12345.678) out[0] = s;
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

int main() {
  double* d; long long* c; int* flag; long long h;
  CK(cudaMalloc(&d, 1024 * sizeof(double))); CK(cudaMemset(d, 0, 1024 * sizeof(double)));
  CK(cudaMalloc(&c, 64)); CK(cudaMalloc(&flag, 64));
  const int N = 4096;
  k_dfma<<<1, 32>>>(d, c, N, 0.999, 1e-3); CK(cudaDeviceSynchronize());
  k_dfma<<<1, 32>>>(d, c, N, 0.999, 1e-3); CK(cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost));
  printf("DFMA dependent latency: %.2f cyc\n", (double)h / N);
  k_dmul<<<1, 32>>>(d, c, N, 0.9999); CK(cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost));
  printf("DMUL dependent latency: %.2f cyc\n", (double)h / N);
  CK(cudaMemset(d, 0, 1024 * sizeof(double)));
  { double one = 1.0; for (int i = 0; i < 32; ++i) CK(cudaMemcpy(d + i, &one, 8, cudaMemcpyHostToDevice)); }
  k_ddiv<<<1, 32>>>(d, c, N, 1.5); CK(cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost));
  printf("DDIV dependent latency: %.2f cyc\n", (double)h / N);
  k_shfl<<<1, 32>>>(d, c, N); CK(cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost));
  printf("fp64 shfl_up + dadd latency: %.2f cyc\n", (double)h / N);
  k_smem_pingpong<<<1, 64>>>(c, N); CK(cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost));
  printf("smem flag round trip (warp<->warp): %.2f cyc\n", (double)h / N);
  CK(cudaMemset(flag, 0, 64));
  k_gmem_pingpong<<<2, 32>>>(flag, c, N); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost));
  printf("gmem acquire/release round trip (SM<->SM): %.2f cyc\n", (double)h / N);
  CK(cudaMemset(flag, 0, 64));
  k_gmem_pingpong_relaxed<<<2, 32>>>(flag, c, N); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost));
  printf("gmem volatile+fence round trip (SM<->SM): %.2f cyc\n", (double)h / N);
  k_dsmem_pingpong<<<2, 32>>>(c, N); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost));
  printf("DSMEM volatile round trip (cluster of 2): %.2f cyc\n", (double)h / N);
  // streaming bandwidth vs number of blocks
  size_t bytes = (size_t)1 << 30; double2* big; CK(cudaMalloc(&big, bytes)); CK(cudaMemset(big, 0, bytes));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int nb : {1, 2, 4, 8, 16, 32, 64, 148, 296, 592}) {
    for (int nt : {256, 1024}) {
      long long per = (long long)(bytes / 16) / 592;  // same bytes per block regardless of nb
      k_stream<<<nb, nt>>>(big, d, per);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) k_stream<<<nb, nt>>>(big, d, per);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double gbs = 5.0 * nb * per * 16 / (ms * 1e-3) / 1e9;
      printf("stream blocks=%d threads=%d : %.1f GB/s total, %.1f GB/s per block\n", nb, nt, gbs, gbs / nb);
    }
  }
  int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("clock attr %d kHz\n", clk_khz);
  return 0;
}
