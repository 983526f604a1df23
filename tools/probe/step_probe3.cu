// What bounds the wavefront step?  The product's compute loop (gs_compute: gs_pre + gs_rec2, operands
// loaded two steps ahead, one store and one fp64 shuffle per step) on static shared-memory data, with
// parts of the step removed one at a time.  One warp, cycles per step by clock64.
//   V 0 product form   1 no store   2 no shuffle (own value instead)   3 no shared-memory loads in the loop
//   4 recurrence only (no gs_pre, no loads)   5 recurrence only, no shuffle   6 product form, 16 active lanes only
//   7 = 6 with lane 0's previous-row value by a predicated load instead of a load + selects
//   8 = 6 without the store   9 = 6 without shared-memory loads in the loop   10 = 7 without the lane mask on the store
#include <cstdio>
#include <cstdlib>
constexpr int R = 16, W = 17, HALF = 22;
struct InSlot {
  double st[R][W][HALF];
  double p[R][W][2];
};
struct Raw {
  double a[19];
  double2 p;
};
struct StepData {
  double q0, q1, w00, w01, w10, w11, c, r0, r1, e00, e01, e10, e11;
};
__device__ __forceinline__ void gs_pre(const double* a, double p0, double p1, double2 xm, double2 xz, double& q0, double& q1) {
  auto chain = [&](int d, double p) {
    double q = fma(-a[0 + 2 * d], xm.x, p);
    q = fma(-a[1 + 2 * d], xm.y, q);
    q = fma(-a[4 + 2 * d], xz.x, q);
    return fma(-a[5 + 2 * d], xz.y, q);
  };
  q0 = chain(0, p0);
  q1 = chain(1, p1);
}
__device__ __forceinline__ double2 gs_rec2(const StepData& c, double2 wp, double2 xq) {
  const double u0 = fma(-c.w01, wp.y, fma(-c.w00, wp.x, c.q0));
  const double u1 = fma(-c.w11, wp.y, fma(-c.w10, wp.x, c.q1));
  const double n0 = fma(-c.e01, xq.y, fma(-c.e00, xq.x, u0)) * c.r0;
  const double n1 = fma(-c.c, n0, fma(-c.e11, xq.y, fma(-c.e10, xq.x, u1))) * c.r1;
  return make_double2(n0, n1);
}
template <int V>
__global__ void __launch_bounds__(512, 1) k(double* sink, long long* cyc, int nwin) {
  extern __shared__ __align__(128) unsigned char raw[];
  InSlot& in = *reinterpret_cast<InSlot*>(raw);
  double2(*out)[W] = reinterpret_cast<double2(*)[W]>(raw + sizeof(InSlot));
  for (int i = threadIdx.x; i < (int)(sizeof(InSlot) / 8); i += blockDim.x)
    reinterpret_cast<double*>(raw)[i] = 1e-3 * (i % 7) + ((i % 22) == 17 || (i % 22) == 18 ? 0.5 : 0.0);
  __syncthreads();
  if (threadIdx.x >= 32) return;
  constexpr bool kHalf16 = V >= 6;
  if (kHalf16 && threadIdx.x >= 16) return;
  constexpr unsigned mask = kHalf16 ? 0xffffu : 0xffffffffu;
  const double2* above = reinterpret_cast<const double2*>(&in.p[R - 1][0][0]);  // stands in for the above ring
  const int l = threadIdx.x, lc = l < R ? l : R - 1, brow = lc;
  double2 win[3] = {make_double2(0, 0), make_double2(0, 0), make_double2(0, 0)};
  double2 wprev = make_double2(0, 0);
  auto load_raw = [&](int st, Raw& r) {
    const double2* a2 = reinterpret_cast<const double2*>(in.st[brow][st]);
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      const double2 v = a2[i];
      r.a[2 * i] = v.x;
      r.a[2 * i + 1] = v.y;
    }
    r.a[18] = in.st[brow][st][18];
    r.p = *reinterpret_cast<const double2*>(in.p[brow][st]);
  };
  auto prepare = [&](const Raw& r, double2 xm, double2 xz) {
    StepData o;
    if (V == 4 || V == 5) {
      o.q0 = r.p.x;
      o.q1 = r.p.y;
    } else {
      gs_pre(r.a, r.p.x, r.p.y, xm, xz, o.q0, o.q1);
    }
    o.e00 = r.a[8], o.e01 = r.a[9], o.e10 = r.a[10], o.e11 = r.a[11];
    o.w00 = r.a[12], o.w01 = r.a[13], o.w10 = r.a[14], o.w11 = r.a[15];
    o.c = r.a[16], o.r0 = r.a[17], o.r1 = r.a[18];
    return o;
  };
  const long long t0 = clock64();
  for (int w = 0; w < nwin; ++w) {
    Raw ra;
    load_raw(0, ra);
    StepData cur = prepare(ra, win[0], win[1]);
    load_raw(1, ra);
#pragma unroll
    for (int st = 0; st < W; ++st) {
      const double2 nv = gs_rec2(cur, wprev, win[2]);
      StepData nxt;
      if (st + 1 < W) nxt = prepare(ra, win[1], win[2]);
      if (V != 3 && V != 4 && V != 5 && V != 9 && st + 2 < W) load_raw(st + 2, ra);
      wprev = nv;
      if (V == 10) out[l][st] = nv;
      else if (V != 1 && V != 8 && l < R) out[l][st] = nv;
      double r0s, r1s;
      if (V == 2 || V == 5) {
        r0s = nv.x * 0.5, r1s = nv.y * 0.5;
      } else {
        r0s = __shfl_up_sync(mask, nv.x, 1);
        r1s = __shfl_up_sync(mask, nv.y, 1);
      }
      double2 up;
      if (V == 7 || V == 10) {
        up = make_double2(r0s, r1s);
        if (l == 0) up = above[st];
      } else {
        const double2 av = above[st];
        up = make_double2(l == 0 ? av.x : r0s, l == 0 ? av.y : r1s);
      }
      win[0] = win[1];
      win[1] = win[2];
      win[2] = up;
      if (st + 1 < W) cur = nxt;
    }
  }
  const long long t1 = clock64();
  if (l == 0) cyc[0] = t1 - t0;
  sink[l] = wprev.x + wprev.y + win[2].x;
}
template <int V>
void run(const char* name, double* sink, long long* cyc) {
  const int nwin = 2000;
  const size_t smem = sizeof(InSlot) + sizeof(double2) * R * W;
  cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<V><<<1, 512, smem>>>(sink, cyc, 10);
  k<V><<<1, 512, smem>>>(sink, cyc, nwin);
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("V%d %-44s %7.1f cycles/step (%s)\n", V, name, (double)c / (nwin * W), cudaGetErrorString(cudaGetLastError()));
}
int main() {
  double* sink;
  long long* cyc;
  cudaMalloc(&sink, 32 * 8);
  cudaMalloc(&cyc, 8);
  run<0>("product form", sink, cyc);
  run<1>("no store", sink, cyc);
  run<2>("no shuffle (own value)", sink, cyc);
  run<3>("no shared-memory loads in the loop", sink, cyc);
  run<4>("recurrence only (no gs_pre, no loads)", sink, cyc);
  run<5>("recurrence only, no shuffle", sink, cyc);
  run<6>("product form, 16 lanes active", sink, cyc);
  run<7>("16 lanes, predicated above load", sink, cyc);
  run<8>("16 lanes, no store", sink, cyc);
  run<9>("16 lanes, no loads in the loop", sink, cyc);
  run<10>("16 lanes, predicated above load, unmasked store", sink, cyc);
  return 0;
}
