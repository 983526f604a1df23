// Shared device helpers for the B200 PBM Newton-step kernels.
//
// Data layout:
//  * nodal vectors live on the node grid of a level, two fp64 dofs per node
//    (x then y), index 2*(iy*NX + ix) + c; Dirichlet dofs are stored as 0;
//    a bordered vector carries the volume multiplier unknown in the slot
//    right after the grid (index 2*NX*NY);
//  * element arrays are indexed e = ex_i + EX*ey_i, the reference's order
//    (mesh.py:253-259);
//  * a level operator is a node-block 9-point stencil (block b = (dy+1)*3 +
//    (dx+1), entries r0c0 r0c1 r1c0 r1c1) stored as two half-stencils of 20
//    doubles (160 B) per node, array-of-structs:
//      L = [SW S SE W | a10 rd0 rd1 a00 | pad pad]   (couplings to earlier nodes)
//      U = [NE N NW E | a01 rd0 rd1 a11 | pad pad]   (couplings to later nodes)
//    A forward Gauss-Seidel sweep is "P = b - U x_old" (parallel) followed by
//    a wavefront solve with L only; a backward sweep swaps the halves, and the
//    mirrored block order makes the two wavefront kernels identical.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#ifndef VTS_DEVICE_INLINE
#define VTS_DEVICE_INLINE __device__ __forceinline__
#endif

namespace vts {

constexpr int kStencilStride = 40;  // doubles per node of the full (setup-time) stencil
constexpr int kHalf = 22;           // doubles per node of one half-stencil (20 used + 2 pad: 176 B rows)
constexpr int kPadRows = 17;        // node rows of zero padding before/after every level array (skewed TMA boxes)
constexpr int kHC = 16;             // a10 (L) / a01 (U)
constexpr int kHRd0 = 17, kHRd1 = 18;
constexpr int kHDiag = 19;          // a00 (L) / a11 (U)
constexpr int kBlockCenter = 4;

// offset of full-stencil block b inside its half (-1 = center), and which half
VTS_DEVICE_INLINE int half_offset(int b) {
  // SW S SE W -> L 0 4 8 12 ; E NW N NE -> U 12 8 4 0
  return b < 4 ? 4 * b : (b > 4 ? 4 * (8 - b) : -1);
}
VTS_DEVICE_INLINE bool in_lower(int b) { return b < 4; }

// entry (r, c) of block b of node nd from the two halves
VTS_DEVICE_INLINE double stencil_entry(const double* __restrict__ L, const double* __restrict__ U, int nd, int b,
                                       int r, int c) {
  const double* l = L + (size_t)nd * kHalf;
  const double* u = U + (size_t)nd * kHalf;
  if (b == kBlockCenter) {
    if (r == 0) return c == 0 ? l[kHDiag] : u[kHC];
    return c == 0 ? l[kHC] : u[kHDiag];
  }
  const int o = half_offset(b) + 2 * r + c;
  return b < 4 ? l[o] : u[o];
}

// Element stiffness of the unit Q1 square, row-major 8x8 (set by the context).
// Defined here: the library is one translation unit (csrc/vts_b200.cu).
__constant__ double c_ke[64];
// K_e in the corner-mode basis (see modal_form in vts_b200.cu), divided by 16:
// {A1 (xi_x xi_x), A2 (eta_y eta_y), B (xi_x eta_y), S1 (xi_y xi_y), S2 (eta_x eta_x),
//  S12 (xi_y eta_x), H1 (h_x h_x), H2 (h_y h_y)}
__constant__ double c_modal[8];

struct LevelDev {
  int ex, ey;         // elements per axis
  int nx, ny;         // nodes per axis
  int nnodes;         // nx * ny
  int ngrid;          // 2 * nnodes (grid dofs, border slot at ngrid)
  int nfree;          // number of free dofs (the reference's n)
  const uint8_t* free_mask;  // [ngrid] 1 = free dof
  const int32_t* free2grid;  // [nfree]
  double* stL;               // [nnodes * kHalf] lower half-stencil
  double* stU;               // [nnodes * kHalf] upper half-stencil
  double* border;            // [ngrid] level border vector (P^T chain)
};

// ---------------------------------------------------------------------------
// deterministic block reductions (fixed shuffle tree, fixed warp order)
// ---------------------------------------------------------------------------
VTS_DEVICE_INLINE double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Sums NV values across the block; result valid in thread 0.  `scratch` must
// hold NV * (blockDim.x / 32) doubles.  Order of additions is fixed.
template <int NV>
VTS_DEVICE_INLINE void block_sum(double (&v)[NV], double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) scratch[i * nw + warp] = v[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += scratch[i * nw + w];
      v[i] = s;
    }
  }
  __syncthreads();
}

// Writes the block's NV partial sums to partials[blockIdx.x * NV + i].
template <int NV>
VTS_DEVICE_INLINE void block_partials(double (&v)[NV], double* scratch, double* partials) {
  block_sum<NV>(v, scratch);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) partials[blockIdx.x * NV + i] = v[i];
  }
}

// penalty/barrier kernel phi (reference penalty.py:49-95); returns phi, phi', phi''
struct PhiOut {
  double v, d1, d2;
};

VTS_DEVICE_INLINE double phi_saturate(double tau, unsigned* flag) {
  // penalty.py:85-95: NaN -> 0, +-inf -> +-1e300, then clip to +-1e150
  if (!(fabs(tau) <= 1e150)) {
    *flag = 1u;
    if (isnan(tau)) tau = 0.0;
    tau = fmin(fmax(tau, -1e150), 1e150);
  }
  return tau;
}

VTS_DEVICE_INLINE PhiOut phi_eval(double tau, double t, unsigned* flag) {
  tau = phi_saturate(tau, flag);
  PhiOut o;
  if (tau >= t) {
    o.v = __dadd_rn(tau, __dmul_rn(__dmul_rn(0.5, tau), tau));
    o.d1 = __dadd_rn(1.0, tau);
    o.d2 = 1.0;
  } else {
    const double c = (1.0 + t) * (1.0 + t);
    const double den = __dsub_rn(__dadd_rn(1.0, 2.0 * t), tau);
    o.v = __dadd_rn(__dadd_rn(-c * log(__ddiv_rn(den, 1.0 + t)), t), 0.5 * t * t);
    o.d1 = __ddiv_rn(c, den);
    o.d2 = __ddiv_rn(c, __dmul_rn(den, den));
  }
  return o;
}

}  // namespace vts
