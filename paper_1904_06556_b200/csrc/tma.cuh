// mbarrier / TMA / release-acquire helpers shared by the kernels, and the
// host-side tensor-map encoder (driver entry point fetched through the runtime).
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include "context.cuh"

namespace vts {

VTS_DEVICE_INLINE unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// a double2 through L1 (CG = false) or L2 only
template <bool CG>
VTS_DEVICE_INLINE double2 ld2(const double* p) {
  return CG ? __ldcg(reinterpret_cast<const double2*>(p)) : *reinterpret_cast<const double2*>(p);
}
VTS_DEVICE_INLINE int ld_relaxed_i32(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// cross-cluster handoff rows: a value slot is empty while either half holds
// this NaN pattern (arithmetic never produces it: the producer maps it to the
// default quiet NaN), so every 8-byte half is its own ready flag
constexpr unsigned long long kXferEmpty = 0xFFFFFFFFFFFFFFFFull;
VTS_DEVICE_INLINE void st_relaxed_v2(double* p, double2 v) {
  asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
VTS_DEVICE_INLINE double2 ld_relaxed_v2(const double* p) {
  double2 v;
  asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
  return v;
}
VTS_DEVICE_INLINE bool xfer_empty(double2 v) {
  return (unsigned long long)__double_as_longlong(v.x) == kXferEmpty ||
         (unsigned long long)__double_as_longlong(v.y) == kXferEmpty;
}
VTS_DEVICE_INLINE double xfer_canon(double v) {
  return (unsigned long long)__double_as_longlong(v) == kXferEmpty ? __longlong_as_double(0x7FF8000000000000ll) : v;
}
VTS_DEVICE_INLINE void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
VTS_DEVICE_INLINE uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
VTS_DEVICE_INLINE void mbar_init(unsigned long long* m, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
VTS_DEVICE_INLINE void mbar_expect_tx(unsigned long long* m, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
VTS_DEVICE_INLINE bool mbar_try_wait(unsigned long long* m, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(m)), "r"(parity)
      : "memory");
  return ok != 0;
}
VTS_DEVICE_INLINE void mbar_wait(unsigned long long* m, unsigned parity) {
  while (!mbar_try_wait(m, parity)) {
  }
}
// bulk global -> shared copy (TMA engine), completion counted on mbarrier m
VTS_DEVICE_INLINE void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(m))
               : "memory");
}
VTS_DEVICE_INLINE void mbar_arrive(unsigned long long* m) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(m)) : "memory");
}
// 3-D TMA tile load (box of the tensor map at {c0, c1, c2}) with mbarrier completion
VTS_DEVICE_INLINE void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, unsigned long long* m) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(m))
      : "memory");
}


static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static int tma_encoder() {
  if (g_encode) return 0;
  cudaDriverEntryPointQueryResult q;
  VTS_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&g_encode), cudaEnableDefault, &q));
  if (q != cudaDriverEntryPointSuccess || !g_encode) {
    set_error(5, "cuTensorMapEncodeTiled unavailable");
    return 5;
  }
  return 0;
}

// plain (unskewed) tiled map over a row-major fp64 array with `rank` dims,
// dims[0] innermost; out-of-bounds box elements read as zeros
static int encode_tiled(CUtensorMap* map, const double* base, int rank, const cuuint64_t* dims,
                        const cuuint64_t* strides_bytes, const cuuint32_t* box) {
  if (int rc = tma_encoder()) return rc;
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<double*>(base), dims,
                              strides_bytes, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error(5, "cuTensorMapEncodeTiled failed");
    return 5;
  }
  return 0;
}

// 2-D TMA tile load with mbarrier completion
VTS_DEVICE_INLINE void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, unsigned long long* m) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(m))
      : "memory");
}

}  // namespace vts
