// tma.cuh -- mbarrier, bulk-copy and TMA tensor-copy helpers (sm_100a) shared by
// the pencil kernels, and the host-side encoding of the octant-spectrum tensor map.
#pragma once
#include <cuda.h>  // CUtensorMap (encoded through the runtime's driver entry point)

#include <array>

#include "kernels.cuh"

namespace vie {

// ---------------------------------------------------------------- mbarrier / bulk copy
static __device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
static __device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
static __device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
static __device__ __forceinline__ bool mbar_try(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
static __device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  while (!mbar_try(b, parity)) {
  }
}
// 3-D tiled TMA load of one spectrum chunk (box [P1P][CG][2 CF doubles]) into smem
static __device__ __forceinline__ void tma_chunk(void* dst, const CUtensorMap* tmap, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// Spectrum slab as a 3-D tensor of doubles: [(n2+1)(n1+1) rows][NC components][2 (n3+1)]
inline void encode_spectrum_map(CUtensorMap* map, const double2* Shat, const Geom& g, const std::array<int, 3>& box,
                                int64_t rows = -1) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    VIE_CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess)
      throw CudaError(cudaErrorNotSupported, "cuTensorMapEncodeTiled entry point", __FILE__, __LINE__);
    return reinterpret_cast<Encode>(fn);
  }();
  const cuuint64_t n3p = static_cast<cuuint64_t>(g.n3) + 1;
  const cuuint64_t dims[3] = {2 * n3p, static_cast<cuuint64_t>(g.NC),
                              static_cast<cuuint64_t>(rows > 0 ? rows : shat_rows(g.n1, g.n2, g.ecompact))};
  const cuuint64_t strides[2] = {n3p * sizeof(double2), n3p * sizeof(double2) * g.NC};
  const cuuint32_t boxd[3] = {static_cast<cuuint32_t>(box[0]), static_cast<cuuint32_t>(box[1]),
                              static_cast<cuuint32_t>(box[2])};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double2*>(Shat), dims, strides, boxd,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError(cudaErrorInvalidValue, "cuTensorMapEncodeTiled", __FILE__, __LINE__);
}

// ---------------------------------------------------------------- pencil-kernel helpers
static __device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
static __device__ __forceinline__ double2 lds2(uint32_t a) {
  double2 r;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(r.x), "=d"(r.y) : "r"(a));
  return r;
}
static __device__ __forceinline__ double2 ldc2(uint32_t a) {  // partner CTA (shared::cluster window)
  double2 r;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];\n" : "=d"(r.x), "=d"(r.y) : "r"(a));
  return r;
}
static __device__ __forceinline__ void sts2(uint32_t a, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
// 5-D TMA load of a slab box, multicast to the CTAs in `mask` (same smem offset, each
// CTA's mbarrier at the same offset receives the bytes landing in it)
static __device__ __forceinline__ double lds1(uint32_t a) {
  double r;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(r) : "r"(a));
  return r;
}
static __device__ __forceinline__ void sts1(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(a), "d"(v) : "memory");
}
static __device__ __forceinline__ void tma_load5_mc(void* dst, const CUtensorMap* m, int c0, int c1, int c2, int c3, int c4,
                                             uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
static __device__ __forceinline__ void tma_prefetch5(const CUtensorMap* m, int c0, int c1, int c2, int c3, int c4) {
  asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];\n" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
               : "memory");
}
static __device__ __forceinline__ void tma_prefetch3(const CUtensorMap* m, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];\n" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
// L2 eviction policies (createpolicy): streaming slab traffic evict_first, the decompressed
// spectrum tiles evict_last (kept resident in L2 between producer and consumers)
static __device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
static __device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
static __device__ __forceinline__ void tma_load5_mc_hint(void* dst, const CUtensorMap* m, int c0, int c1, int c2,
                                                         int c3, int c4, uint64_t* bar, uint16_t mask,
                                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
      ".L2::cache_hint [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8, %9;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar)), "h"(mask),
      "l"(pol)
      : "memory");
}
static __device__ __forceinline__ void tma_store5_hint(const CUtensorMap* m, const void* src, int c0, int c1, int c2,
                                                       int c3, int c4, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group.L2::cache_hint [%0, {%2, %3, %4, %5, %6}], [%1], "
      "%7;\n" ::"l"(reinterpret_cast<uint64_t>(m)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "l"(pol)
      : "memory");
}
static __device__ __forceinline__ void st_hint(double2* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
}
static __device__ __forceinline__ void tma_store5(const CUtensorMap* m, const void* src, int c0, int c1, int c2, int c3,
                                           int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];\n" ::"l"(
          reinterpret_cast<uint64_t>(m)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}

// Slab B / Bo as a 5-D tensor of doubles: [R blocks][nk k][m2 p2][S s][2 W (p1, re/im)]
// (innermost first: 2 W, S, m2, nk, R), box [4][12][p2box][kb][1] = one k-run of p2box axis-2 positions of an axis-1 pair.
inline void encode_slab_map(CUtensorMap* map, const double2* base, const Geom& g, int kb, int p2box) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    VIE_CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess)
      throw CudaError(cudaErrorNotSupported, "cuTensorMapEncodeTiled entry point", __FILE__, __LINE__);
    return reinterpret_cast<Encode>(fn);
  }();
  const cuuint64_t R = static_cast<cuuint64_t>(g.n3 / g.nk);
  const cuuint64_t dims[5] = {2 * static_cast<cuuint64_t>(g.W), static_cast<cuuint64_t>(g.S),
                              static_cast<cuuint64_t>(g.m2), static_cast<cuuint64_t>(g.nk), R};
  const cuuint64_t e16 = sizeof(double2);
  const cuuint64_t strides[4] = {static_cast<cuuint64_t>(g.bps) * g.nk * e16, static_cast<cuuint64_t>(g.W) * e16,
                                 static_cast<cuuint64_t>(g.bps) * e16,
                                 static_cast<cuuint64_t>(g.bps) * g.nk * g.S * e16};
  const cuuint32_t boxd[5] = {4, 12, static_cast<cuuint32_t>(p2box), static_cast<cuuint32_t>(kb), 1};
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<double2*>(base), dims, strides, boxd,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError(cudaErrorInvalidValue, "cuTensorMapEncodeTiled (slab)", __FILE__, __LINE__);
}

}  // namespace vie
