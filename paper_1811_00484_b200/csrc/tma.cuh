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
inline void encode_spectrum_map(CUtensorMap* map, const double2* Shat, const Geom& g, const std::array<int, 3>& box) {
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
                              static_cast<cuuint64_t>(g.n1 + 1) * static_cast<cuuint64_t>(g.n2 + 1)};
  const cuuint64_t strides[2] = {n3p * sizeof(double2), n3p * sizeof(double2) * g.NC};
  const cuuint32_t boxd[3] = {static_cast<cuuint32_t>(box[0]), static_cast<cuuint32_t>(box[1]),
                              static_cast<cuuint32_t>(box[2])};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double2*>(Shat), dims, strides, boxd,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError(cudaErrorInvalidValue, "cuTensorMapEncodeTiled", __FILE__, __LINE__);
}

}  // namespace vie
