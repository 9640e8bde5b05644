// kernels_pencil4.cu -- PWL pencil kernel, HALF a mirror group per 2-CTA cluster so that two
// clusters share every SM pair: axis-3 FFT + 144-block Hadamard on the FP64 tensor cores +
// inverse FFT + crop.
//
// Math as kernels_pencil3.cu (read its header): axis 3 is two half-length branches (CTA b of
// the cluster owns the frequencies 2k + b) and every octant spectrum value S^_c(p1o, p2o, f3o)
// serves the mirror points (+-p1, +-p2, +-p3).  The difference is the work unit:
//
//  * Unit.  A cluster owns the two pencils (p1, m1-p1) at ONE axis-2 position (24 lines =
//    2 pencils x 12 currents, line L = 2 s + m1f) instead of all four of the mirror group.
//    The line buffer is N3 x 24 x 16 B (76.8 KB at n3 = 200) and the CTA has 256 threads,
//    so two CTAs (of different clusters) are resident per SM and one CTA's load / barrier /
//    store phases overlap the other's FP64 work -- the pencil3 CTA (48 lines, 154 KB, 512
//    threads) runs alone on its SM and every phase boundary idles it.  The two clusters of
//    an axis-2 mirror pair are adjacent in launch order, so the second one reads the
//    octant spectrum row from L2.
//
//  * Hadamard.  One octant frequency has 4 points here (n = m1f | m3f << 1).  The complex
//    product is a real GEMM with the real and imaginary parts of X stacked as the 8 columns:
//
//      D1 = Ar [Xr | Xi],  D2 = Ai [Xr | Xi]     (M = 12 targets in two m8 tiles, K = 12 sources)
//      Yr = D1[:, n] - D2[:, n + 4],  Yi = D1[:, n + 4] + D2[:, n]
//
//    with A[t][s] = coef(t,s) S^_{c(t,s)} (mma.sync.m8n8k4.f64: 12 DMMAs per octant
//    frequency; the lanes holding columns n and n + 4 exchange one D2 value by a shuffle and
//    each stores one double of Y).  Mirror signs are split onto X and Y (hadamard.cuh
//    SignSplit) with the point's full flag set m1f | m2f << 1 | m3f << 2.
//
// Reference: apply_operator's component loop + mac_elementwise over every (target, source,
// component) block (operator.hpp:303-364, 263-265), and the pad / forward3 / inverse3 / crop
// around it (:290-297, :367-375).
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <numeric>

#include "pencil4.cuh"

namespace vie {

namespace {

using p4::Pencil4Args;
using p4::Shape4;

template <int KIND, int R0, int R1>
__global__ void __launch_bounds__(256, 2)
    k_pencil4(Pencil4Args a, const __grid_constant__ CUtensorMap tmS, const __grid_constant__ CUtensorMap tmIn,
              const __grid_constant__ CUtensorMap tmOut) {
  using SH = Shape4<KIND, R0, R1>;
  extern __shared__ __align__(128) unsigned char smraw[];
  const p4::P4Smem sm = p4::p4_smem<SH::NBUF>(smraw);
  const int tid = threadIdx.x;
  const int b = static_cast<int>(blockIdx.x & 1);    // axis-3 branch = rank in the cluster
  const int cl = static_cast<int>(blockIdx.x >> 1);  // cluster column: (axis-1 pair group, m2f)
  const int i1 = a.gfirst + (cl >> 1);
  const int j2 = 1 + static_cast<int>(blockIdx.y);
  if (tid == 0) {
    for (int i = 0; i < SH::NBUF; ++i) {
      mbar_init(sm.full + i, 1);
      sm.cnt[i] = 0u;
    }
    mbar_init(sm.inbar, 1);
    mbar_init(sm.rdone, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // both CTAs' input barriers exist before either multicasts into them (the init fence above
  // is the release: the arrive itself can be relaxed)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  p4::p4_item<KIND, R0, R1, true>(a, &tmS, &tmIn, &tmOut, sm, i1, cl & 1, j2, b, j2 * (a.n1 + 1) + i1, 0u, 0u,
                                  [] {}, [] {});
}

#define VIE_PENCIL4_SHAPES(X) X(10, 20) X(10, 10) X(8, 16) X(8, 8) X(4, 8) X(8, 20) X(10, 12) X(8, 12) X(8, 10) X(6, 8)

// k extent of the load boxes: a divisor of nk, at most 128 (<= 256 per TMA box dim)
int load_box_k4(int nk) {
  int kb = nk;
  while (kb > 128 && kb % 2 == 0) kb /= 2;
  return kb <= 256 ? kb : -1;
}

template <int KIND>
bool launch4_t(int n3, const double2* Bin, double2* Bout, const double2* Shat, const Geom& g, const double2* twm3,
               cudaStream_t st, bool dry) {
  auto go = [&](auto fn, size_t smem, int UB, int NC, int R1) {
    const int kb = load_box_k4(g.nk), kbs = std::gcd(R1 / 2, g.nk);
    if (kb < 1 || g.n3 % kb) return false;
    if (dry) return true;
    // interior axis-1 pair groups of this rank's positions [p1off, p1off + W); group 0 is the edge launch
    const int glo = std::max(1, g.p1off / 2);
    const int ghi = std::min(g.m1, g.p1off + g.W) / 2;
    if (ghi <= glo || g.n2 < 2) return true;
    VIE_CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    Pencil4Args a{twm3, g.n1, g.W, g.p1off, glo, g.nk, kb, kbs, 0};
    CUtensorMap tmS, tmIn, tmOut;
    encode_spectrum_map(&tmS, Shat, g, {2 * UB, NC, 1});
    encode_slab_map(&tmIn, Bin, g, kb, 1);
    encode_slab_map(&tmOut, Bout, g, kbs, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(4 * (ghi - glo), g.n2 - 1);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    static const int pf_env = std::getenv("VIE_P4_PF") ? std::atoi(std::getenv("VIE_P4_PF")) : 0;
    if (pf_env != 0) {
      int ncl = 0;
      VIE_CUDA_CHECK(cudaOccupancyMaxActiveClusters(&ncl, reinterpret_cast<const void*>(fn), &cfg));
      a.pf = pf_env > 0 ? pf_env : ncl;
    }
    VIE_CUDA_CHECK(cudaLaunchKernelEx(&cfg, fn, a, tmS, tmIn, tmOut));
    VIE_CUDA_CHECK(cudaGetLastError());
    return true;
  };
#define VIE_CASE4(A, B)                                                     \
  if (n3 == (A) * (B)) {                                                    \
    using SH = Shape4<KIND, A, B>;                                          \
    if (SH::smem_bytes > kMaxSmem) return false;                            \
    return go(k_pencil4<KIND, A, B>, SH::smem_bytes, SH::UB, SH::NC, B);    \
  }
  VIE_PENCIL4_SHAPES(VIE_CASE4)
#undef VIE_CASE4
  return false;
}

}  // namespace

#ifdef VIE_PENCIL_PROFILE
void pencil4_phase_read(unsigned long long* out8, bool reset) {
  cudaMemcpyFromSymbol(out8, p4::g_p4_phase, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(p4::g_p4_phase, z, sizeof(z));
  }
}
#endif

bool pencil4_supported(int kind, int basis, int n3, uint64_t active_mask, int NC) {
  if (basis != 1) return false;
  const uint64_t all = NC >= 64 ? ~0ull : ((1ull << NC) - 1);
  if (active_mask != all) return false;
  if (std::getenv("VIE_NO_PENCIL4")) return false;
  Geom g{};
  g.n3 = n3;
  g.nk = n3;
  return kind == 0 ? launch4_t<0>(n3, nullptr, nullptr, nullptr, g, nullptr, nullptr, true)
                   : launch4_t<1>(n3, nullptr, nullptr, nullptr, g, nullptr, nullptr, true);
}

void launch_pencil4(int kind, const double2* Bin, double2* Bout, const double2* Shat, const Geom& g,
                    const double2* twm3, cudaStream_t st) {
  const bool ok = kind == 0 ? launch4_t<0>(g.n3, Bin, Bout, Shat, g, twm3, st, false)
                            : launch4_t<1>(g.n3, Bin, Bout, Shat, g, twm3, st, false);
  if (!ok) throw CudaError(cudaErrorInvalidValue, "pencil4: unsupported slab geometry", __FILE__, __LINE__);
}

}  // namespace vie
