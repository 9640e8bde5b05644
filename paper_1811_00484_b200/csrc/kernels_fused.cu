// kernels_fused.cu -- decompression x pencil in ONE persistent kernel: the Tucker-compressed
// spectrum is decompressed tile by tile into a small L2-resident ring and consumed from there by
// the pencil work items (axis-3 FFT + 144-block Hadamard + inverse FFT), so the octant spectra
// of the interior rows are never written to HBM as a whole.  This is the B200 form of the
// reference's buffer-free HosvdLoop strategy (operator.hpp:327-345: decompress one component,
// use it, drop it), at the granularity that lets the 25-wide factor GEMMs run on the FP64
// tensor cores: a TILE = 32 octant rows p1o (dtile::kBM) of one axis-2 octant row p2o, all components.
//
// Work items (a global queue, one atomicAdd per cluster item, both CTAs of a 2-CTA cluster work
// on the same item):
//   D(tau, cg): decompress components [cg CG, (cg+1) CG) of tile tau into ring slot tau % RING;
//               CTA b takes every other component of the group, both axis-3 parities, so T =
//               U1 Z is formed once per component (decomp_tile.cuh)
//   P(tau, i1, m2f): one pencil item of kernels_pencil4.cu (pencil4.cuh p4_item) whose spectrum
//               row is read from the ring
// Queue order: D(0..LA-1, *), then per tile tau: D(tau + LA, *), P(tau, *).  Dependencies are
// counters in global memory: a P item of tile tau waits (thread 0, before its first spectrum
// TMA) until both CTAs of all NG component groups are done; a D item writing slot
// tau % RING waits until every pencil CTA of tile tau - RING has consumed it.  Every wait is on
// items that precede it in the queue, and items are dequeued only by running clusters, so the
// earliest unfinished item can always proceed (no deadlock whatever the residency).
//
// The edge rows (p2o in {0, n2}, p1o in {0, n1}) are decompressed by their own small launches
// into a compact edge buffer (Geom::ecompact) read by the edge pencil kernels.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <numeric>
#include <vector>

#include "decomp_tile.cuh"
#include "pencil4.cuh"

namespace vie {

namespace {

struct FusedArgs {
  p4::Pencil4Args pa;
  const double2* forms;
  const double2* u3img;
  const CompDev* comps;
  const double2* Z;
  double2* ring;         // [RING * BM rows][NC][n3 + 1] branch-major spectrum rows
  const int4* items;     // {type (0 = D, 1 = P), tau, cg | i1, m2f}
  int nitems;
  unsigned* next;        // queue head
  unsigned* done;        // [tiles]: finished D-item CTAs (2 per component group)
  unsigned* consumed;    // [tiles]: pencil CTAs done with the tile's spectrum
  int NC, n1, n3;
  int CG, NG;            // components per D item, D items per tile
  int RING, BM, NB;      // ring slots, rows per tile, tiles per axis-2 octant row
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void spin_until(const unsigned* p, unsigned target) {
  while (ld_acquire(p) < target) __nanosleep(64);
}

template <int KIND, int R0, int R1>
__global__ void __launch_bounds__(256, 2)
    k_fused(FusedArgs f, const __grid_constant__ CUtensorMap tmS, const __grid_constant__ CUtensorMap tmIn,
            const __grid_constant__ CUtensorMap tmOut) {
  using SH = p4::Shape4<KIND, R0, R1>;
  extern __shared__ __align__(128) unsigned char smraw[];
  const p4::P4Smem sm = p4::p4_smem<SH::NBUF>(smraw);
  const int tid = threadIdx.x;
  const int b = static_cast<int>(blockIdx.x & 1);  // cluster rank = axis-3 parity / branch
  if (tid == 0) {
    for (int i = 0; i < SH::NBUF; ++i) {
      mbar_init(sm.full + i, 1);
      sm.cnt[i] = 0u;
    }
    mbar_init(sm.inbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  uint32_t item_remote;  // the partner's item slot (rank 0 publishes each item to both)
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(item_remote) : "r"(smem_u32(sm.item)), "r"(b ^ 1));
  const int64_t rs = static_cast<int64_t>(f.NC) * (f.n3 + 1);
  uint32_t qbase = 0, npen = 0;
  for (;;) {
    if (b == 0 && tid == 0) {
      const int w = static_cast<int>(atomicAdd(f.next, 1u));
      *reinterpret_cast<volatile int*>(sm.item) = w;
      asm volatile("st.shared::cluster.s32 [%0], %1;\n" ::"r"(item_remote), "r"(w) : "memory");
    }
    // publishes the item; also: the partner is done with the previous item (its DSMEM reads of
    // this CTA's line buffer, its multicast targets are free)
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    const int w = *reinterpret_cast<volatile int*>(sm.item);
    if (w >= f.nitems) break;
    const int4 it = f.items[w];
    const int tau = it.y;
    const int j2 = 1 + tau / f.NB, lo = 1 + (tau % f.NB) * f.BM, hi = min(f.n1, lo + f.BM);
    if (it.x == 0) {
      // ---- D(tau, cg): decompress into ring slot tau % RING
      if (tid == 0 && tau >= f.RING) {
        const int tp = tau - f.RING;
        const int plo = 1 + (tp % f.NB) * f.BM, phi = min(f.n1, plo + f.BM);
        spin_until(f.consumed + tp, static_cast<unsigned>(4 * (phi - plo)));
      }
      __syncthreads();
      double2* out = f.ring + static_cast<int64_t>(tau % f.RING) * f.BM * rs;
      // CTA b: components c0 + b, c0 + b + 2, .. of the group, both axis-3 parities (T once per component)
      const int c0 = it.z * f.CG, c1 = min(f.NC, c0 + f.CG);
      dtile::run<256, false, true>(f.forms, f.u3img, f.comps, f.Z, c0 + b, c1, 2, f.n1, f.n3, j2, lo, hi, 0, 2, out,
                                    rs, sm.chunk);
      // each writer orders its generic-proxy stores before the async-proxy (TMA) reads of the
      // consumers; thread 0 then publishes the group (release, cumulative over the barrier)
      asm volatile("fence.proxy.async.global;\n" ::: "memory");
      __syncthreads();
      if (tid == 0) red_release_add(f.done + tau, 1u);
    } else {
      // ---- P(tau, i1, m2f): pencil item on ring row (tau % RING) BM + (i1 - lo)
      const int i1 = it.z, m2f = it.w;
      const int srow = (tau % f.RING) * f.BM + (i1 - lo);
      p4::p4_item<KIND, R0, R1, false>(
          f.pa, &tmS, &tmIn, &tmOut, sm, i1, m2f, j2, b, srow, qbase, npen & 1u,
          [&] {
            spin_until(f.done + tau, static_cast<unsigned>(2 * f.NG));  // both CTAs of every group
            asm volatile("fence.proxy.async.global;\n" ::: "memory");
          },
          [&] {
            if (tid == 0) red_release_add(f.consumed + tau, 1u);
          });
      qbase += static_cast<uint32_t>(((b ? SH::O : SH::E) + SH::U - 1) / SH::U);
      ++npen;
    }
  }
}

// Edge rows of the octant spectrum into the compact edge buffer (shat_row, Geom::ecompact):
// P2ROWS = false: rows p2o in {0, n2} (y), all p1o in kBM-row blocks;
// P2ROWS = true:  rows p1o in {0, n1} (y), p2o in [1, n2) in kBM-row blocks.
// x = 2 * block + parity, z = component group.
template <bool P2ROWS>
__global__ void __launch_bounds__(256, 2) k_decomp_edge(const double2* __restrict__ forms,
                                                        const double2* __restrict__ u3img,
                                                        const CompDev* __restrict__ comps,
                                                        const double2* __restrict__ Z, double2* __restrict__ Sedge,
                                                        int NC, int n1, int n2, int n3, int CG) {
  extern __shared__ __align__(128) double2 smd[];
  const int b = static_cast<int>(blockIdx.x & 1), blk = static_cast<int>(blockIdx.x >> 1);
  const int64_t rs = static_cast<int64_t>(NC) * (n3 + 1);
  const int c0 = static_cast<int>(blockIdx.z) * CG, c1 = min(NC, c0 + CG);
  if (!P2ROWS) {
    const int p2o = blockIdx.y ? n2 : 0;
    const int lo = blk * dtile::kBM, hi = min(n1 + 1, lo + dtile::kBM);
    dtile::run<256, false>(forms, u3img, comps, Z, c0, c1, 1, n1, n3, p2o, lo, hi, b, b + 1,
                           Sedge + shat_row(p2o, lo, n1, n2, 1) * rs, rs, smd);
  } else {
    const int p1o = blockIdx.y ? n1 : 0;
    const int lo = 1 + blk * dtile::kBM, hi = min(n2, lo + dtile::kBM);
    if (lo >= hi) return;
    dtile::run<256, true>(forms, u3img, comps, Z, c0, c1, 1, n1, n3, p1o, lo, hi, b, b + 1,
                          Sedge + shat_row(lo, p1o, n1, n2, 1) * rs, 2 * rs, smd);
  }
}

#define VIE_FUSED_SHAPES(X) X(10, 20) X(10, 10) X(8, 16) X(8, 8) X(4, 8) X(8, 20) X(10, 12) X(8, 12) X(8, 10) X(6, 8)

int env_or(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

template <int KIND>
bool fused_t(const FusedPlan& fp, const double2* Bin, double2* Bout, const Geom& g, const double2* twm3,
             cudaStream_t st, bool dry) {
  auto go = [&](auto fn, size_t smem_p, int UB, int NC, int R1) {
    const size_t smem = std::max(smem_p, 128 + dtile::smem_bytes(g.n3, fp.rmax));
    if (smem > 113 * 1024) return false;  // two CTAs per SM
    if (g.nk != g.n3 || g.W != g.m1 || g.n2 < 2 || g.n1 < 2) return false;
    if (dry) return true;
    const int kb = [&] {
      int k = g.nk;
      while (k > 128 && k % 2 == 0) k /= 2;
      return k;
    }();
    const int kbs = std::gcd(R1 / 2, g.nk);
    VIE_CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    FusedArgs f{};
    f.pa = p4::Pencil4Args{twm3, g.n1, g.W, g.p1off, 1, g.nk, kb, kbs, 0};
    f.forms = fp.forms;
    f.u3img = fp.u3img;
    f.comps = fp.comps;
    f.Z = fp.Z;
    f.ring = fp.ring;
    f.items = fp.items;
    f.nitems = fp.nitems;
    f.next = fp.counters;
    f.done = fp.counters + 1;
    f.consumed = fp.counters + 1 + 2 * fp.ntiles;  // (done uses the first ntiles of its 2 ntiles)
    f.NC = g.NC;
    f.n1 = g.n1;
    f.n3 = g.n3;
    f.CG = fp.CG;
    f.NG = fp.NG;
    f.RING = fp.RING;
    f.BM = fp.BM;
    f.NB = fp.NB;
    CUtensorMap tmS, tmIn, tmOut;
    encode_spectrum_map(&tmS, fp.ring, g, {2 * UB, NC, 1}, static_cast<int64_t>(fp.RING) * fp.BM);
    encode_slab_map(&tmIn, Bin, g, kb, 1);
    encode_slab_map(&tmOut, Bout, g, kbs, 1);
    cudaLaunchConfig_t cfg = {};
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
    cfg.gridDim = dim3(2);
    int ncl = 0;
    VIE_CUDA_CHECK(cudaOccupancyMaxActiveClusters(&ncl, reinterpret_cast<const void*>(fn), &cfg));
    ncl = std::max(1, env_or("VIE_FUSED_CLUSTERS", ncl));
    cfg.gridDim = dim3(2 * ncl);
    VIE_CUDA_CHECK(cudaMemsetAsync(fp.counters, 0, sizeof(unsigned) * (1 + 3 * static_cast<size_t>(fp.ntiles)), st));
    VIE_CUDA_CHECK(cudaLaunchKernelEx(&cfg, fn, f, tmS, tmIn, tmOut));
    VIE_CUDA_CHECK(cudaGetLastError());
    return true;
  };
#define VIE_CASEF(A, B)                                                                    \
  if (g.n3 == (A) * (B)) {                                                                 \
    using SH = p4::Shape4<KIND, A, B>;                                                     \
    return go(k_fused<KIND, A, B>, SH::smem_bytes, SH::UB, SH::NC, B);                     \
  }
  VIE_FUSED_SHAPES(VIE_CASEF)
#undef VIE_CASEF
  return false;
}

}  // namespace

bool fused_supported(int kind, int basis, const Geom& g, uint64_t active_mask, int rmax) {
  if (basis != 1 || std::getenv("VIE_NO_FUSED")) return false;
  const uint64_t all = g.NC >= 64 ? ~0ull : ((1ull << g.NC) - 1);
  if (active_mask != all || rmax > 28) return false;
  FusedPlan fp{};
  fp.rmax = rmax;
  return kind == 0 ? fused_t<0>(fp, nullptr, nullptr, g, nullptr, nullptr, true)
                   : fused_t<1>(fp, nullptr, nullptr, g, nullptr, nullptr, true);
}

void fused_plan_items(FusedPlan& fp, const Geom& g, std::vector<int4>& items) {
  fp.BM = dtile::kBM;
  fp.NB = (g.n1 - 1 + fp.BM - 1) / fp.BM;
  fp.ntiles = fp.NB * (g.n2 - 1);
  fp.CG = std::max(1, env_or("VIE_FUSED_CG", 4));
  fp.NG = (g.NC + fp.CG - 1) / fp.CG;
  const int LA = std::max(1, env_or("VIE_FUSED_LA", 4));
  fp.RING = LA + 1;
  items.clear();
  auto emit_d = [&](int tau) {
    for (int cg = 0; cg < fp.NG; ++cg) items.push_back(make_int4(0, tau, cg, 0));
  };
  for (int tau = 0; tau < std::min(LA, fp.ntiles); ++tau) emit_d(tau);
  for (int tau = 0; tau < fp.ntiles; ++tau) {
    if (tau + LA < fp.ntiles) emit_d(tau + LA);
    const int lo = 1 + (tau % fp.NB) * fp.BM, hi = std::min(g.n1, lo + fp.BM);
    for (int i1 = lo; i1 < hi; ++i1)
      for (int m2f = 0; m2f < 2; ++m2f) items.push_back(make_int4(1, tau, i1, m2f));
  }
  fp.nitems = static_cast<int>(items.size());
}

void launch_fused(int kind, const FusedPlan& fp, const double2* Bin, double2* Bout, const Geom& g,
                  const double2* twm3, cudaStream_t st) {
  const bool ok = kind == 0 ? fused_t<0>(fp, Bin, Bout, g, twm3, st, false)
                            : fused_t<1>(fp, Bin, Bout, g, twm3, st, false);
  if (!ok) throw CudaError(cudaErrorInvalidValue, "fused decompress x pencil: unsupported geometry", __FILE__,
                           __LINE__);
}

void launch_decomp_edges(const FusedPlan& fp, double2* Sedge, const Geom& g, cudaStream_t st) {
  const size_t smem = dtile::smem_bytes(g.n3, fp.rmax);
  const int cg = 4, ng = (g.NC + cg - 1) / cg;
  VIE_CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_decomp_edge<false>),
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  VIE_CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_decomp_edge<true>),
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int nb1 = (g.n1 + 1 + dtile::kBM - 1) / dtile::kBM;
  k_decomp_edge<false><<<dim3(2 * nb1, 2, ng), 256, smem, st>>>(fp.forms, fp.u3img, fp.comps, fp.Z, Sedge, g.NC,
                                                                g.n1, g.n2, g.n3, cg);
  VIE_CUDA_CHECK(cudaGetLastError());
  const int nb2 = (g.n2 - 1 + dtile::kBM - 1) / dtile::kBM;
  if (nb2 > 0) {
    k_decomp_edge<true><<<dim3(2 * nb2, 2, ng), 256, smem, st>>>(fp.forms, fp.u3img, fp.comps, fp.Z, Sedge, g.NC,
                                                                 g.n1, g.n2, g.n3, cg);
    VIE_CUDA_CHECK(cudaGetLastError());
  }
}

}  // namespace vie
