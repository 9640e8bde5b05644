// kernels_pencil.cu -- fused axis-3 FFT + Tucker-spectrum Hadamard + IFFT.
//
// CTA = one mirror group: P1P pairs of axis-1 positions (p1, m1-p1) x the
// axis-2 position pair (p2, m2-p2), all S source currents, whole axis 3.
// Every octant spectrum value S^_c(p1o, p2o, f3o) (read once, from the
// decompression slab) serves all 8 mirror points (+-p1, +-p2, +-p3):
// with U_q(m-p) = sign_q U_q(p) (embed_column, operator.hpp:64-70),
// S^(m1-p1, p2, p3) = sign_1 S^(p1, p2, p3) and likewise per axis.
//
// Axis 3 is processed as two half-length branches (even / odd frequencies:
// the first DIF radix-2 stage of the zero-padded length-m3 transform done
// analytically), so 12 currents x 4 pencils fit in shared memory:
//   branch b:  X(2k+b) = DFT_n3( x[n] w_m3^{n b} )       (pad never touched)
//   y[n] = sum_b conj(w_m3^{n b}) IDFT_n3( Y(2k+b) ),  n < n3   (crop)
// Per branch: load -> FFT -> Hadamard over the branch's octant frequencies
// (spectrum chunks streamed with cp.async, double buffered) -> IFFT -> store
// (branch 0 writes the output slab, branch 1 accumulates).
//
// Hadamard = apply_operator's component loop + mac_elementwise
// (operator.hpp:303-364) fused over all components: x^ read once per point,
// y^_t = sum_blocks coef * sign * S^_c * x^_s kept in registers.
#include <cooperative_groups.h>

#include <utility>

#include "fft.cuh"
#include "hadamard.cuh"
#include "kernels.cuh"

namespace vie {

namespace {

using namespace had;

__host__ __device__ __forceinline__ int line_stride(int n) { return n + 1; }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

struct PencilArgs {
  const double2* Bin;
  double2* Bout;   // branch 0 output slab
  double2* Bout1;  // branch 1 output slab (conj-twiddled); summed by the axis-2 inverse pass
  const double2* Shat;
  const double2* twm3;  // w_m3^e, e < m3 (full-length plan table)
  Geom g;
  FftPlan PH;           // n3-point plan (branch transforms)
  int P1P;              // axis-1 mirror pairs per CTA
  int P2N;              // axis-2 positions per CTA (1 or 2)
  int NBUF;             // spectrum chunk buffers (1 or 2)
  int CF;               // octant frequencies per spectrum chunk
  uint64_t active;
  FastDiv div_n3;       // element index -> (line, k) without runtime division
  FastDiv div_nk;       // k -> slab block
  int g0;               // first axis-1 group of this launch
  FastDiv div_cf;
  FastDiv div_nc;
};

// Launch shapes: THREADS x MINB CTAs per SM.  P2N axis-2 positions per CTA
// (2 = full mirror group, Ŝ read once; 1 = half group, the axis-2 mirror CTA is
// the next blockIdx.x and re-reads Ŝ from L2).  NBUF spectrum chunk buffers.
#ifdef VIE_PENCIL_PROFILE
__device__ unsigned long long g_pencil_phase[8];
#define VIE_PHASE(i)                                                   \
  do {                                                                 \
    if (threadIdx.x == 0) {                                            \
      const long long t_ = clock64();                                  \
      atomicAdd(&g_pencil_phase[i], static_cast<unsigned long long>(t_ - t_last)); \
      t_last = t_;                                                     \
    }                                                                  \
  } while (0)
#else
#define VIE_PHASE(i) \
  do {               \
  } while (0)
#endif

template <int KIND, int BASIS, int THREADS, int MINB, bool ALL>
__global__ void __launch_bounds__(THREADS, MINB) k_pencil(PencilArgs a) {
#ifdef VIE_PENCIL_PROFILE
  long long t_last = clock64();
#endif
  constexpr int S = TableDims<KIND, BASIS>::S;
  constexpr int NB = TableDims<KIND, BASIS>::NB;
  constexpr int NC = TableDims<KIND, BASIS>::NC;
  constexpr int TS = S >= 12 ? 2 : 1;  // target split: 2 threads per spectral point (register budget)
  constexpr int TH = S / TS;
  extern __shared__ double2 sm[];
  const Geom& g = a.g;
  const int n1 = g.n1, n2 = g.n2, n3 = g.n3, m1 = g.m1, m2 = g.m2, m3 = g.m3;
  constexpr int NG = n_groups<NC>();
  constexpr int CG = group_size<NC>();
  const int P1P = a.P1P, CF = a.CF, P2N = a.P2N;
  const int W = 2 * P1P;
  const int NP = P2N * W;  // pencils: [p2sel][w], w < W  (powers of two)
  const int lgW = __ffs(W) - 1, lgNP = __ffs(NP) - 1;
  const int ls = line_stride(n3);
  const SmemPlan SP = load_plan(sm, a.PH);
  double2* twb = sm + plan_smem_elems(n3);  // w_m3^k, k < n3
  double2* shb = twb + n3;                  // 2 x [P1P][CG][CF] spectrum sub-chunks
  const int chunk_elems = P1P * CG * CF;
  double2* buf = shb + 2 * chunk_elems;     // [S][NP] lines of ls
  for (int e = threadIdx.x; e < n3; e += blockDim.x) twb[e] = a.twm3[e];

  // blockIdx.x runs over axis-1 groups: neighbouring CTAs read neighbouring
  // 32-byte segments of every pencil row, so L2 sectors fetched from DRAM are
  // fully used (the transposed order measured 2.8x the DRAM reads).
  const int b = blockIdx.x & 1;        // axis-3 branch (even / odd frequencies)
  const int c0 = (a.g0 + (blockIdx.x >> 1)) * W;  // first axis-1 position (global)
  const int q0 = c0 >> 1;         // tile octant row of axis 1
  const int pos2_0 = blockIdx.y * P2N;  // first axis-2 position (pair 2j, 2j+1 when P2N = 2)
  const int f2t = freq_of_pos(pos2_0, n2);
  const int p2o_tile = f2t > n2 ? m2 - f2t : f2t;
  const int n3p = n3 + 1;
  const int E = n3 / 2 + 1;            // even octant frequencies 0,2,..
  const int O = (n3 + 1) / 2;          // odd octant frequencies 1,3,..
  const int64_t kstride = g.bps;
  const int64_t sstride = kstride * g.nk;
  // slab offset of k-plane k (Geom blocked layout: block r = k / nk)
  auto koff = [&](int k) -> int64_t {
    const int r = static_cast<int>(a.div_nk.div(static_cast<uint32_t>(k)));
    return static_cast<int64_t>(k + r * (S - 1) * g.nk) * kstride;
  };

  {
    // ---- spectrum sub-chunks q = round * NG + group: CF octant frequencies x
    // CG components; sub-chunk 0 is prefetched so it lands during the FFT
    const int nbo = b ? O : E;
    const int nrounds = (nbo + CF - 1) / CF;
    const int nsub = nrounds * NG;
    auto issue_chunk = [&](int q) {
      double2* dst = shb + (q & 1) * chunk_elems;
      const int r = q / NG, grp = q - r * NG;
      const int u0 = r * CF;
      for (int e = threadIdx.x; e < chunk_elems; e += blockDim.x) {
        const int rc = static_cast<int>(a.div_cf.div(e));
        const int ul = e - rc * CF;
        const int tr = static_cast<int>(a.div_nc.div(rc));  // div_nc divides by CG
        const int c = grp * CG + (rc - tr * CG);
        const int p1o = q0 + tr;
        if (c < NC && p1o <= n1 && u0 + ul < nbo)
          cp_async16(dst + e, a.Shat + (shat_row(p2o_tile, p1o, n1, g.n2, g.ecompact) * NC + c) * n3p +
                                  b * E + u0 + ul);
      }
      cp_async_commit();
    };
    issue_chunk(0);

    // ---- load the pencils (k < n3) with cp.async (no register staging)
    for (int e = threadIdx.x; e < S * n3 * NP; e += blockDim.x) {
      const int p = e & (NP - 1);  // NP, W are powers of two
      const int w = p & (W - 1);
      const int p2sel = p >> lgW;
      const int sk = e >> lgNP;
      const int s = static_cast<int>(a.div_n3.div(sk)), k = sk - s * n3;
      const int pos1 = c0 + w, pos2 = pos2_0 + p2sel;
      double2* dst = buf + (s * NP + p) * ls + k;
      if (pos1 < m1)
        cp_async16(dst, a.Bin + s * sstride + koff(k) + static_cast<int64_t>(pos2) * g.W + (pos1 - g.p1off));
      else *dst = make_double2(0.0, 0.0);
    }
    cp_async_commit();
    cp_async_wait_all();  // also lands spectrum chunk 0 (committed earlier)
    __syncthreads();
    VIE_PHASE(0);
    if (b) {  // branch twiddle w_m3^{k} (odd frequencies)
      for (int e = threadIdx.x; e < S * NP * n3; e += blockDim.x) {
        const int line = static_cast<int>(a.div_n3.div(e)), k = e - line * n3;
        buf[line * ls + k] = cmul(buf[line * ls + k], twb[k]);
      }
    }
    __syncthreads();
    VIE_PHASE(1);
    fft_forward<true>(buf, S * NP, ls, SP, false);
    VIE_PHASE(2);

    // ---- Hadamard: one spectral point (x one target half) per thread per
    // round; x^ and y^ in registers for the whole round while the spectrum of
    // the round streams in NG component groups (next group prefetched).
    // lanes: mirror pair (mir) x pencil x frequency (slowest)
    const int items = CF * NP * 2;
    for (int r = 0; r < nrounds; ++r) {
      const int unit = threadIdx.x;
      const int half = unit >= items ? 1 : 0;
      const int it = unit - half * items;
      const int mir = it & 1;
      const int rest = it >> 1;
      const int p = rest & (NP - 1);
      const int ul = rest >> lgNP;
      const int u = r * CF + ul;
      const int f3o = 2 * u + b;
      const int w = p & (W - 1), p2sel = p >> lgW;
      const int pos1 = c0 + w;
      const bool valid = unit < items * TS && u < nbo && !(mir && (f3o == 0 || f3o == n3)) && pos1 < m1;
      double2 xh[S], yh[TH];
      double2* pl = buf;
      int m1flag = 0, m2flag = 0, p1o = 0, p2o = 0, tr = 0;
      bool in_tile = false;
      if (valid) {
        const int f1 = freq_of_pos(pos1, n1);
        m1flag = f1 > n1;
        p1o = m1flag ? m1 - f1 : f1;
        const int f2 = freq_of_pos(pos2_0 + p2sel, n2);
        m2flag = f2 > n2;
        p2o = m2flag ? m2 - f2 : f2;
        const int f3 = mir ? m3 - f3o : f3o;
        pl = buf + p * ls + SP.slot[(f3 - b) >> 1];
#pragma unroll
        for (int s = 0; s < S; ++s) xh[s] = pl[s * NP * ls];
        tr = p1o - q0;
        in_tile = p2o == p2o_tile && tr >= 0 && tr < P1P;
      }
#pragma unroll
      for (int t = 0; t < TH; ++t) yh[t] = make_double2(0.0, 0.0);
      sfor_g(std::make_integer_sequence<int, NG>{}, [&](auto gc) {
        constexpr int GRP = decltype(gc)::value;
        const int q = r * NG + GRP;
        cp_async_wait_all();
        __syncthreads();  // sub-chunk q visible; all threads done with q-1 (and with x^ reads of this round)
        if (q + 1 < nsub) issue_chunk(q + 1);
        if (valid) {
          const double2* sh_base;
          int cstride;
          if (in_tile) {  // smem sub-chunk [tr][c - GRP*CG][ul]
            sh_base = shb + (q & 1) * chunk_elems + (tr * CG - GRP * CG) * CF + ul;
            cstride = CF;
          } else {  // boundary pencils (frequencies 0 / n of a pair) outside the tile
            sh_base = a.Shat + (shat_row(p2o, p1o, n1, g.n2, g.ecompact) * NC) * n3p + b * E + u;
            cstride = n3p;
          }
          if (half == 0) {
            had_all<KIND, BASIS, S, TH, 0, ALL, GRP, CG>(std::make_integer_sequence<int, NB>{}, yh, xh, sh_base,
                                                         cstride, a.active, m1flag, m2flag, mir);
          } else if constexpr (TS > 1) {
            had_all<KIND, BASIS, S, TH, 1, ALL, GRP, CG>(std::make_integer_sequence<int, NB>{}, yh, xh, sh_base,
                                                         cstride, a.active, m1flag, m2flag, mir);
          }
        }
      });
      if (valid) {
#pragma unroll
        for (int t = 0; t < TH; ++t) pl[(half * TH + t) * NP * ls] = yh[t];
      }
    }
    __syncthreads();
    VIE_PHASE(3);
    fft_inverse<true>(buf, S * NP, ls, SP, false);
    VIE_PHASE(4);

    // ---- combine the two branches through DSMEM and store the cropped pencils:
    // y[n] = A_0[n] + conj(w_m3^n) A_1[n]; CTA b of the cluster writes half
    // of the lines, reading the partner branch from the partner's smem.
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();  // both branches' inverse transforms done
    const double2* rbuf = cluster.map_shared_rank(buf, b ^ 1);
    const int nlines = S * NP;
    const int l0 = b ? nlines / 2 : 0, l1 = b ? nlines : nlines / 2;
    constexpr int U = 4;  // remote (DSMEM) loads issued before use
    for (int e0 = l0 * n3 + threadIdx.x; e0 < l1 * n3; e0 += U * blockDim.x) {
      double2 own[U], rem[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int e = e0 + q * blockDim.x;
        if (e < l1 * n3) {
          const int line = static_cast<int>(a.div_n3.div(e)), k = e - line * n3;
          own[q] = buf[line * ls + k];
          rem[q] = rbuf[line * ls + k];
        }
      }
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int e = e0 + q * blockDim.x;
        if (e >= l1 * n3) break;
        const int line = static_cast<int>(a.div_n3.div(e)), k = e - line * n3;
        const int s = line >> lgNP, p = line & (NP - 1);
        const int w = p & (W - 1), p2sel = p >> lgW;
        const int pos1 = c0 + w, pos2 = pos2_0 + p2sel;
        if (pos1 >= m1) continue;
        const double2 a0 = b ? rem[q] : own[q], a1 = b ? own[q] : rem[q];
        a.Bout[s * sstride + koff(k) + static_cast<int64_t>(pos2) * g.W + (pos1 - g.p1off)] =
            cadd(a0, cmulc(a1, twb[k]));
      }
    }
    cluster.sync();  // partner finished reading this CTA's smem
    VIE_PHASE(5);
  }
}

int pencil_p1pairs(int S) { return S >= 12 ? 1 : (S >= 6 ? 2 : 4); }

struct PencilShape {
  int P1P, P2N, NBUF, CF;
};

size_t pencil_smem_shape(int n3, int S, int NC, const PencilShape& sh) {
  const int cg = NC >= 16 ? (NC + 2) / 3 : NC;  // group_size<NC>()
  const size_t e = static_cast<size_t>(plan_smem_elems(n3)) + n3 + 2ull * sh.P1P * cg * sh.CF +
                   static_cast<size_t>(S) * 2 * sh.P1P * sh.P2N * line_stride(n3);
  return e * sizeof(double2);
}

// Two 256-thread CTAs per SM (half mirror group) when they fit in half the
// SM's shared memory; else one 512-thread full-group CTA.  CF is set so a
// round gives every thread one (point, target half): CF = threads / (NP 2 TS).
constexpr size_t kHalfSmSmem = 112 * 1024;

#ifndef VIE_PENCIL_HALF_FIRST
#define VIE_PENCIL_HALF_FIRST 1
#endif

bool pencil_shape(int n3, int S, int NC, PencilShape& sh, bool& two_per_sm) {
  const int P1P = pencil_p1pairs(S);
  const int TS = S >= 12 ? 2 : 1;
  auto full = [&]() {
    sh = PencilShape{P1P, 2, 2, 512 / (4 * P1P * 2 * TS)};
    two_per_sm = false;
    return pencil_smem_shape(n3, S, NC, sh) <= kMaxSmem;
  };
  auto half = [&]() {
    sh = PencilShape{P1P, 1, 2, 256 / (2 * P1P * 2 * TS)};
    two_per_sm = true;
    return pencil_smem_shape(n3, S, NC, sh) <= kHalfSmSmem;
  };
  return VIE_PENCIL_HALF_FIRST ? (half() || full()) : (full() || half());
}

template <int KIND, int BASIS>
void launch_pencil_t(const double2* Bin, double2* Bout, double2* Bout1, const double2* Shat, const Geom& g,
                     const FftPlan& PH,
                     const double2* twm3, uint64_t active, int groups, cudaStream_t st) {
  constexpr int S = TableDims<KIND, BASIS>::S;
  constexpr int NC = TableDims<KIND, BASIS>::NC;
  PencilShape sh{};
  bool two = false;
  if (!pencil_shape(g.n3, S, NC, sh, two)) throw std::invalid_argument("pencil kernel: grid edge n3 too large");
  PencilArgs a{Bin, Bout, Bout1, Shat, twm3, g, PH, sh.P1P, sh.P2N, sh.NBUF, sh.CF, active, {}, {}, {}, {}, 0};
  a.div_n3.init(static_cast<uint32_t>(g.n3));
  a.div_nk.init(static_cast<uint32_t>(g.nk));
  a.div_cf.init(static_cast<uint32_t>(sh.CF));
  a.div_nc.init(static_cast<uint32_t>(group_size<NC>()));
  const size_t smem = pencil_smem_shape(g.n3, S, NC, sh);
  // this rank's axis-1 groups [g0, g1) (all of them on one GPU); groups > 0: only the first
  a.g0 = g.p1off / (2 * sh.P1P);
  const int g1 = (std::min(g.m1, g.p1off + g.W) + 2 * sh.P1P - 1) / (2 * sh.P1P);
  const int ng = groups > 0 ? std::min(groups, g1 - a.g0) : g1 - a.g0;
  if (ng <= 0) return;
  dim3 grid(2 * ng, g.m2 / sh.P2N);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;  // the two axis-3 branches of a group
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const bool all = active == ((NC >= 64) ? ~0ull : ((1ull << NC) - 1));
  auto launch = [&](auto fn, int threads) {
    VIE_CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    cfg.blockDim = dim3(threads);
    VIE_CUDA_CHECK(cudaLaunchKernelEx(&cfg, fn, a));
  };
  if (two) {
    if (all) launch(k_pencil<KIND, BASIS, 256, 2, true>, 256);
    else launch(k_pencil<KIND, BASIS, 256, 2, false>, 256);
  } else {
    if (all) launch(k_pencil<KIND, BASIS, 512, 1, true>, 512);
    else launch(k_pencil<KIND, BASIS, 512, 1, false>, 512);
  }
  VIE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace

#ifdef VIE_PENCIL_PROFILE
void pencil_phase_read(unsigned long long* out8, bool reset) {
  cudaMemcpyFromSymbol(out8, g_pencil_phase, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_pencil_phase, z, sizeof(z));
  }
}
#endif

size_t pencil_smem(int n3, int S, int NC) {
  PencilShape sh{};
  bool two = false;
  return pencil_shape(n3, S, NC, sh, two) ? pencil_smem_shape(n3, S, NC, sh) : static_cast<size_t>(-1);
}

void launch_pencil(int kind, int basis, const double2* Bin, double2* Bout, double2* Bout1, const double2* Shat,
                   const Geom& g, const FftPlan& PH, const double2* twm3, uint64_t active, cudaStream_t st,
                   int groups) {
  if (kind == 0 && basis == 0) launch_pencil_t<0, 0>(Bin, Bout, Bout1, Shat, g, PH, twm3, active, groups, st);
  else if (kind == 1 && basis == 0) launch_pencil_t<1, 0>(Bin, Bout, Bout1, Shat, g, PH, twm3, active, groups, st);
  else if (kind == 0 && basis == 1) launch_pencil_t<0, 1>(Bin, Bout, Bout1, Shat, g, PH, twm3, active, groups, st);
  else launch_pencil_t<1, 1>(Bin, Bout, Bout1, Shat, g, PH, twm3, active, groups, st);
}

}  // namespace vie
