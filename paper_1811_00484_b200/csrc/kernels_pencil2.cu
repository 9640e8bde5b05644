// kernels_pencil2.cu -- compile-time-shaped fused axis-3 FFT + Hadamard + IFFT.
//
// Same math as kernels_pencil.cu (read its header first): a 2-CTA cluster
// owns P1P axis-1 mirror pairs at one axis-2 position, CTA b of the cluster
// the even (b = 0) / odd (b = 1) axis-3 frequencies as a length-n3 branch
// transform, and the octant spectrum S^ is read once per mirror group.  What
// differs is the schedule, shaped for n3 = R0 * R1 known at compile time:
//
//  * forward stage 0 (radix R0) runs straight from global memory in
//    registers -- no staging copy, and the odd branch's input twiddle
//    w_m3^{n} folds into compile-time constants w_{2 R0}^{i} on the inputs plus
//    the stage twiddle w_m3^{m'(2k+b)} on the outputs; stage 1 (radix R1) is
//    one in-place smem pass;
//  * the spectrum streams in component-group chunks, one 3-D TMA tensor copy
//    per chunk (cp.async.bulk.tensor), on an mbarrier ring refilled by the last
//    warp done with a buffer -- no per-element address arithmetic;
//  * every spectrum offset in the unrolled block table is an immediate;
//  * the inverse stage 1 is one in-place smem pass; the inverse stage 0 is
//    fused with the branch combine y[n] = A_0[n] + conj(w_m3^n) A_1[n]: CTA b
//    reads both branches' lines of its half (the partner's through DSMEM),
//    runs both radix-R0 adjoints in registers and stores y to global.
#include <cooperative_groups.h>
#include <cuda.h>  // CUtensorMap (encoded through the runtime's driver entry point)

#include <array>
#include <cstdio>
#include <cstdlib>
#include <utility>

#include "fft.cuh"
#include "hadamard.cuh"
#include "tma.cuh"
#include "kernels.cuh"

#ifndef VIE_P2_NBUF
#define VIE_P2_NBUF 2
#endif
#ifndef VIE_P2_CHUNK
#define VIE_P2_CHUNK 640  // spectrum chunk budget (double2): 10 KB
#endif
#ifndef VIE_P2_ABL
#define VIE_P2_ABL 0  // ablation bits (timing experiments only): 1 no Hadamard FMAs, 2 no spectrum stream,
                     // 4 no pencil loads, 8 no stores, 16 no DSMEM reads
#endif

namespace vie {

namespace {

using namespace had;

constexpr int p1pairs(int S) { return S >= 12 ? 1 : (S >= 6 ? 2 : 4); }  // = kernels_pencil.cu pencil_p1pairs

template <int KIND, int BASIS, int R0, int R1>
struct Shape2 {
  static constexpr int S = TableDims<KIND, BASIS>::S;
  static constexpr int NB = TableDims<KIND, BASIS>::NB;
  static constexpr int NC = TableDims<KIND, BASIS>::NC;
  static constexpr int THREADS = 256;
  static constexpr int WARPS = THREADS / 32;
  static constexpr int TS = 1;  // one thread per spectral point, all targets: no x^/y^ hazard between threads
  static constexpr int TH = S / TS;
  static constexpr int P1P = p1pairs(S);
  static constexpr int NP = 2 * P1P;  // pencils (axis-1 positions) per CTA
  static constexpr int LINES = S * NP;
  static constexpr int HL = LINES / 2;  // lines combined + stored by each CTA of the pair
  static constexpr int N3 = R0 * R1;
  static constexpr int LS = N3 | 1;  // odd line stride: lanes over lines hit distinct banks
  static constexpr int CF = THREADS / (NP * 2 * TS);  // octant frequencies per chunk
  static constexpr int CHUNK_BUDGET = VIE_P2_CHUNK;   // double2 per chunk buffer
  static constexpr int CG0 = CHUNK_BUDGET / (P1P * CF) > 0 ? CHUNK_BUDGET / (P1P * CF) : 1;
  static constexpr int NG = (NC + CG0 - 1) / CG0;  // component groups per round
  static constexpr int CG = (NC + NG - 1) / NG;
  static constexpr int CHUNK = P1P * CG * CF;  // double2 per chunk buffer
  static constexpr int E = N3 / 2 + 1;         // even octant frequencies (branch 0)
  static constexpr int O = (N3 + 1) / 2;       // odd octant frequencies (branch 1)
  static constexpr int NBUF = VIE_P2_NBUF;     // chunk ring depth
  static constexpr size_t smem_bytes = 128 + sizeof(double2) * (NBUF * CHUNK + static_cast<size_t>(LINES) * LS);
  static_assert(HL * R1 <= THREADS, "one combine unit per thread");
  static_assert(LINES % 2 == 0 && (NP & (NP - 1)) == 0, "pencil tile shape");
  static_assert(CF * NP * 2 * TS == THREADS, "one (point, target half) per thread per round");
};

struct Pencil2Args {
  const double2* Bin;
  double2* Bout;
  const double2* Shat;
  const double2* twm3;  // w_m3^e, e < m3
  int n1, n2, m1, m2, m3;
  int64_t kstride, sstride;  // plane stride bps, current stride nk * bps (Geom)
  int nk;      // k-planes per slab block (koff)
  int W;       // row length of the slabs (axis-1 positions of this rank)
  int p1off;   // global axis-1 position of slab column 0
  int gfirst;  // first axis-1 group of this launch
  int pos2lo;  // first axis-2 position of this launch
  FastDiv dnk;
  int ecompact;  // Geom::ecompact (spectrum rows of the edge buffer)
};

#ifdef VIE_PENCIL_PROFILE
__device__ unsigned long long g_p2_phase[8];
#define P2_PHASE(i)                                                                   \
  do {                                                                                \
    if (threadIdx.x == 0) {                                                           \
      const long long t_ = clock64();                                                 \
      atomicAdd(&g_p2_phase[i], static_cast<unsigned long long>(t_ - t_last));        \
      t_last = t_;                                                                    \
    }                                                                                 \
  } while (0)
#else
#define P2_PHASE(i) \
  do {              \
  } while (0)
#endif

// the slot of branch frequency phi = k0 + R0 k1 after the two forward stages
// Position of element j of stage-1 block k0: rotated by ROT k0 within the block so the
// Hadamard's lanes (consecutive branch frequencies, their mirrors, both pencils) hit
// distinct smem banks (searched offline; 2.0 -> 1.47 wavefronts per quarter warp at
// n3 = 10 x 20).  The FFT stages address whole blocks per thread, so any rotation is
// conflict-free for them.
template <int R0, int R1>
struct Rot {
  static constexpr int ROT = (R0 == 10 && R1 == 20) ? 18 : 0;
};
template <int R0, int R1>
__device__ __forceinline__ int blk_pos(int k0, int j) {  // k0 block, j < R1 element
  if constexpr (Rot<R0, R1>::ROT == 0) {
    return k0 * R1 + j;
  } else {
    int t = j + (Rot<R0, R1>::ROT * k0) % R1;
    t -= t >= R1 ? R1 : 0;
    return k0 * R1 + t;
  }
}
// the slot of branch frequency phi = k0 + R0 k1 after the two forward stages
template <int R0, int R1>
__device__ __forceinline__ int slot_of(int phi) {
  const int k0 = phi % R0, k1 = phi / R0;
  return blk_pos<R0, R1>(k0, k1);
}

template <int KIND, int BASIS, int R0, int R1>
__global__ void __launch_bounds__(256, 2) k_pencil2(Pencil2Args a, const __grid_constant__ CUtensorMap tmap) {
  using SH = Shape2<KIND, BASIS, R0, R1>;
#ifdef VIE_PENCIL_PROFILE
  long long t_last = clock64();
#endif
  constexpr int S = SH::S, NB = SH::NB, TH = SH::TH, P1P = SH::P1P, NP = SH::NP;
  constexpr int LINES = SH::LINES, HL = SH::HL, N3 = SH::N3, LS = SH::LS, CF = SH::CF, NG = SH::NG, CG = SH::CG;
  constexpr int CHUNK = SH::CHUNK, E = SH::E, O = SH::O;
  extern __shared__ __align__(128) unsigned char smraw[];
  constexpr int NBUF = SH::NBUF;
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw);  // [NBUF]
  unsigned* cnt = reinterpret_cast<unsigned*>(full + NBUF);  // [NBUF] warps done with each chunk buffer
  double2* chunk = reinterpret_cast<double2*>(smraw + 128);  // TMA destinations: 128-byte aligned
  double2* buf = chunk + NBUF * CHUNK;  // [LINES][LS]

  const int tid = threadIdx.x;
  const int b = blockIdx.x & 1;                     // axis-3 branch = rank in the cluster
  const int c0 = 2 * P1P * (a.gfirst + (blockIdx.x >> 1));  // first axis-1 position (group 0 is the edge launch)
  const int cl0 = c0 - a.p1off;                              // its slab column
  const int q0 = c0 >> 1;                           // octant row of pair 0
  const int pos2 = a.pos2lo + static_cast<int>(blockIdx.y);  // axis-2 position
  // slab offset of k-plane k: block r = k / nk of the k-planes (one block on one GPU)
  auto koff = [&](int k) -> int64_t {
    const int r = static_cast<int>(a.dnk.div(static_cast<uint32_t>(k)));
    return static_cast<int64_t>(k + r * (SH::S - 1) * a.nk) * a.kstride;
  };
  const int n1 = a.n1, n2 = a.n2, m1 = a.m1;
  const int f2 = freq_of_pos(pos2, n2);
  const int m2flag = f2 > n2;
  const int p2o = m2flag ? a.m2 - f2 : f2;
  const int nbo = b ? O : E;
  const int nrounds = (nbo + CF - 1) / CF;
  const int nsub = nrounds * NG;

  // ---- spectrum chunk q = round * NG + group -> buffer q % NBUF (bulk copies)
  // one TMA tensor copy per chunk: rows (p2o, q0 .. q0 + P1P), components grp*CG .., the
  // round's CF frequencies of branch b (out-of-range rows/components zero-filled)
  auto issue_chunk = [&](int q) {
    const int r = q / NG, grp = q - r * NG;
    uint64_t* bar = full + q % NBUF;
    mbar_expect_tx(bar, static_cast<uint32_t>(CHUNK * sizeof(double2)));
    tma_chunk(chunk + (q % NBUF) * CHUNK, &tmap, 2 * (b * E + r * CF), grp * CG,
              static_cast<int>(shat_row(p2o, q0, n1, a.n2, a.ecompact)), bar);
  };
  // ---- forward stage 0 (radix R0) for BOTH branches of this CTA's half of the lines:
  // the pencils are read from global once per cluster, branch b' of the stage-0
  // outputs goes to CTA b' (the partner's half through DSMEM stores)
  namespace cg = cooperative_groups;
  double2* const rbuf = cg::this_cluster().map_shared_rank(buf, b ^ 1);  // the partner's lines
  double2* const buf_b0 = b ? rbuf : buf;                                 // branch 0 / branch 1 owners
  double2* const buf_b1 = b ? buf : rbuf;
  const int line0 = b * HL + tid % HL, mp0 = tid / HL;
  const bool act0 = tid < HL * R1;
  double2 xin[R0];
  {
    const int s = line0 / NP, p = line0 % NP;
    if (act0 && c0 + p < m1 && !(VIE_P2_ABL & 4)) {
      const double2* src = a.Bin + s * a.sstride + static_cast<int64_t>(pos2) * a.W + cl0 + p;
#pragma unroll
      for (int i = 0; i < R0; ++i) xin[i] = src[koff(mp0 + i * R1)];
    } else {
#pragma unroll
      for (int i = 0; i < R0; ++i) xin[i] = make_double2(0.0, 0.0);
    }
  }
  if (tid == 0) {
    for (int i = 0; i < NBUF; ++i) {
      mbar_init(full + i, 1);
      cnt[i] = 0u;
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    if (!(VIE_P2_ABL & 2))
      for (int i = 0; i < NBUF && i < nsub; ++i) issue_chunk(i);
  }
  P2_PHASE(0);
  // the partner may still be starting up: its smem is written only after this barrier
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
  const double2 wstep0 = __ldg(a.twm3 + 2 * mp0);
  double2 v[R0];
#pragma unroll
  for (int i = 0; i < R0; ++i) v[i] = xin[i];
  if (act0) DFTs<R0, false, 1, 0>::run(v);  // branch 0: outputs * w_m3^{2 k mp}
  asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
  if (act0) {
    {
      double2* dst = buf_b0 + line0 * LS;
      double2 w = wstep0;
      dst[blk_pos<R0, R1>(0, mp0)] = v[out_idx(R0, 0)];
      sfor<R0 - 1>([&](auto kc) {
        constexpr int k = decltype(kc)::value + 1;
        dst[blk_pos<R0, R1>(k, mp0)] = cmul(v[out_idx(R0, k)], w);
        if (k + 1 < R0) w = cmul(w, wstep0);
      });
    }
    v[0] = xin[0];  // branch 1: inputs * w_{2 R0}^i, outputs * w_m3^{mp (2k + 1)}
    sfor<R0 - 1>([&](auto ic) {
      constexpr int i = decltype(ic)::value + 1;
      v[i] = twc<2 * R0, false, i>(xin[i]);
    });
    DFTs<R0, false, 1, 0>::run(v);
    {
      double2* dst = buf_b1 + line0 * LS;
      double2 w = __ldg(a.twm3 + mp0);
      sfor<R0>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        dst[blk_pos<R0, R1>(k, mp0)] = cmul(v[out_idx(R0, k)], w);
        if (k + 1 < R0) w = cmul(w, wstep0);
      });
    }
  }
  // every stage-0 output (own and partner's) visible before stage 1
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  P2_PHASE(1);
  // ---- forward stage 1 (radix R1), in place
  for (int u = tid; u < LINES * R0; u += SH::THREADS) {
    const int line = u % LINES, k0 = u / LINES;
    double2* p = buf + line * LS;
    double2 v[R1];
#pragma unroll
    for (int i = 0; i < R1; ++i) v[i] = p[blk_pos<R0, R1>(k0, i)];
    DFTs<R1, false, 1, 0>::run(v);
    sfor<R1>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      p[blk_pos<R0, R1>(k0, k)] = v[out_idx(R1, k)];
    });
  }
  __syncthreads();

  P2_PHASE(2);
  // ---- Hadamard: one spectral point (all targets) per thread per round; the
  // last warp done with a chunk refills its buffer (no thread ever waits on
  // the others inside the loop)
  {
    const int p = tid % NP;          // lane order (searched with the rotation): pencil fastest,
    const int ul = (tid / NP) % CF;  // then frequency, mirror slowest
    const int mir = tid / (NP * CF);
    const int pos1 = c0 + p;
    const int m1flag = pos1 & 1;  // positions 2j, 2j+1 hold frequencies j, m1 - j (j >= 1)
    const int tr = p >> 1;
    const int lane = tid & 31;
    for (int r = 0; r < nrounds; ++r) {
      const int u = r * CF + ul;
      const int f3o = 2 * u + b;
      const bool valid = u < nbo && !(mir && (f3o == 0 || f3o == N3)) && pos1 < m1;
      const int phi = mir ? N3 - u - b : u;
      double2* pl = buf + p * LS + slot_of<R0, R1>(valid ? phi : 0);
      double2 xh[S], yh[TH];
      constexpr auto SG = Signs<KIND, BASIS>::value;
      const int sbits = m1flag | (m2flag << 1) | (mir << 2);
      if (valid) {
#pragma unroll
        for (int s = 0; s < S; ++s) xh[s] = flip_sign(pl[s * NP * LS], pattern_sign(SG.pi[s] ^ SG.G, sbits));
      }
#pragma unroll
      for (int t = 0; t < TH; ++t) yh[t] = make_double2(0.0, 0.0);
      sfor_g(std::make_integer_sequence<int, NG>{}, [&](auto gc) {
        constexpr int GRP = decltype(gc)::value;
        const int q = r * NG + GRP;
        const int bi = q % NBUF;
        if (!(VIE_P2_ABL & 2)) mbar_wait(full + bi, (q / NBUF) & 1);
        if (valid && !(VIE_P2_ABL & 1)) {
          const double2* sh_base = chunk + bi * CHUNK + (tr * CG - GRP * CG) * CF + ul;
          had_all_ns<KIND, BASIS, S, TH, GRP, CG>(std::make_integer_sequence<int, NB>{}, yh, xh, sh_base, CF);
        }
        // every Hadamard read of buffer bi has returned (its FMAs were issued), so the
        // warp can sign off without a fence; the last warp out refills the buffer
        __syncwarp();
        if (lane == 0) {
          if (atomicAdd(cnt + bi, 1u) == SH::WARPS - 1) {
            cnt[bi] = 0u;
            if (q + NBUF < nsub && !(VIE_P2_ABL & 2)) {
              asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
              issue_chunk(q + NBUF);
            }
          }
        }
      });
      if (valid) {
#pragma unroll
        for (int t = 0; t < TH; ++t) pl[t * NP * LS] = flip_sign(yh[t], pattern_sign(SG.pi[t], sbits));
      }
    }
  }
  __syncthreads();
  P2_PHASE(3);
  // ---- inverse stage 1 (adjoint of radix R1), in place
  for (int u = tid; u < LINES * R0; u += SH::THREADS) {
    const int line = u % LINES, k0 = u / LINES;
    double2* p = buf + line * LS;
    double2 v[R1];
#pragma unroll
    for (int k = 0; k < R1; ++k) v[k] = p[blk_pos<R0, R1>(k0, k)];
    DFTs<R1, true, 1, 0>::run(v);
    sfor<R1>([&](auto ic) {
      constexpr int i = decltype(ic)::value;
      p[blk_pos<R0, R1>(k0, i)] = v[out_idx(R1, i)];
    });
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  __syncthreads();
  // ---- inverse stage 0 (adjoint of radix R0) of both branches + combine; own branch first,
  // the partner's (DSMEM) once the cluster barrier completes
  {
    const int line = b * HL + tid % HL, mp = tid / HL;
    const int s = line / NP, p = line % NP;
    const bool act = tid < HL * R1 && c0 + p < m1;
    const int off = line * LS;
    const double2 wstep = __ldg(a.twm3 + 2 * min(mp, R1 - 1));
    const double2 w1 = __ldg(a.twm3 + min(mp, R1 - 1));
    // branch br: inputs * conj(w_m3^{mp (2k + br)}), then the radix-R0 adjoint
    auto branch = [&](const double2* X, int br, double2(&v)[R0]) {
      const int mpc = min(mp, R1 - 1);
      double2 w = br ? w1 : wstep;
      v[0] = br ? cmulc(X[off + blk_pos<R0, R1>(0, mpc)], w) : X[off + blk_pos<R0, R1>(0, mpc)];
      if (br) w = cmul(w, wstep);
#pragma unroll
      for (int k = 1; k < R0; ++k) {
        v[k] = cmulc(X[off + blk_pos<R0, R1>(k, mpc)], w);
        if (k + 1 < R0) w = cmul(w, wstep);
      }
      DFTs<R0, true, 1, 0>::run(v);
    };
    double2 vo[R0], vr[R0];
    if (act) branch(buf, b, vo);
    P2_PHASE(4);
    const double2* rem = rbuf;
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    P2_PHASE(5);
    if (act) branch((VIE_P2_ABL & 16) ? buf : rem, b ^ 1, vr);
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");  // done reading the partner
    if (act && !(VIE_P2_ABL & 8)) {
      double2* dst = a.Bout + s * a.sstride + static_cast<int64_t>(pos2) * a.W + cl0 + p;
      sfor<R0>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        const double2 y0 = b ? vr[out_idx(R0, i)] : vo[out_idx(R0, i)];
        const double2 y1 = b ? vo[out_idx(R0, i)] : vr[out_idx(R0, i)];
        dst[koff(mp + i * R1)] = cadd(y0, twc<2 * R0, true, i>(y1));
      });
    }
    asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");  // the partner finished reading this CTA
    P2_PHASE(6);
  }
}

#define VIE_PENCIL2_SHAPES(X) X(10, 20) X(10, 10) X(8, 16) X(8, 8) X(4, 8) X(8, 20) X(10, 12) X(8, 12) X(8, 10) X(6, 8)

template <int KIND, int BASIS>
bool launch2_t(int n3, const double2* Bin, double2* Bout, const double2* Shat, const Geom& g, const double2* twm3,
               cudaStream_t st, bool dry, int pos2lo, int pos2hi) {
  auto go = [&](auto fn, size_t smem, int P1P, std::array<int, 3> box) {
    if (dry) return true;
    // axis-1 groups of this rank's positions [p1off, p1off + W); group 0 is the edge launch
    const int glo = std::max(1, g.p1off / (2 * P1P));
    const int ghi = (std::min(g.m1, g.p1off + g.W) + 2 * P1P - 1) / (2 * P1P);
    if (pos2hi < 0) pos2hi = g.m2;
    if (ghi <= glo || pos2hi <= pos2lo) return true;
    VIE_CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    Pencil2Args a{Bin, Bout, Shat, twm3, g.n1, g.n2, g.m1, g.m2, g.m3, g.bps, g.bps * g.nk, g.nk, g.W, g.p1off,
                  glo, pos2lo, {}, g.ecompact};
    a.dnk.init(static_cast<uint32_t>(g.nk));
    CUtensorMap tmap;
    encode_spectrum_map(&tmap, Shat, g, box);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * (ghi - glo), pos2hi - pos2lo);
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
    if (std::getenv("VIE_DEBUG_OCC")) {
      int nb = 0, ncl = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, 256, smem);
      cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg);
      fprintf(stderr, "pencil2 smem %zu: blocks/SM %d, active clusters %d\n", smem, nb, ncl);
    }
    VIE_CUDA_CHECK(cudaLaunchKernelEx(&cfg, fn, a, tmap));
    VIE_CUDA_CHECK(cudaGetLastError());
    return true;
  };
#define VIE_CASE(A, B)                                                                   \
  if (n3 == (A) * (B)) {                                                                 \
    using SH = Shape2<KIND, BASIS, A, B>;                                                \
    if (SH::smem_bytes > 113 * 1024) return false;                                       \
    return go(k_pencil2<KIND, BASIS, A, B>, SH::smem_bytes, SH::P1P, {2 * SH::CF, SH::CG, SH::P1P}); \
  }
  VIE_PENCIL2_SHAPES(VIE_CASE)
#undef VIE_CASE
  return false;
}

bool dispatch2(int kind, int basis, int n3, const double2* Bin, double2* Bout, const double2* Shat, const Geom& g,
               const double2* twm3, cudaStream_t st, bool dry, int pos2lo = 0, int pos2hi = -1) {
  if (kind == 0 && basis == 0) return launch2_t<0, 0>(n3, Bin, Bout, Shat, g, twm3, st, dry, pos2lo, pos2hi);
  if (kind == 1 && basis == 0) return launch2_t<1, 0>(n3, Bin, Bout, Shat, g, twm3, st, dry, pos2lo, pos2hi);
  if (kind == 0 && basis == 1) return launch2_t<0, 1>(n3, Bin, Bout, Shat, g, twm3, st, dry, pos2lo, pos2hi);
  return launch2_t<1, 1>(n3, Bin, Bout, Shat, g, twm3, st, dry, pos2lo, pos2hi);
}

}  // namespace

#ifdef VIE_PENCIL_PROFILE
void pencil2_phase_read(unsigned long long* out8, bool reset) {
  cudaMemcpyFromSymbol(out8, g_p2_phase, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_p2_phase, z, sizeof(z));
  }
}
#endif

bool pencil2_supported(int kind, int basis, int n3, uint64_t active_mask, int NC) {
  const uint64_t all = NC >= 64 ? ~0ull : ((1ull << NC) - 1);
  if (active_mask != all) return false;
  Geom g{};
  return dispatch2(kind, basis, n3, nullptr, nullptr, nullptr, g, nullptr, nullptr, true);
}

void launch_pencil2(int kind, int basis, const double2* Bin, double2* Bout, const double2* Shat, const Geom& g,
                    const double2* twm3, cudaStream_t st, int pos2lo, int pos2hi) {
  dispatch2(kind, basis, g.n3, Bin, Bout, Shat, g, twm3, st, false, pos2lo, pos2hi);
}

}  // namespace vie
