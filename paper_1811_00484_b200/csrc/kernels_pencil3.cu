// kernels_pencil3.cu -- PWL pencil kernel: axis-3 FFT + 144-block Hadamard on the FP64
// tensor cores + IFFT, one whole mirror group per 2-CTA cluster, all data movement by TMA.
//
// Math as kernels_pencil.cu / kernels_pencil2.cu (read their headers): axis 3 is two
// half-length branches (CTA b of the cluster owns the frequencies 2k + b), and every
// octant spectrum value S^_c(p1o, p2o, f3o) serves the 8 mirror points (+-p1, +-p2, +-p3).
// New here:
//
//  * Grouping.  The cluster owns all four pencils (p1, m1-p1) x (p2, m2-p2) of one octant
//    row, so a CTA holds all 8 mirror points of each of its octant frequencies (p3 and
//    m3-p3 lie in the same branch) and the Hadamard of one octant frequency is a small
//    complex GEMM over the 8 points n = m1f | m2f << 1 | m3f << 2:
//
//      Y'[n][t] = sum_s X'[n][s] A[s][t],   A[s][t] = coef(t,s) S^_{c(t,s)},
//      X'[n][s] = chi_n(pi_s ^ G) x^_s(n),  y^_t(n) = chi_n(pi_t) Y'[n][t]
//
//    (hadamard.cuh SignSplit moves every mirror sign onto X and Y, so A is common to the
//    8 points).  One warp = one octant frequency on mma.sync.m8n8k4.f64: M = the 8
//    points, N = 12 targets (two n8 tiles, 4 padding columns), K = 12 sources (three k4
//    steps), complex by the 3-multiplication (Gauss) product: 18 DMMAs per octant
//    frequency instead of 8 x 144 x 4 DFMAs, and no per-thread x^ / y^ register arrays.
//
//  * Layout.  The line buffer is slot-major: element (slot p, m2f, s, m1f) at
//    p * 48 + 24 m2f + 2 s + m1f, i.e. line L = 24 m2f + 2 s + m1f.  That is exactly the
//    box order of a TMA tensor copy of the slab [s][k][p2][p1] (p1 pair innermost), so
//    the 48 input lines of the group arrive by a handful of TMA boxes (each CTA issues
//    half of them, multicast to both CTAs: no DSMEM traffic in the forward), and the
//    outputs leave by TMA stores.  The FFT stages are in place (a radix-R column reads
//    and writes the same slots); lanes run over lines, so every FFT access is a run of
//    consecutive 16-byte words (conflict free), as are the X-fragment loads (lanes pair
//    m1f and 4 consecutive sources) and the Y-fragment stores (targets permuted to
//    columns by tau() so one quarter warp hits 8 distinct bank groups).
//
//  * Branch combine.  y[n] = A_0[n] + conj(w_m3^n) A_1[n] (n < n3, the crop): CTA b
//    finalises the columns mp in [b R1/2, (b+1) R1/2) of the last inverse stage for all
//    48 lines (own branch from smem, the partner's through ld.shared::cluster), in
//    place, then TMA-stores the output slots k = i R1 + mp.
//
// Reference: apply_operator's component loop + mac_elementwise over every (target,
// source, component) block (operator.hpp:303-364, 263-265), and the pad / forward3 /
// inverse3 / crop around it (:290-297, :367-375).
#include <cuda.h>

#include <array>
#include <cstdio>
#include <cstdlib>
#include <numeric>

#include "fft.cuh"
#include "hadamard.cuh"
#include "kernels.cuh"
#include "tma.cuh"

#ifndef VIE_P3_NBUF
#define VIE_P3_NBUF 3
#endif

namespace vie {

namespace {

using namespace had;

template <int KIND, int R0, int R1>
struct Shape3 {
  static constexpr int S = 12;  // PWL currents
  static constexpr int NC = TableDims<KIND, 1>::NC;
  static constexpr int THREADS = 512;
  static constexpr int WARPS = THREADS / 32;
  static constexpr int LINES = 48;         // 4 pencils x 12 currents, line L = 24 m2f + 2 s + m1f
  static constexpr int N3 = R0 * R1;       // branch length (= n3)
  static constexpr int HR1 = R1 / 2;       // last-stage columns finalised per CTA
  static constexpr int U = WARPS;          // octant frequencies per chunk (one per warp)
  static constexpr int UB = U + 1;         // box width: one pad column (bank spread of the gather)
  static constexpr int E = N3 / 2 + 1;     // even octant frequencies (branch 0)
  static constexpr int O = (N3 + 1) / 2;   // odd octant frequencies (branch 1)
  static constexpr int NBUF = VIE_P3_NBUF;
  static constexpr int CHUNK = UB * NC;                              // double2 per chunk
  static constexpr int CHUNK_STRIDE = (CHUNK * 16 + 127) / 128 * 8;  // double2, 128-byte aligned buffers
  static constexpr int BUF_ELEMS = N3 * LINES;
  static constexpr size_t smem_bytes =
      128 + sizeof(double2) * (static_cast<size_t>(NBUF) * CHUNK_STRIDE + BUF_ELEMS);
  static_assert(LINES * HR1 <= THREADS && LINES * R0 <= THREADS, "one FFT unit per thread");
  static_assert(R1 % 2 == 0, "the last inverse stage splits its columns between the CTAs");
  static_assert(U == 16, "chunk = one octant frequency per warp");
};

// N-tile columns -> targets (tile 1 columns 4..7 are padding): the two columns a lane
// holds (2 tq, 2 tq + 1) map to targets whose 2 t differ mod 8 across a quarter warp.
__device__ __forceinline__ int tau(int nt, int j) {
  constexpr int t0 = 0x73625140;  // 8 nibbles: 0 4 1 5 2 6 3 7
  constexpr int t1 = 0xb9a8;      // 8 10 9 11
  return nt == 0 ? (t0 >> (4 * j)) & 15 : (j < 4 ? (t1 >> (4 * j)) & 15 : -1);
}

template <int R0, int R1>
__device__ __forceinline__ int slot3(int phi) {  // slot of branch frequency phi = k0 + R0 k1
  return (phi % R0) * R1 + phi / R0;
}

// (component, coefficient) of block (t, s) of the PWL table; c = -1: no block.
// Statically initialised from the compile-time tables (common.cuh make_table), so every
// device gets it with the module image; global (not __constant__): the per-lane gather
// is divergent.
struct BlockMatrix {
  int c[144];
  int coef[144];
};
template <int KIND>
constexpr BlockMatrix make_block_matrix() {
  BlockMatrix m{};
  for (int e = 0; e < 144; ++e) {
    m.c[e] = -1;
    m.coef[e] = 0;
  }
  const auto tb = make_table<KIND, 1>();
  for (const auto& bk : tb.blocks) {
    m.c[bk.t * 12 + bk.s] = bk.c;
    m.coef[bk.t * 12 + bk.s] = bk.coef;
  }
  return m;
}
__device__ const BlockMatrix c_bm3[2] = {make_block_matrix<0>(), make_block_matrix<1>()};

struct Pencil3Args {
  const double2* twm3;  // w_m3^e, e < m3
  int n1;
  int W;
  int p1off;
  int gfirst;  // first axis-1 pair group of this launch (>= 1)
  int nk;      // k-planes per slab block
  int KB;      // k extent of a load box (divides nk)
  int KBS;     // k extent of a store box (divides nk and R1 / 2)
  int pf;      // L2 prefetch distance in clusters (co-resident clusters; 0 = off)
};

#ifdef VIE_PENCIL_PROFILE
__device__ unsigned long long g_p3_phase[8];
#define P3_PHASE(i)                                                                   \
  do {                                                                                \
    if (threadIdx.x == 0) {                                                           \
      const long long t_ = clock64();                                                 \
      atomicAdd(&g_p3_phase[i], static_cast<unsigned long long>(t_ - t_last));        \
      t_last = t_;                                                                    \
    }                                                                                 \
  } while (0)
#else
#define P3_PHASE(i) \
  do {              \
  } while (0)
#endif

template <int KIND, int R0, int R1>
__global__ void __launch_bounds__(512, 1)
    k_pencil3(Pencil3Args a, const __grid_constant__ CUtensorMap tmS, const __grid_constant__ CUtensorMap tmIn,
              const __grid_constant__ CUtensorMap tmOut) {
  using SH = Shape3<KIND, R0, R1>;
#ifdef VIE_PENCIL_PROFILE
  long long t_last = clock64();
#endif
  constexpr int LINES = SH::LINES, N3 = SH::N3, HR1 = SH::HR1;
  constexpr int U = SH::U, UB = SH::UB, E = SH::E, O = SH::O, NBUF = SH::NBUF;
  constexpr int CHUNK = SH::CHUNK, CSTR = SH::CHUNK_STRIDE;
  extern __shared__ __align__(128) unsigned char smraw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw);  // [NBUF] spectrum ring
  uint64_t* inbar = full + NBUF;                          // input boxes
  unsigned* cnt = reinterpret_cast<unsigned*>(inbar + 1);
  double2* chunk = reinterpret_cast<double2*>(smraw + 128);
  double2* buf = chunk + NBUF * CSTR;  // [slot][L]
  const uint32_t buf_sa = smem_u32(buf);

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int b = static_cast<int>(blockIdx.x & 1);  // axis-3 branch = rank in the cluster
  const int i1 = a.gfirst + static_cast<int>(blockIdx.x >> 1);  // axis-1 pair group: positions 2 i1, 2 i1 + 1
  const int cl0 = 2 * i1 - a.p1off;
  const int j2 = 1 + static_cast<int>(blockIdx.y);  // axis-2 pair: positions 2 j2, 2 j2 + 1
  const int p1o = i1, p2o = j2;
  const int nbo = b ? O : E;
  const int nch = (nbo + U - 1) / U;

  auto issue_chunk = [&](int q) {
    uint64_t* bar = full + q % NBUF;
    mbar_expect_tx(bar, static_cast<uint32_t>(CHUNK * sizeof(double2)));
    tma_chunk(chunk + (q % NBUF) * CSTR, &tmS, 2 * (b * E + q * U), 0, p2o * (a.n1 + 1) + p1o, bar);
  };
  uint32_t rbuf_sa;  // the partner CTA's line buffer (other branch)
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rbuf_sa) : "r"(buf_sa), "r"(b ^ 1));

  if (tid == 0) {
    for (int i = 0; i < NBUF; ++i) {
      mbar_init(full + i, 1);
      cnt[i] = 0u;
    }
    mbar_init(inbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // both CTAs' input barriers exist before either multicasts into them
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  if (tid == 0) {
    mbar_expect_tx(inbar, static_cast<uint32_t>(N3 * LINES * sizeof(double2)));
    // input boxes j (k in [j KB, (j + 1) KB)): this CTA issues j == b (mod 2), multicast to both
    const int nbox = N3 / a.KB;
    for (int j = b; j < nbox; j += 2) {
      const int k = j * a.KB;
      const int r = k / a.nk;
      tma_load5_mc(buf + static_cast<size_t>(k) * LINES, &tmIn, 2 * cl0, 0, 2 * j2, k - r * a.nk, r, inbar, 3);
    }
    for (int i = 0; i < NBUF && i < nch; ++i) issue_chunk(i);
    // L2 prefetch of the cluster that will run on this SM pair next (about pf clusters on in
    // launch order): its input boxes (this CTA's half) and its spectrum rows of branch b
    if (a.pf > 0) {
      const int ng = static_cast<int>(gridDim.x >> 1);
      const int nxt = static_cast<int>(blockIdx.y) * ng + static_cast<int>(blockIdx.x >> 1) + a.pf;
      if (nxt < ng * static_cast<int>(gridDim.y)) {
        const int ni1 = a.gfirst + nxt % ng, nj2 = 1 + nxt / ng;
        for (int j = b; j < nbox; j += 2) {
          const int k = j * a.KB;
          const int r = k / a.nk;
          tma_prefetch5(&tmIn, 2 * (2 * ni1 - a.p1off), 0, 2 * nj2, k - r * a.nk, r);
        }
        for (int q = 0; q < nch; ++q) tma_prefetch3(&tmS, 2 * (b * E + q * U), 0, nj2 * (a.n1 + 1) + ni1);
      }
    }
  }
  P3_PHASE(0);
  mbar_wait(inbar, 0);
  P3_PHASE(1);

  // ---- forward stage 0 (radix R0) of this CTA's branch, in place: column (L, mp) reads the
  // inputs k = mp + i R1 and writes outputs k0 at slot k0 R1 + mp (the same slots)
  for (int t = tid; t < LINES * R1; t += SH::THREADS) {
    const int L = t % LINES, mp = t / LINES;
    double2 v[R0];
    const uint32_t base = buf_sa + 16u * static_cast<uint32_t>(mp * LINES + L);
#pragma unroll
    for (int i = 0; i < R0; ++i) v[i] = lds2(base + 16u * (i * R1 * LINES));
    // branch b: inputs * w_{2 R0}^{i b}, outputs * w_m3^{mp (2k + b)}
    if (b) {
      sfor<R0 - 1>([&](auto ic) {
        constexpr int i = decltype(ic)::value + 1;
        v[i] = twc<2 * R0, false, i>(v[i]);
      });
    }
    DFTs<R0, false, 1, 0>::run(v);
    const double2 wstep = __ldg(a.twm3 + 2 * mp);
    double2 w = b ? __ldg(a.twm3 + mp) : make_double2(1.0, 0.0);
    sfor<R0>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      sts2(base + 16u * (k * R1 * LINES), cmul(v[out_idx(R0, k)], w));
      if (k + 1 < R0) w = cmul(w, wstep);
    });
  }
  __syncthreads();
  P3_PHASE(2);
  // ---- forward stage 1 (radix R1), in place
  for (int t = tid; t < LINES * R0; t += SH::THREADS) {
    const int L = t % LINES, k0 = t / LINES;
    const uint32_t base = buf_sa + 16u * static_cast<uint32_t>(k0 * R1 * LINES + L);
    double2 w[R1];
#pragma unroll
    for (int i = 0; i < R1; ++i) w[i] = lds2(base + 16u * (i * LINES));
    DFTs<R1, false, 1, 0>::run(w);
    sfor<R1>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      sts2(base + 16u * (k * LINES), w[out_idx(R1, k)]);
    });
  }
  // ---- per-lane fragment bookkeeping (overlaps the barrier wait)
  constexpr auto SG = Signs<KIND, 1>::value;
  // pi[s] (3 bits each) packed into one constant: runtime-indexed without a local array
  constexpr unsigned long long PI = [] {
    unsigned long long v = 0;
    for (int i = 0; i < 12; ++i) v |= static_cast<unsigned long long>(Signs<KIND, 1>::value.pi[i]) << (3 * i);
    return v;
  }();
  auto pi_of = [](int i) { return static_cast<int>((PI >> (3 * i)) & 7ull); };
  const int gq = lane >> 2, tq = lane & 3;  // fragment group / thread in group
  // X (A operand, 8 x 4 row): point n = gq, source s = 4 ks + tq
  const int n_pt = gq;  // n = m1f | m2f << 1 | m3f << 2 (its bits are the mirror flags)
  const int xflag = n_pt >> 2;
  const uint32_t xline = static_cast<uint32_t>(24 * ((n_pt >> 1) & 1) + (n_pt & 1));
  unsigned long long xsg[3];
#pragma unroll
  for (int ks = 0; ks < 3; ++ks) xsg[ks] = pattern_sign(pi_of(4 * ks + tq) ^ SG.G, n_pt);
  // A (B operand, 4 x 8 col): source s = 4 ks + tq, target t = tau(nt, gq)
  int aoff[6];
  unsigned long long asg[6];
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    const int nt = f / 3, ks = f % 3;
    const int t = tau(nt, gq), s = 4 * ks + tq;
    const int c = t >= 0 ? c_bm3[KIND].c[t * 12 + s] : -1;
    aoff[f] = c >= 0 ? c * UB : -1;
    asg[f] = (c >= 0 && c_bm3[KIND].coef[t * 12 + s] < 0) ? (1ull << 63) : 0ull;
  }
  // Y (D, 8 x 8): point n = gq, targets tau(nt, 2 tq + e)
  int yt[2][2];
  unsigned long long ysg[2][2];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int t = tau(nt, 2 * tq + e);
      yt[nt][e] = t;
      ysg[nt][e] = t >= 0 ? pattern_sign(pi_of(t), n_pt) : 0ull;
    }
  __syncthreads();
  P3_PHASE(3);

  // ---- Hadamard: chunk q, warp w -> octant frequency u = q U + w
  for (int q = 0; q < nch; ++q) {
    const int bi = q % NBUF;
    const int u = q * U + warp;
    mbar_wait(full + bi, (q / NBUF) & 1);
    if (u < nbo) {
      const int f3o = 2 * u + b;
      const bool selfm = f3o == 0 || f3o == N3;
      const int slot0 = slot3<R0, R1>(u);
      const int slot1 = slot3<R0, R1>(selfm ? u : N3 - u - b);
      const uint32_t pbase = buf_sa + 16u * (static_cast<uint32_t>((xflag ? slot1 : slot0) * LINES) + xline);
      const double2* ch = chunk + bi * CSTR + warp;
      double2 xa[3], aa[6];
#pragma unroll
      for (int ks = 0; ks < 3; ++ks) xa[ks] = flip_sign(lds2(pbase + 16u * (2 * (4 * ks + tq))), xsg[ks]);
#pragma unroll
      for (int f = 0; f < 6; ++f)
        aa[f] = aoff[f] >= 0 ? flip_sign(ch[aoff[f]], asg[f]) : make_double2(0.0, 0.0);
      double p1[2][2] = {}, p2[2][2] = {}, p3[2][2] = {};
#pragma unroll
      for (int ks = 0; ks < 3; ++ks) {
        const double xr = xa[ks].x, xi = xa[ks].y, xs = xr + xi;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const double2 av = aa[nt * 3 + ks];
          dmma(p1[nt][0], p1[nt][1], xr, av.x);
          dmma(p2[nt][0], p2[nt][1], xi, av.y);
          dmma(p3[nt][0], p3[nt][1], xs, av.x + av.y);
        }
      }
      if (!(selfm && xflag)) {
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            if (yt[nt][e] < 0) continue;
            const double2 y = make_double2(p1[nt][e] - p2[nt][e], p3[nt][e] - p1[nt][e] - p2[nt][e]);
            sts2(pbase + 16u * (2 * yt[nt][e]), flip_sign(y, ysg[nt][e]));
          }
      }
    }
    // every read of buffer bi has been consumed by the DMMAs above; the last warp out refills it
    __syncwarp();
    if (lane == 0) {
      if (atomicAdd(cnt + bi, 1u) == SH::WARPS - 1) {
        cnt[bi] = 0u;
        if (q + NBUF < nch) {
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          issue_chunk(q + NBUF);
        }
      }
    }
  }
  __syncthreads();
  P3_PHASE(4);
  // ---- inverse stage 1 (adjoint of radix R1), in place
  for (int t = tid; t < LINES * R0; t += SH::THREADS) {
    const int L = t % LINES, k0 = t / LINES;
    const uint32_t base = buf_sa + 16u * static_cast<uint32_t>(k0 * R1 * LINES + L);
    double2 w[R1];
#pragma unroll
    for (int k = 0; k < R1; ++k) w[k] = lds2(base + 16u * (k * LINES));
    DFTs<R1, true, 1, 0>::run(w);
    sfor<R1>([&](auto ic) {
      constexpr int i = decltype(ic)::value;
      sts2(base + 16u * (i * LINES), w[out_idx(R1, i)]);
    });
  }
  // the partner's inverse stage 1 is complete (release / acquire) before its slots are read
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  P3_PHASE(5);
  // ---- inverse stage 0 of both branches + combine + crop: columns mp in [b HR1, (b+1) HR1)
  // of all 48 lines; y[n], n = mp + i R1, written in place (slot n)
  {
    const int L = tid % LINES, mp = b * HR1 + tid / LINES;
    const bool act = tid < LINES * HR1;
    const int mpc = act ? mp : 0;
    const uint32_t off = 16u * static_cast<uint32_t>(mpc * LINES + L);
    const double2 wstep = __ldg(a.twm3 + 2 * mpc);
    const double2 w1 = __ldg(a.twm3 + mpc);
    // branch br: inputs * conj(w_m3^{mp (2k + br)}), then the radix-R0 adjoint
    auto branch = [&](auto LD, int br, double2(&vv)[R0]) {
      double2 w = br ? w1 : wstep;
      vv[0] = br ? cmulc(LD(off), w) : LD(off);
      if (br) w = cmul(w, wstep);
#pragma unroll
      for (int k = 1; k < R0; ++k) {
        vv[k] = cmulc(LD(off + 16u * (k * R1 * LINES)), w);
        if (k + 1 < R0) w = cmul(w, wstep);
      }
      DFTs<R0, true, 1, 0>::run(vv);
    };
    double2 vo[R0], vr[R0];
    if (act) {
      branch([&](uint32_t o) { return lds2(buf_sa + o); }, b, vo);
      branch([&](uint32_t o) { return ldc2(rbuf_sa + o); }, b ^ 1, vr);
      P3_PHASE(6);
      sfor<R0>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        const double2 y0 = b ? vr[out_idx(R0, i)] : vo[out_idx(R0, i)];
        const double2 y1 = b ? vo[out_idx(R0, i)] : vr[out_idx(R0, i)];
        sts2(buf_sa + off + 16u * (i * R1 * LINES), cadd(y0, twc<2 * R0, true, i>(y1)));
      });
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    // output slots k = i R1 + [b HR1, (b+1) HR1) of all 48 lines -> Bout (KBS-slot boxes)
    if (tid == 0) {
      for (int i = 0; i < R0; ++i)
        for (int kk = 0; kk < HR1; kk += a.KBS) {
          const int k = i * R1 + b * HR1 + kk;
          const int r = k / a.nk;
          tma_store5(&tmOut, buf + static_cast<size_t>(k) * LINES, 2 * cl0, 0, 2 * j2, k - r * a.nk, r);
        }
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    }
    // the partner finished reading this CTA's slots before either exits
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    P3_PHASE(7);
  }
}

#define VIE_PENCIL3_SHAPES(X) X(10, 20) X(10, 10) X(8, 16) X(8, 8) X(4, 8) X(8, 20) X(10, 12) X(8, 12) X(8, 10) X(6, 8)

// k extent of the load boxes: a divisor of nk, at most 128 (<= 256 per TMA box dim)
int load_box_k(int nk) {
  int kb = nk;
  while (kb > 128 && kb % 2 == 0) kb /= 2;
  return kb <= 256 ? kb : -1;
}

template <int KIND>
bool launch3_t(int n3, const double2* Bin, double2* Bout, const double2* Shat, const Geom& g, const double2* twm3,
               cudaStream_t st, bool dry) {
  auto go = [&](auto fn, size_t smem, int UB, int NC, int R1) {
    const int kb = load_box_k(g.nk), kbs = std::gcd(R1 / 2, g.nk);
    if (kb < 1 || g.n3 % kb) return false;
    if (dry) return true;
    // interior axis-1 pair groups of this rank's positions [p1off, p1off + W); group 0 is the edge launch
    const int glo = std::max(1, g.p1off / 2);
    const int ghi = std::min(g.m1, g.p1off + g.W) / 2;
    if (ghi <= glo || g.n2 < 2) return true;
    VIE_CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    Pencil3Args a{twm3, g.n1, g.W, g.p1off, glo, g.nk, kb, kbs, 0};
    CUtensorMap tmS, tmIn, tmOut;
    encode_spectrum_map(&tmS, Shat, g, {2 * UB, NC, 1});
    encode_slab_map(&tmIn, Bin, g, kb, 2);
    encode_slab_map(&tmOut, Bout, g, kbs, 2);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * (ghi - glo), g.n2 - 1);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    static const int pf_env = std::getenv("VIE_P3_PF") ? std::atoi(std::getenv("VIE_P3_PF")) : -1;
    if (pf_env != 0) {
      int ncl = 0;
      VIE_CUDA_CHECK(cudaOccupancyMaxActiveClusters(&ncl, reinterpret_cast<const void*>(fn), &cfg));
      a.pf = pf_env > 0 ? pf_env : ncl;
    }
    VIE_CUDA_CHECK(cudaLaunchKernelEx(&cfg, fn, a, tmS, tmIn, tmOut));
    VIE_CUDA_CHECK(cudaGetLastError());
    return true;
  };
#define VIE_CASE3(A, B)                                                     \
  if (n3 == (A) * (B)) {                                                    \
    using SH = Shape3<KIND, A, B>;                                          \
    if (SH::smem_bytes > kMaxSmem) return false;                            \
    return go(k_pencil3<KIND, A, B>, SH::smem_bytes, SH::UB, SH::NC, B);    \
  }
  VIE_PENCIL3_SHAPES(VIE_CASE3)
#undef VIE_CASE3
  return false;
}

}  // namespace

#ifdef VIE_PENCIL_PROFILE
void pencil3_phase_read(unsigned long long* out8, bool reset) {
  cudaMemcpyFromSymbol(out8, g_p3_phase, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_p3_phase, z, sizeof(z));
  }
}
#endif

bool pencil3_supported(int kind, int basis, int n3, uint64_t active_mask, int NC) {
  if (basis != 1) return false;
  const uint64_t all = NC >= 64 ? ~0ull : ((1ull << NC) - 1);
  if (active_mask != all) return false;
  if (std::getenv("VIE_NO_PENCIL3")) return false;
  Geom g{};
  g.n3 = n3;
  g.nk = n3;
  return kind == 0 ? launch3_t<0>(n3, nullptr, nullptr, nullptr, g, nullptr, nullptr, true)
                   : launch3_t<1>(n3, nullptr, nullptr, nullptr, g, nullptr, nullptr, true);
}

void launch_pencil3(int kind, const double2* Bin, double2* Bout, const double2* Shat, const Geom& g,
                    const double2* twm3, cudaStream_t st) {
  const bool ok = kind == 0 ? launch3_t<0>(g.n3, Bin, Bout, Shat, g, twm3, st, false)
                            : launch3_t<1>(g.n3, Bin, Bout, Shat, g, twm3, st, false);
  if (!ok) throw CudaError(cudaErrorInvalidValue, "pencil3: unsupported slab geometry", __FILE__, __LINE__);
}

}  // namespace vie
