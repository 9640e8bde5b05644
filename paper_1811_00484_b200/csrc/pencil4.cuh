// pencil4.cuh -- the work item of the half-mirror-group DMMA pencil kernel (see
// kernels_pencil4.cu for the math), shared by the standalone launch (k_pencil4) and the fused
// decompress x pencil persistent kernel (kernels_fused.cu).
#pragma once
#include <cuda.h>

#include "fft.cuh"
#include "hadamard.cuh"
#include "kernels.cuh"
#include "tma.cuh"

#ifndef VIE_P4_NBUF
#define VIE_P4_NBUF 3
#endif
#ifndef VIE_P4_SMTW  // 1: the w_m3 table (2 n3 entries) staged in shared memory per item
#define VIE_P4_SMTW 1
#endif

namespace vie {
namespace p4 {

using namespace had;

template <int KIND, int R0, int R1>
struct Shape4 {
  static constexpr int NC = TableDims<KIND, 1>::NC;
  static constexpr int THREADS = 256;
  static constexpr int WARPS = THREADS / 32;
  static constexpr int LINES = 24;         // 2 pencils x 12 currents, line L = 2 s + m1f
  static constexpr int N3 = R0 * R1;       // branch length (= n3)
  static constexpr int HR1 = R1 / 2;       // last-stage columns finalised per CTA
  static constexpr int U = WARPS;          // octant frequencies per chunk (one per warp)
  static constexpr int UB = U + 1;         // box width: one pad column (bank spread of the gather)
  static constexpr int E = N3 / 2 + 1;     // even octant frequencies (branch 0)
  static constexpr int O = (N3 + 1) / 2;   // odd octant frequencies (branch 1)
  static constexpr int NBUF = VIE_P4_NBUF;
  static constexpr int CHUNK = UB * NC;                              // double2 per chunk
  static constexpr int ZOFF = CHUNK;                                   // 8 zero double2 after the TMA box
  static constexpr int CHUNK_STRIDE = ((CHUNK + 8) * 16 + 127) / 128 * 8;  // double2, 128-byte aligned buffers
  static constexpr int BUF_ELEMS = N3 * LINES;
  static constexpr int TW_ELEMS = VIE_P4_SMTW ? 2 * N3 : 0;  // w_m3^e, e < m3 (after the line buffer)
  static constexpr size_t smem_bytes =
      128 + sizeof(double2) * (static_cast<size_t>(NBUF) * CHUNK_STRIDE + BUF_ELEMS + TW_ELEMS);
  static_assert(LINES * HR1 <= THREADS && LINES * R0 <= THREADS, "one FFT unit per thread");
  static_assert(R1 % 2 == 0, "the last inverse stage splits its columns between the CTAs");
};

// m-tile rows -> targets (tile 1 rows 4..7 are padding)
__device__ __forceinline__ int tau4(int mt, int r) { return mt == 0 ? r : (r < 4 ? 8 + r : -1); }

template <int R0, int R1>
__device__ __forceinline__ int slot4(int phi) {  // slot of branch frequency phi = k0 + R0 k1
  return (phi % R0) * R1 + phi / R0;
}

// (component, coefficient) of block (t, s) of the PWL table; c = -1: no block.
struct BlockMatrix4 {
  int c[144];
  int coef[144];
};
template <int KIND>
constexpr BlockMatrix4 make_block_matrix4() {
  BlockMatrix4 m{};
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
static __device__ const BlockMatrix4 c_bm4[2] = {make_block_matrix4<0>(), make_block_matrix4<1>()};

struct Pencil4Args {
  const double2* twm3;  // w_m3^e, e < m3
  int n1;
  int W;
  int p1off;
  int gfirst;  // first axis-1 pair group of this launch (>= 1)
  int nk;      // k-planes per slab block
  int KB;      // k extent of a load box (divides nk)
  int KBS;     // k extent of a store box (divides nk and R1 / 2)
  int pf;      // L2 prefetch distance in clusters (0 = off)
};

#ifdef VIE_PENCIL_PROFILE
static __device__ unsigned long long g_p4_phase[8];
#define P4_PHASE(i)                                                                   \
  do {                                                                                \
    if (threadIdx.x == 0) {                                                           \
      const long long t_ = clock64();                                                 \
      atomicAdd(&g_p4_phase[i], static_cast<unsigned long long>(t_ - t_last));        \
      t_last = t_;                                                                    \
    }                                                                                 \
  } while (0)
#else
#define P4_PHASE(i) \
  do {              \
  } while (0)
#endif

__device__ __forceinline__ double flip1(double v, unsigned long long sbit) {
  return __longlong_as_double(__double_as_longlong(v) ^ static_cast<long long>(sbit));
}

// Shared-memory header of the pencil CTAs (kernels_pencil4.cu k_pencil4, kernels_fused.cu)
struct P4Smem {
  uint64_t* full;   // [NBUF] spectrum ring mbarriers
  uint64_t* inbar;  // input boxes
  uint64_t* rdone;  // standalone: the partner's DSMEM reads of this CTA are done
  unsigned* cnt;    // [NBUF] refill counters
  int* item;        // fused: the cluster's current work item
  double2* chunk;   // [NBUF][CSTR] spectrum ring, then the line buffer
};
template <int NBUF>
__device__ __forceinline__ P4Smem p4_smem(unsigned char* smraw) {
  P4Smem s;
  s.full = reinterpret_cast<uint64_t*>(smraw);
  s.inbar = s.full + NBUF;
  s.rdone = s.inbar + 1;
  s.cnt = reinterpret_cast<unsigned*>(s.rdone + 1);
  s.item = reinterpret_cast<int*>(s.cnt + NBUF);
  s.chunk = reinterpret_cast<double2*>(smraw + 128);
  return s;
}

// One work item of the pencil kernel: the two pencils (p1, m1-p1) = axis-1 pair group i1 at
// axis-2 position 2 j2 + m2f, branch b (cluster rank).  srow: spectrum row of the octant line
// (p1o, p2o) = (i1, j2) in tmS; qbase: spectrum chunks this CTA issued before (ring slot and
// mbarrier phase); inpar: phase of the input mbarrier.  spectrum_ready() runs on thread 0
// before the first chunk is issued, spectrum_consumed() on every thread after the Hadamard.
template <int KIND, int R0, int R1, bool STANDALONE, class Ready, class Consumed>
__device__ __forceinline__ void p4_item(const Pencil4Args& a, const CUtensorMap* tmS, const CUtensorMap* tmIn,
                                        const CUtensorMap* tmOut, const P4Smem& sm, int i1, int m2f, int j2, int b,
                                        int srow, uint32_t qbase, uint32_t inpar, Ready spectrum_ready,
                                        Consumed spectrum_consumed) {
  using SH = Shape4<KIND, R0, R1>;
#ifdef VIE_PENCIL_PROFILE
  long long t_last = clock64();
#endif
  constexpr int LINES = SH::LINES, N3 = SH::N3, HR1 = SH::HR1;
  constexpr int U = SH::U, UB = SH::UB, E = SH::E, O = SH::O, NBUF = SH::NBUF;
  constexpr int CHUNK = SH::CHUNK, CSTR = SH::CHUNK_STRIDE;
  uint64_t* full = sm.full;
  uint64_t* inbar = sm.inbar;
  uint64_t* rdone = sm.rdone;
  unsigned* cnt = sm.cnt;
  double2* chunk = sm.chunk;
  double2* buf = chunk + NBUF * CSTR;  // [slot][L]
  const uint32_t buf_sa = smem_u32(buf);
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int cl = 2 * (i1 - a.gfirst) + m2f;  // standalone launch order (L2 prefetch)
  const int cl0 = 2 * i1 - a.p1off;
  const int pos2 = 2 * j2 + m2f;
  const int nbo = b ? O : E;
  const int nch = (nbo + U - 1) / U;
  (void)rdone;
  (void)cl;
  // chunk q of this item is the (qbase + q)-th use of the ring: slot and mbarrier phase follow it
  auto issue_chunk = [&](int q) {
    const uint32_t gq = qbase + static_cast<uint32_t>(q);
    uint64_t* bar = full + gq % NBUF;
    mbar_expect_tx(bar, static_cast<uint32_t>(CHUNK * sizeof(double2)));
    tma_chunk(chunk + (gq % NBUF) * CSTR, tmS, 2 * (b * E + q * U), 0, srow, bar);
  };
  uint32_t rbuf_sa;  // the partner CTA's line buffer (other branch)
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rbuf_sa) : "r"(buf_sa), "r"(b ^ 1));

  if (tid < NBUF * 8) chunk[(tid >> 3) * CSTR + SH::ZOFF + (tid & 7)] = make_double2(0.0, 0.0);
  if (tid == 0) {
    mbar_expect_tx(inbar, static_cast<uint32_t>(N3 * LINES * sizeof(double2)));
    // input boxes j (k in [j KB, (j + 1) KB)): this CTA issues j == b (mod 2), multicast to both
    const int nbox = N3 / a.KB;
    for (int j = b; j < nbox; j += 2) {
      const int k = j * a.KB;
      const int r = k / a.nk;
      if (STANDALONE) tma_load5_mc(buf + static_cast<size_t>(k) * LINES, tmIn, 2 * cl0, 0, pos2, k - r * a.nk, r, inbar, 3);
      else
        tma_load5_mc_hint(buf + static_cast<size_t>(k) * LINES, tmIn, 2 * cl0, 0, pos2, k - r * a.nk, r, inbar, 3,
                          l2_evict_first());
    }
  }
#if VIE_P4_SMTW
  // the stage-0 / inverse-stage-0 twiddles w_m3^e from shared memory instead of L1 (__ldg);
  // filled after the input loads are issued and before (fused kernel) thread 0 waits for the
  // spectrum tile, so this barrier never waits on that spin
  const double2* twm3 = buf + SH::BUF_ELEMS;
  for (int e = tid; e < 2 * N3; e += SH::THREADS) buf[SH::BUF_ELEMS + e] = __ldg(a.twm3 + e);
  __syncthreads();
#define P4_TW(e) twm3[e]
#else
#define P4_TW(e) __ldg(a.twm3 + (e))
#endif
  if (tid == 0) {
    spectrum_ready();  // the fused kernel waits here for this item's spectrum tile
    for (int i = 0; i < NBUF && i < nch; ++i) issue_chunk(i);
  }
  P4_PHASE(0);
  mbar_wait(inbar, inpar);
  P4_PHASE(1);

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
    // outputs * w_m3^{mp (2k + b)}: exponents walked in integers, twiddles from the table (L1)
    int ex = b ? mp : 0;
    sfor<R0>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      const double2 y = (k == 0 && b == 0) ? v[out_idx(R0, k)] : cmul(v[out_idx(R0, k)], P4_TW(ex));
      sts2(base + 16u * (k * R1 * LINES), y);
      ex += 2 * mp;
      if (ex >= 2 * N3) ex -= 2 * N3;
    });
  }
  __syncthreads();
  P4_PHASE(2);
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
  constexpr unsigned long long PI = [] {
    unsigned long long v = 0;
    for (int i = 0; i < 12; ++i) v |= static_cast<unsigned long long>(Signs<KIND, 1>::value.pi[i]) << (3 * i);
    return v;
  }();
  auto pi_of = [](int i) { return static_cast<int>((PI >> (3 * i)) & 7ull); };
  const int gq = lane >> 2, tq = lane & 3;  // fragment group / thread in group
  // X (B operand, 4 x 8 col): source s = 4 ks + tq; column gq = m1f | part << 1 | m3f << 2, so a
  // half warp (gq < 4 / gq >= 4) reads one 128-byte run of one slot (no bank conflict between
  // the two mirror slots)
  const int xm1 = gq & 1, xpart = (gq >> 1) & 1, xm3 = gq >> 2;
  const uint32_t xoff = static_cast<uint32_t>(16 * xm1 + 8 * xpart);  // bytes: m1f line, re / im
  unsigned long long xsg[3];
#pragma unroll
  for (int ks = 0; ks < 3; ++ks)
    xsg[ks] = pattern_sign(pi_of(4 * ks + tq) ^ SG.G, xm1 | (m2f << 1) | (xm3 << 2));
  // A (8 x 4 row): target t = tau4(mt, gq), source s = 4 ks + tq
  int aoff[6];
  unsigned long long asg[6];
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    const int mt = f / 3, ks = f % 3;
    const int t = tau4(mt, gq), s = 4 * ks + tq;
    const int c = t >= 0 ? c_bm4[KIND].c[t * 12 + s] : -1;
    aoff[f] = c >= 0 ? c * UB : SH::ZOFF - warp;  // no block / padding row: a zero slot
    asg[f] = (c >= 0 && c_bm4[KIND].coef[t * 12 + s] < 0) ? (1ull << 63) : 0ull;
  }
  // D (8 x 8): row gq = target tau4(mt, gq); columns 2 tq + e = m1f e, part tq & 1, m3f tq >> 1
  // (after the exchange with lane tq ^ 1 each lane finalises one double)
  const int ym3 = tq >> 1, ypart = tq & 1;
  const unsigned long long ysub = ypart ? 0ull : (1ull << 63);  // Yr = D1 - D2', Yi = D1 + D2'
  uint32_t yoff[2][2];  // [mt][e] bytes within a slot; ~0u: padding row
  unsigned long long ysg[2][2];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int t = tau4(mt, gq);
      yoff[mt][e] = t >= 0 ? static_cast<uint32_t>(16 * (2 * t + e) + 8 * ypart) : ~0u;
      ysg[mt][e] = t >= 0 ? pattern_sign(pi_of(t), e | (m2f << 1) | (ym3 << 2)) : 0ull;
    }
  __syncthreads();
  P4_PHASE(3);

  // ---- Hadamard: chunk q, warp w -> octant frequency u = q U + w
  for (int q = 0; q < nch; ++q) {
    const uint32_t gq = qbase + static_cast<uint32_t>(q);
    const int bi = static_cast<int>(gq % NBUF);
    const int u = q * U + warp;
    mbar_wait(full + bi, (gq / NBUF) & 1);
    if (u < nbo) {
      const int f3o = 2 * u + b;
      const bool selfm = f3o == 0 || f3o == N3;
      const int slot0 = slot4<R0, R1>(u);
      const int slot1 = slot4<R0, R1>(selfm ? u : N3 - u - b);
      const uint32_t xbase = buf_sa + 16u * static_cast<uint32_t>((xm3 ? slot1 : slot0) * LINES) + xoff;
      const double2* ch = chunk + bi * CSTR + warp;
      double xb[3];
      double2 aa[6];
#pragma unroll
      for (int ks = 0; ks < 3; ++ks) xb[ks] = flip1(lds1(xbase + 32u * (4 * ks + tq)), xsg[ks]);
#pragma unroll
      for (int f = 0; f < 6; ++f) aa[f] = flip_sign(ch[aoff[f]], asg[f]);
      double d1[2][2] = {}, d2[2][2] = {};
#pragma unroll
      for (int ks = 0; ks < 3; ++ks)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const double2 av = aa[mt * 3 + ks];
          dmma(d1[mt][0], d1[mt][1], av.x, xb[ks]);
          dmma(d2[mt][0], d2[mt][1], av.y, xb[ks]);
        }
      const uint32_t ybase = buf_sa + 16u * static_cast<uint32_t>((ym3 ? slot1 : slot0) * LINES);
      const bool ystore = !(selfm && ym3);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double v = __shfl_xor_sync(0xffffffffu, d2[mt][e], 1);
          const double r = d1[mt][e] + flip1(v, ysub);
          if (ystore && yoff[mt][e] != ~0u) sts1(ybase + yoff[mt][e], flip1(r, ysg[mt][e]));
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
  spectrum_consumed();  // every chunk of this item has landed and been read
  P4_PHASE(4);
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
  P4_PHASE(5);
  // ---- inverse stage 0 of both branches + combine + crop: columns mp in [b HR1, (b+1) HR1)
  // of all 24 lines; y[n], n = mp + i R1, written in place (slot n)
  {
    const int L = tid % LINES, mp = b * HR1 + tid / LINES;
    const bool act = tid < LINES * HR1;
    const int mpc = act ? mp : 0;
    const uint32_t off = 16u * static_cast<uint32_t>(mpc * LINES + L);
    // branch br: inputs * conj(w_m3^{mp (2k + br)}) (exponents walked in integers, twiddles
    // from the table), then the radix-R0 adjoint
    auto branch = [&](auto LD, int br, double2(&vv)[R0]) {
      int ex = br ? mpc : 0;
      vv[0] = br ? cmulc(LD(off), P4_TW(ex)) : LD(off);
#pragma unroll
      for (int k = 1; k < R0; ++k) {
        ex += 2 * mpc;
        if (ex >= 2 * N3) ex -= 2 * N3;
        vv[k] = cmulc(LD(off + 16u * (k * R1 * LINES)), P4_TW(ex));
      }
      DFTs<R0, true, 1, 0>::run(vv);
    };
    double2 vo[R0], vr[R0];
    if (act) {
      branch([&](uint32_t o) { return lds2(buf_sa + o); }, b, vo);
      branch([&](uint32_t o) { return ldc2(rbuf_sa + o); }, b ^ 1, vr);
      P4_PHASE(6);
      sfor<R0>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        const double2 y0 = b ? vr[out_idx(R0, i)] : vo[out_idx(R0, i)];
        const double2 y1 = b ? vo[out_idx(R0, i)] : vr[out_idx(R0, i)];
        sts2(buf_sa + off + 16u * (i * R1 * LINES), cadd(y0, twc<2 * R0, true, i>(y1)));
      });
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    // output slots k = i R1 + [b HR1, (b+1) HR1) of all 24 lines -> Bout (KBS-slot boxes).
    // Only thread 0 stays: it tells the partner that this CTA's reads of the partner's slots
    // are over (remote arrive, after the barrier above), and keeps this CTA's shared memory
    // alive until the partner has said the same (the CTA's resources outlive the other threads).
    if (tid == 0) {
      if (STANDALONE) {
        uint32_t prd;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(prd) : "r"(smem_u32(rdone)), "r"(b ^ 1));
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(prd) : "memory");
      }
      for (int i = 0; i < R0; ++i)
        for (int kk = 0; kk < HR1; kk += a.KBS) {
          const int k = i * R1 + b * HR1 + kk;
          const int r = k / a.nk;
          if (STANDALONE) tma_store5(tmOut, buf + static_cast<size_t>(k) * LINES, 2 * cl0, 0, pos2, k - r * a.nk, r);
          else
            tma_store5_hint(tmOut, buf + static_cast<size_t>(k) * LINES, 2 * cl0, 0, pos2, k - r * a.nk, r,
                            l2_evict_first());
        }
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
      if (STANDALONE) mbar_wait(rdone, 0);
    }
    P4_PHASE(7);
  }
#undef P4_TW
}

}  // namespace p4
}  // namespace vie
