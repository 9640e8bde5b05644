// kernels_decomp.cu -- Tucker decompression of the component spectra on their
// octant (|p_q| <= n_q), and the device-side factor transform.
//
// Reference: decompress_tucker (operator.hpp:224-244) materialises the full
// m1 x m2 x m3 spectrum per component (GEMM chain c1 = U1 G, c2 = c1 U2^T,
// dst = c2 U3^T).  Here only the octant is formed (1/8 of the entries and of
// the dominant r3 * N_e flops), for all components at once:
//   k_decomp_z : Z_c[p2][a][g] = sum_b G_c[a,b,g] U2_c[p2,b]        (r^3 per p2)
//   k_decomp_s : T = U1_c Z_c[p2]  (n1+1 x r3),  S^_c[p2][p1][f3] = T U3_c^T
// Output layout Shat[p2o][p1o][c][bidx(f3o)], axis 3 branch-major (even
// octant frequencies 0,2,.. first, then odd 1,3,..) to match the pencil
// kernel's even/odd half-length branches.
#include <cstdlib>

#include "decomp_tile.cuh"
#include "kernels.cuh"

namespace vie {

namespace {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all_d() {
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// CTA per (component, g): Z_c[p2][a][g] for one core slice G[:,:,g] (read through the
// cache: consecutive threads take consecutive a, so the slice reads coalesce).
__global__ void __launch_bounds__(kThreads) k_decomp_z(const double2* __restrict__ forms,
                                                       const CompDev* __restrict__ comps, double2* __restrict__ Z,
                                                       int n2) {
  const CompDev cd = comps[blockIdx.x];
  const int g = blockIdx.y;
  if (!cd.active || g >= cd.r3) return;
  const int r1 = cd.r1, r2 = cd.r2, r3 = cd.r3;
  const double2* core = forms + cd.off_core + static_cast<int64_t>(g) * r1 * r2;  // core[a + r1*b]
  const double2* u2 = forms + cd.off_u2;  // (n2+1) x r2
  const int np = n2 + 1;
  double2* zc = Z + cd.off_z;
  for (int e = threadIdx.x; e < np * r1; e += blockDim.x) {
    const int a = e % r1, p2 = e / r1;
    // four independent partial sums: the loads of four b run ahead of the FMA chain
    double2 acc[4] = {};
    int b = 0;
    for (; b + 4 <= r2; b += 4)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        cfma(acc[i], __ldg(core + a + r1 * (b + i)), __ldg(u2 + p2 + static_cast<int64_t>(np) * (b + i)));
    for (; b < r2; ++b) cfma(acc[0], __ldg(core + a + r1 * b), __ldg(u2 + p2 + static_cast<int64_t>(np) * b));
    zc[(static_cast<int64_t>(p2) * r1 + a) * r3 + g] =
        make_double2((acc[0].x + acc[1].x) + (acc[2].x + acc[3].x), (acc[0].y + acc[1].y) + (acc[2].y + acc[3].y));
  }
}

constexpr int kTP1 = 32;  // p1 rows per chunk
constexpr int kQ = 4;     // micro-tile 4 x 4

// CTA per (component, p2o).
__global__ void __launch_bounds__(kThreads) k_decomp_s(const double2* __restrict__ forms,
                                                       const CompDev* __restrict__ comps,
                                                       const double2* __restrict__ Z, double2* __restrict__ Shat,
                                                       Geom geo, int NC, int p2lo, int p1lo, int p1hi) {
  extern __shared__ double2 sm[];
  const int c = blockIdx.x;
  const CompDev cd = comps[c];
  if (!cd.active) return;
  const int p2o = p2lo + blockIdx.y;
  const int r1 = cd.r1, r3 = cd.r3;
  const int n1p = geo.n1 + 1, n3p = geo.n3 + 1;
  double2* zs = sm;                                   // r1 x r3   zs[a*r3 + g]
  double2* us = zs + r1 * r3;                         // r3 x n3p  us[g*n3p + f]
  double2* ts = us + static_cast<int64_t>(r3) * n3p;  // r3 x kTP1 ts[g*kTP1 + i]
  const double2* zsrc = Z + cd.off_z + static_cast<int64_t>(p2o) * r1 * r3;
  for (int e = threadIdx.x; e < r1 * r3; e += blockDim.x) zs[e] = zsrc[e];
  const double2* u3 = forms + cd.off_u3;  // n3p x r3 col-major: u3[f + n3p*g]
  for (int e = threadIdx.x; e < r3 * n3p; e += blockDim.x) us[e] = u3[e];
  const double2* u1 = forms + cd.off_u1;  // n1p x r1
  for (int p10 = p1lo; p10 < p1hi; p10 += kTP1) {
    const int np1 = min(kTP1, p1hi - p10);
    __syncthreads();
    for (int e = threadIdx.x; e < kTP1 * r3; e += blockDim.x) {
      const int i = e % kTP1, g = e / kTP1;
      double2 acc = make_double2(0.0, 0.0);
      if (i < np1)
        for (int a = 0; a < r1; ++a) cfma(acc, __ldg(u1 + (p10 + i) + static_cast<int64_t>(n1p) * a), zs[a * r3 + g]);
      ts[g * kTP1 + i] = acc;
    }
    __syncthreads();
    // warp tile: 4 rows (p1o) x 128 columns (f3o = fb + lane + 32 j): T values
    // are warp broadcasts, U3 values are read by consecutive lanes (no bank
    // conflicts), 16 complex accumulators per thread.
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    const int nfb = (n3p + 127) / 128;
    const int wtiles = (kTP1 / kQ) * nfb;
    const int E = geo.n3 / 2 + 1;
    for (int t = warp; t < wtiles; t += nwarp) {
      const int fb = (t % nfb) * 128, rq = t / nfb;
      double2 acc[kQ][kQ];
#pragma unroll
      for (int i = 0; i < kQ; ++i)
#pragma unroll
        for (int j = 0; j < kQ; ++j) acc[i][j] = make_double2(0.0, 0.0);
      for (int g = 0; g < r3; ++g) {
        double2 tv[kQ], uv[kQ];
#pragma unroll
        for (int i = 0; i < kQ; ++i) tv[i] = ts[g * kTP1 + rq * kQ + i];
#pragma unroll
        for (int j = 0; j < kQ; ++j) {
          const int f = fb + lane + 32 * j;
          uv[j] = f < n3p ? us[g * n3p + f] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int i = 0; i < kQ; ++i)
#pragma unroll
          for (int j = 0; j < kQ; ++j) cfma(acc[i][j], tv[i], uv[j]);
      }
#pragma unroll
      for (int i = 0; i < kQ; ++i) {
        const int p1o = p10 + rq * kQ + i;
        if (rq * kQ + i >= np1) break;
        double2* dst = Shat + ((static_cast<int64_t>(p2o) * n1p + p1o) * NC + c) * n3p;
#pragma unroll
        for (int j = 0; j < kQ; ++j) {
          const int f = fb + lane + 32 * j;
          if (f < n3p) dst[(f & 1) ? E + (f >> 1) : (f >> 1)] = acc[i][j];
        }
      }
    }
  }
}

// Large-rank fallback (ranks beyond both tiles above, e.g. tight-tolerance HOSVD forms):
// CTA per (component, p2o); only the T chunk (r3 x kTP1) is staged, Z and U3 are read
// through the cache (Z_c[p2o] and U3_c are re-read by every chunk: L1/L2 resident).
__global__ void __launch_bounds__(kThreads) k_decomp_s_big(const double2* __restrict__ forms,
                                                           const CompDev* __restrict__ comps,
                                                           const double2* __restrict__ Z, double2* __restrict__ Shat,
                                                           Geom geo, int NC, int p2lo, int p1lo, int p1hi) {
  extern __shared__ double2 sm[];
  const int c = blockIdx.x;
  const CompDev cd = comps[c];
  if (!cd.active) return;
  const int p2o = p2lo + blockIdx.y;
  const int r1 = cd.r1, r3 = cd.r3;
  const int n1p = geo.n1 + 1, n3p = geo.n3 + 1;
  double2* ts = sm;  // r3 x kTP1: ts[g*kTP1 + i]
  const double2* zsrc = Z + cd.off_z + static_cast<int64_t>(p2o) * r1 * r3;  // [a][g]
  const double2* u3 = forms + cd.off_u3;  // n3p x r3 col-major
  const double2* u1 = forms + cd.off_u1;  // n1p x r1
  const int E = geo.n3 / 2 + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  for (int p10 = p1lo; p10 < p1hi; p10 += kTP1) {
    const int np1 = min(kTP1, p1hi - p10);
    __syncthreads();
    for (int e = threadIdx.x; e < kTP1 * r3; e += blockDim.x) {
      const int i = e % kTP1, g = e / kTP1;
      double2 acc = make_double2(0.0, 0.0);
      if (i < np1)
        for (int a = 0; a < r1; ++a)
          cfma(acc, __ldg(u1 + (p10 + i) + static_cast<int64_t>(n1p) * a), __ldg(zsrc + static_cast<int64_t>(a) * r3 + g));
      ts[g * kTP1 + i] = acc;
    }
    __syncthreads();
    const int nfb = (n3p + 127) / 128;
    const int wtiles = (kTP1 / kQ) * nfb;
    for (int t = warp; t < wtiles; t += nwarp) {
      const int fb = (t % nfb) * 128, rq = t / nfb;
      double2 acc[kQ][kQ];
#pragma unroll
      for (int i = 0; i < kQ; ++i)
#pragma unroll
        for (int j = 0; j < kQ; ++j) acc[i][j] = make_double2(0.0, 0.0);
      for (int g = 0; g < r3; ++g) {
        double2 tv[kQ], uv[kQ];
#pragma unroll
        for (int i = 0; i < kQ; ++i) tv[i] = ts[g * kTP1 + rq * kQ + i];
#pragma unroll
        for (int j = 0; j < kQ; ++j) {
          const int f = fb + lane + 32 * j;
          uv[j] = f < n3p ? __ldg(u3 + f + static_cast<int64_t>(n3p) * g) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int i = 0; i < kQ; ++i)
#pragma unroll
          for (int j = 0; j < kQ; ++j) cfma(acc[i][j], tv[i], uv[j]);
      }
#pragma unroll
      for (int i = 0; i < kQ; ++i) {
        const int p1o = p10 + rq * kQ + i;
        if (rq * kQ + i >= np1) break;
        double2* dst = Shat + ((static_cast<int64_t>(p2o) * n1p + p1o) * NC + c) * n3p;
#pragma unroll
        for (int j = 0; j < kQ; ++j) {
          const int f = fb + lane + 32 * j;
          if (f < n3p) dst[(f & 1) ? E + (f >> 1) : (f >> 1)] = acc[i][j];
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Octant decompression on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64).
// CTA = (component c, PP consecutive p2o).  U3_c staged once in smem as the
// B operand; per p2o: T = U1_c Z_c[p2o] (FMA, 4% of the flops) into smem as the
// A operand, then S^ = T U3^T as a complex GEMM = 3 real DMMAs per 8x8x4 step (Gauss).
// Fragment smem layout [row][Kp] with Kp = 4 (mod 8): conflict-free quarter-warps.
constexpr int kMmaMC = 64;   // rows (p1o) per T chunk
#ifndef VIE_DECOMP_PP
#define VIE_DECOMP_PP 4
#endif
constexpr int kMmaPP = VIE_DECOMP_PP;  // p2o values per CTA (U3 / U1 staging reuse)
constexpr int kZS = 34;      // Z row stride (== 2 mod 8: conflict-free B fragments over k)
#ifndef VIE_DECOMP_THREADS
#define VIE_DECOMP_THREADS 384
#endif
constexpr int kMmaThreads = VIE_DECOMP_THREADS;  // 12 warps: 256 -> 384 measured 0.8 % faster, 512 5 % slower; warps beyond the T tiles only run the S^ GEMM
constexpr int kTWarps = kMmaMC / 16 * 2;          // one 16 x 16 T tile per warp
static_assert(kMmaThreads / 32 >= kTWarps, "every T tile needs a warp");

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__host__ __device__ __forceinline__ int mma_kp(int r3) {
  int kp = (r3 + 3) / 4 * 4;
  if (kp % 8 == 0) kp += 4;
  return kp;
}

__global__ void __launch_bounds__(kMmaThreads, 1) k_decomp_s_mma(const double2* __restrict__ forms,
                                                              const CompDev* __restrict__ comps,
                                                              const double2* __restrict__ Z,
                                                              double2* __restrict__ Shat, Geom geo, int NC, int p2lo,
                                                              int p2hi, int p1lo, int p1hi) {
  extern __shared__ double2 sm[];
  const int c = blockIdx.x;
  const CompDev cd = comps[c];
  if (!cd.active) return;
  const int r1 = cd.r1, r3 = cd.r3;
  const int n1p = geo.n1 + 1, n3p = geo.n3 + 1;
  const int Kp = mma_kp(r3);
  const int KA = mma_kp(r1);  // T = U1 Z inner dimension (padded)
  const int NPad = (n3p + 15) / 16 * 16;
  double2* us = sm;                                    // [NPad][Kp]  B operand (U3)
  double2* zs = us + static_cast<int64_t>(NPad) * Kp;  // [KA][kZS]   B operand of T (Z, zero padded)
  double2* ts = zs + KA * kZS;                         // [kMmaMC][Kp] A operand (T chunk)
  const int NPad1 = (n1p + 15) / 16 * 16;
  double2* u1s = ts + kMmaMC * Kp;                     // [NPad1][KA] A operand of T: all of U1, staged once
  const double2* u3 = forms + cd.off_u3;  // n3p x r3 col-major
  // Z staging block zeroed (pads included) and the barrier before any cp.async: the r1 x r3 block
  // is written by load_z's cp.async of OTHER threads, unordered with a generic store otherwise
  for (int e = threadIdx.x; e < KA * kZS; e += blockDim.x) zs[e] = make_double2(0.0, 0.0);
  __syncthreads();
  for (int e = threadIdx.x; e < NPad * Kp; e += blockDim.x) {
    const int n = e / Kp, k = e - n * Kp;
    if (n < n3p && k < r3) cp_async16(us + e, u3 + n + static_cast<int64_t>(n3p) * k);
    else us[e] = make_double2(0.0, 0.0);
  }
  const double2* u1 = forms + cd.off_u1;  // n1p x r1
  for (int e = threadIdx.x; e < NPad1 * KA; e += blockDim.x) {
    const int a = e / NPad1, i = e - a * NPad1;  // i fastest: coalesced column reads
    if (a < KA) {
      if (i < n1p && a < r1) cp_async16(u1s + i * KA + a, u1 + i + static_cast<int64_t>(n1p) * a);
      else u1s[i * KA + a] = make_double2(0.0, 0.0);
    }
  }
  auto load_z = [&](int p2o) {
    const double2* zsrc = Z + cd.off_z + static_cast<int64_t>(p2o) * r1 * r3;
    for (int e = threadIdx.x; e < r1 * r3; e += blockDim.x) {
      const int a = e / r3, gcol = e - a * r3;
      cp_async16(zs + a * kZS + gcol, zsrc + e);
    }
  };
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int fr = lane >> 2, fk = lane & 3;  // fragment row / k (A), col / k (B)
  const int E = geo.n3 / 2 + 1;
  const int nct = NPad / 16;
  const int p2end = min(p2hi, p2lo + (static_cast<int>(blockIdx.y) + 1) * kMmaPP);
  const int p2beg = p2lo + blockIdx.y * kMmaPP;
  if (p2beg < p2end) load_z(p2beg);
  for (int p2o = p2beg; p2o < p2end; ++p2o) {
    cp_async_wait_all_d();  // U3, U1 (first p2o) and this p2o's Z landed
    __syncthreads();
    const int m0beg = p1lo / 16 * 16;  // chunks start on a 16-row tile (rows < p1lo are not stored)
    for (int m0 = m0beg; m0 < p1hi; m0 += kMmaMC) {
      if (m0 > m0beg) __syncthreads();  // previous chunk's GEMM done with ts
      if (warp < kTWarps) {
        // T chunk = U1 rows x Z on the tensor cores: one 16 x 16 tile per warp
        // (kMmaMC / 16 row tiles x 2 column tiles of the <= 32 Z columns), 3M product
        const int rt = warp >> 1, ct = warp & 1;
        const bool tile_ok = m0 + rt * 16 < NPad1;  // rows past U1's padded end are never used
        double p1[2][2][2] = {}, p2[2][2][2] = {}, p3[2][2][2] = {};
        const double2* ta = u1s + (m0 + rt * 16 + fr) * KA + fk;
        const double2* zb = zs + fk * kZS + ct * 16 + fr;
        for (int k0 = 0; tile_ok && k0 < KA; k0 += 4) {
          const double2 av[2] = {ta[k0], ta[8 * KA + k0]};
          const double2 bv[2] = {zb[k0 * kZS], zb[k0 * kZS + 8]};
          const double as[2] = {av[0].x + av[0].y, av[1].x + av[1].y};
          const double bs[2] = {bv[0].x + bv[0].y, bv[1].x + bv[1].y};
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) dmma(p1[i][j][0], p1[i][j][1], av[i].x, bv[j].x);
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) dmma(p2[i][j][0], p2[i][j][1], av[i].y, bv[j].y);
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) dmma(p3[i][j][0], p3[i][j][1], as[i], bs[j]);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int row = rt * 16 + i * 8 + fr;
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int col = ct * 16 + j * 8 + 2 * fk + h;
              if (col < Kp)
                ts[row * Kp + col] = make_double2(p1[i][j][h] - p2[i][j][h], p3[i][j][h] - p1[i][j][h] - p2[i][j][h]);
            }
        }
      }
      __syncthreads();
      if (m0 + kMmaMC >= p1hi && p2o + 1 < p2end) load_z(p2o + 1);  // zs free: lands during the GEMM
      const int nrt = (min(kMmaMC, p1hi - m0) + 15) / 16;
      for (int t = warp; t < nrt * nct; t += nwarp) {
        const int rt = t / nct, ct = t - rt * nct;
        // 3-multiplication complex product (Gauss): P1 = Ar Br, P2 = Ai Bi,
        // P3 = (Ar + Ai)(Br + Bi); re = P1 - P2, im = P3 - P1 - P2 -> 3 DMMAs per step
        double p1[2][2][2], p2[2][2][2], p3[2][2][2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) p1[i][j][0] = p1[i][j][1] = p2[i][j][0] = p2[i][j][1] = p3[i][j][0] = p3[i][j][1] = 0.0;
        const double2* ta = ts + (rt * 16 + fr) * Kp + fk;
        const double2* ub = us + (ct * 16 + fr) * Kp + fk;
        for (int k0 = 0; k0 < Kp; k0 += 4) {
          const double2 av[2] = {ta[k0], ta[8 * Kp + k0]};
          const double2 bv[2] = {ub[k0], ub[8 * Kp + k0]};
          const double as[2] = {av[0].x + av[0].y, av[1].x + av[1].y};
          const double bs[2] = {bv[0].x + bv[0].y, bv[1].x + bv[1].y};
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) dmma(p1[i][j][0], p1[i][j][1], av[i].x, bv[j].x);
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) dmma(p2[i][j][0], p2[i][j][1], av[i].y, bv[j].y);
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) dmma(p3[i][j][0], p3[i][j][1], as[i], bs[j]);
        }
        double accr[2][2][2], acci[2][2][2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              accr[i][j][h] = p1[i][j][h] - p2[i][j][h];
              acci[i][j][h] = p3[i][j][h] - p1[i][j][h] - p2[i][j][h];
            }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int row = m0 + rt * 16 + i * 8 + fr;
          if (row >= p1hi || row < p1lo) continue;
          double2* dst = Shat + ((static_cast<int64_t>(p2o) * n1p + row) * NC + c) * n3p;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            // columns f = 2 hb + h: even f (h = 0) at hb, odd f at E + hb (branch-major)
            const int hb = ct * 8 + j * 4 + fk;
            if (2 * hb < n3p) dst[hb] = make_double2(accr[i][j][0], acci[i][j][0]);
            if (2 * hb + 1 < n3p) dst[E + hb] = make_double2(accr[i][j][1], acci[i][j][1]);
          }
        }
      }
    }
  }
}

// Image of U3_c for the tile GEMM: img[b][i][k] = U3_c(2 i + b, k) for i < nb3(b), k < r3, else 0
// (NP3 x Kp per parity, the exact shared-memory layout of the B operand).
__global__ void k_u3_image(const double2* __restrict__ u3, int n3, int r3, double2* __restrict__ img) {
  const int Kp = dtile::kpad(r3), NP3 = (dtile::nb3(n3, 0) + 15) / 16 * 16, n3p = n3 + 1;
  const int total = 2 * NP3 * Kp;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int b = e / (NP3 * Kp), r = e - b * NP3 * Kp, i = r / Kp, k = r - i * Kp;
    img[e] = (i < dtile::nb3(n3, b) && k < r3) ? u3[(2 * i + b) + static_cast<int64_t>(n3p) * k] : make_double2(0.0, 0.0);
  }
}

// Tile decomposition as its own launch (the tile code of the fused kernel, decomp_tile.cuh):
// CTA = (64-row p1o block, parity b) x p2o row, 256 threads, two CTAs per SM.
__global__ void __launch_bounds__(256, 2) k_decomp_tile(const double2* __restrict__ forms,
                                                        const double2* __restrict__ u3img,
                                                        const CompDev* __restrict__ comps,
                                                        const double2* __restrict__ Z, double2* __restrict__ Shat,
                                                        Geom geo, int NC, int p2lo, int p1lo, int p1hi) {
  extern __shared__ double2 sm[];
  const int b = static_cast<int>(blockIdx.x & 1);
  const int lo = p1lo + static_cast<int>(blockIdx.x >> 1) * dtile::kBM;
  const int hi = min(p1hi, lo + dtile::kBM);
  const int p2o = p2lo + static_cast<int>(blockIdx.y);
  const int64_t rs = static_cast<int64_t>(NC) * (geo.n3 + 1);
  double2* out = Shat + (static_cast<int64_t>(p2o) * (geo.n1 + 1) + lo) * rs;
  dtile::run<256>(forms, u3img, comps, Z, 0, NC, 1, geo.n1, geo.n3, p2o, lo, hi, b, b + 1, out, rs, sm);
}

// Factor transform: out[p + (n+1) c] = sum_m e_c[m] w_{2n}^{p m}, p <= n,
// with e_c the parity embedding of column c (embed_column).
__global__ void k_factor_transform(const double2* __restrict__ u, int n, int r, int sign,
                                   const double2* __restrict__ tw, double2* __restrict__ out) {
  const int m = 2 * n;
  const int total = (n + 1) * r;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int p = e % (n + 1), c = e / (n + 1);
    const double2* col = u + static_cast<int64_t>(n) * c;
    double2 acc = make_double2(0.0, 0.0);
    for (int k = 0; k < m; ++k) {
      if (k == n) continue;
      const double2 v = k < n ? col[k] : cscale(col[m - k], static_cast<double>(sign));
      const int e2 = static_cast<int>((static_cast<int64_t>(p) * k) % m);
      cfma(acc, v, tw[e2]);
    }
    out[p + static_cast<int64_t>(n + 1) * c] = acc;
  }
}

}  // namespace

size_t decomp_mma_smem(int n1, int n3, int rmax) {
  if (rmax > 28) return static_cast<size_t>(-1);  // T tiles cover <= 32 columns, Kp <= 28 (else the FMA kernel)
  const int kp = mma_kp(rmax);
  const size_t npad = static_cast<size_t>((n3 + 1 + 15) / 16 * 16);
  const size_t npad1 = static_cast<size_t>((n1 + 1 + 15) / 16 * 16);
  return sizeof(double2) * (npad * kp + static_cast<size_t>(kp) * kZS + static_cast<size_t>(kMmaMC) * kp +
                            npad1 * kp);
}

size_t decomp_smem(int n3, int rmax) {
  return sizeof(double2) * (static_cast<size_t>(rmax) * rmax + static_cast<size_t>(rmax) * (n3 + 1) +
                            static_cast<size_t>(rmax) * kTP1);
}

void launch_decomp_z(const double2* forms, const CompDev* comps_dev, double2* Z, const Geom& g, int rmax,
                     cudaStream_t st) {
  k_decomp_z<<<dim3(g.NC, rmax), kThreads, 0, st>>>(forms, comps_dev, Z, g.n2);
  VIE_CUDA_CHECK(cudaGetLastError());
}

int64_t u3_image_elems(int n3, int r3) {
  return 2 * static_cast<int64_t>((dtile::nb3(n3, 0) + 15) / 16 * 16) * dtile::kpad(r3);
}

void launch_u3_image(const double2* forms, const CompDev* comps_host, int NC, int n3, double2* img, cudaStream_t st) {
  for (int c = 0; c < NC; ++c) {
    const CompDev& cd = comps_host[c];
    if (!cd.active) continue;
    k_u3_image<<<64, 256, 0, st>>>(forms + cd.off_u3, n3, cd.r3, img + cd.off_u3i);
    VIE_CUDA_CHECK(cudaGetLastError());
  }
}

void launch_decomp(const double2* forms, const CompDev* comps_dev, const CompDev* comps_host, double2* Z,
                   double2* Shat, const Geom& g, int rmax, cudaStream_t st, int p2lo, int p2hi, bool with_z, int p1lo,
                   int p1hi, const double2* u3img) {
  (void)comps_host;
  if (p2hi < 0) p2hi = g.n2 + 1;
  if (p1hi < 0) p1hi = g.n1 + 1;
  if (p2hi <= p2lo || p1hi <= p1lo) return;
  if (with_z) {
    k_decomp_z<<<dim3(g.NC, rmax), kThreads, 0, st>>>(forms, comps_dev, Z, g.n2);
    VIE_CUDA_CHECK(cudaGetLastError());
  }
  const size_t sms = decomp_mma_smem(g.n1, g.n3, rmax);
  static const bool tile = std::getenv("VIE_DECOMP_TILE") && std::atoi(std::getenv("VIE_DECOMP_TILE")) != 0;
  const size_t smt = dtile::smem_bytes(g.n3, rmax);
  if (tile && u3img && smt <= kMaxSmem) {
    VIE_CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_decomp_tile),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smt)));
    const int nblk = (p1hi - p1lo + dtile::kBM - 1) / dtile::kBM;
    k_decomp_tile<<<dim3(2 * nblk, p2hi - p2lo), 256, smt, st>>>(forms, u3img, comps_dev, Z, Shat, g, g.NC, p2lo,
                                                                   p1lo, p1hi);
  } else if (sms <= kMaxSmem) {
    VIE_CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_decomp_s_mma),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sms)));
    k_decomp_s_mma<<<dim3(g.NC, (p2hi - p2lo + kMmaPP - 1) / kMmaPP), kMmaThreads, sms, st>>>(
        forms, comps_dev, Z, Shat, g, g.NC, p2lo, p2hi, p1lo, p1hi);
  } else if (decomp_smem(g.n3, rmax) <= kMaxSmem) {
    const size_t smf = decomp_smem(g.n3, rmax);
    VIE_CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_decomp_s),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smf)));
    k_decomp_s<<<dim3(g.NC, p2hi - p2lo), kThreads, smf, st>>>(forms, comps_dev, Z, Shat, g, g.NC, p2lo, p1lo, p1hi);
  } else {
    const size_t smb = sizeof(double2) * static_cast<size_t>(rmax) * kTP1;
    VIE_CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_decomp_s_big),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smb)));
    k_decomp_s_big<<<dim3(g.NC, p2hi - p2lo), kThreads, smb, st>>>(forms, comps_dev, Z, Shat, g, g.NC, p2lo, p1lo,
                                                                     p1hi);
  }
  VIE_CUDA_CHECK(cudaGetLastError());
}

void launch_factor_transform(const double2* u, int n, int r, int sign, const double2* tw2n, double2* out,
                             cudaStream_t st) {
  const int total = (n + 1) * r;
  const int blocks = (total + 255) / 256;
  k_factor_transform<<<blocks, 256, 0, st>>>(u, n, r, sign, tw2n, out);
  VIE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace vie
