// decomp_tile.cuh -- Tucker decompression of one spectrum TILE on the FP64 tensor cores:
// S^_c(p1o in [p1lo, p1hi), p2o, f3o of parity b) for every active component c, written
// branch-major (f3o = 2 i + b at column (b ? E : 0) + i).  A tile is what the fused
// decompress x pencil kernel (kernels_fused.cu) hands to the pencil clusters of one axis-2
// octant row: it lives in an L2-resident ring and is never a whole-spectrum buffer.
//
// Per component (reference: decompress_tucker, operator.hpp:224-244, restricted to the
// octant as in kernels_decomp.cu):  T = U1[p1 rows] Z_c[p2o]  (Z = core x2 U2, k_decomp_z),
// then S^ = T U3_c[parity-b rows]^T, both as complex GEMMs on mma.sync.m8n8k4.f64 with the
// 3-multiplication (Gauss) product.  U3's parity-b rows and Z_c[p2o] are staged in shared
// memory per component; U1 fragments come straight from global (L1/L2: 64 x r rows).
#pragma once
#include "kernels.cuh"
#include "tma.cuh"

namespace vie {
namespace dtile {

#ifndef VIE_TILE_BM
#define VIE_TILE_BM 32
#endif
constexpr int kBM = VIE_TILE_BM;  // p1o rows per tile
constexpr int kZS = 34;   // Z row stride (== 2 mod 8: conflict-free B fragments over k)

__host__ __device__ __forceinline__ int kpad(int r) {  // padded inner dimension (== 4 mod 8)
  int kp = (r + 3) / 4 * 4;
  if (kp % 8 == 0) kp += 4;
  return kp;
}
// parity-b row count of the octant axis 3 (n3 + 1 frequencies): E = n3/2 + 1 even, O = (n3+1)/2 odd
__host__ __device__ __forceinline__ int nb3(int n3, int b) { return b ? (n3 + 1) / 2 : n3 / 2 + 1; }

// shared memory of one tile CTA (bytes) for ranks <= rmax; (size_t)-1 beyond the T tiles (32 cols)
inline size_t smem_bytes(int n3, int rmax) {
  if (rmax > 28) return static_cast<size_t>(-1);
  const size_t kp = static_cast<size_t>(kpad(rmax));
  const size_t np3 = static_cast<size_t>((nb3(n3, 0) + 15) / 16 * 16);
  return sizeof(double2) * (np3 * kp + kp * kZS + static_cast<size_t>(kBM) * kp);
}

__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_wait_all() {
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void mma_f64(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// One tile on a CTA of NT threads (NT / 32 >= 8 warps): components c0, c0 + cstep, .. < c1,
// axis-3 parities [b0, b1) (T is formed once per component and serves both parities).
// P2ROWS = false: rows are p1o in [lo, hi) at p2o = fixed (T = U1 rows x Z_c[p2o], DMMA);
// P2ROWS = true:  rows are p2o in [lo, hi) at p1o = fixed (the axis-1 edge rows p1o = 0, n1:
//                 T[p2o] = U1_c(p1o, :) Z_c[p2o], FMA).
// out + (row - lo) * rs is the branch-major spectrum row (c * (n3 + 1) + column) of the row.
// KEEP_L2: stores with an L2 evict_last policy (the fused kernel's tile ring).
template <int NT, bool P2ROWS = false, bool KEEP_L2 = false>
__device__ __forceinline__ void run(const double2* __restrict__ forms, const double2* __restrict__ u3img,
                                    const CompDev* __restrict__ comps, const double2* __restrict__ Z, int c0,
                                    int c1, int cstep, int n1, int n3, int fixed, int lo, int hi, int b0, int b1,
                                    double2* __restrict__ out, int64_t rs, double2* sm) {
  static_assert(NT / 32 >= 2 * kBM / 16, "one 16 x 16 T tile per warp");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  const int n1p = n1 + 1, n3p = n3 + 1;
  const int E = nb3(n3, 0);
  const int NP3 = (E + 15) / 16 * 16;  // both branches use the even branch's padding
  const int p2o = fixed, p1lo = lo, p1hi = hi;
  const uint64_t pol = KEEP_L2 ? l2_evict_last() : 0ull;
  for (int c = c0; c < c1; c += cstep) {
    const CompDev cd = comps[c];
    if (!cd.active) continue;
    const int r1 = cd.r1, r3 = cd.r3;
    const int Kp = kpad(r3), KA = kpad(r1);
    double2* us = sm;                                   // [NP3][Kp]  U3 parity-b rows (B operand)
    double2* zs = us + static_cast<int64_t>(NP3) * Kp;  // [KA][kZS]  Z_c[p2o] (B operand of T)
    double2* ts = zs + KA * kZS;                        // [kBM][Kp]  T (A operand)
    // U3 parity-b rows, zero padded: a contiguous copy of the operator's image (k_u3_image)
    auto stage_u3 = [&](int b) {
      const double2* u3 = u3img + cd.off_u3i + static_cast<int64_t>(b) * NP3 * Kp;
      for (int e = tid; e < NP3 * Kp; e += NT) cp16(us + e, u3 + e);
    };
    __syncthreads();  // the previous component's GEMMs are done with us / zs / ts
    stage_u3(b0);
    if constexpr (!P2ROWS) {
      const double2* zsrc = Z + cd.off_z + static_cast<int64_t>(p2o) * r1 * r3;  // [a][g]
      for (int e = tid; e < KA * kZS; e += NT) {
        const int a = e / kZS, g = e - a * kZS;
        if (a < r1 && g < r3) cp16(zs + e, zsrc + a * r3 + g);
        else zs[e] = make_double2(0.0, 0.0);
      }
    } else {
      // T[r][g] = sum_a U1_c(p1o, a) Z_c[lo + r](a, g)  (64 x r3 outputs, r1 MACs each)
      const double2* u1 = forms + cd.off_u1 + fixed;  // U1_c(p1o, a) at u1[n1p * a]
      for (int e = tid; e < kBM * Kp; e += NT) {
        const int r = e / Kp, g = e - r * Kp;
        double2 acc = make_double2(0.0, 0.0);
        if (lo + r < hi && g < r3) {
          const double2* zr = Z + cd.off_z + static_cast<int64_t>(lo + r) * r1 * r3 + g;
          for (int a = 0; a < r1; ++a) cfma(acc, __ldg(u1 + static_cast<int64_t>(n1p) * a), __ldg(zr + a * r3));
        }
        ts[e] = acc;
      }
    }
    cp_wait_all();
    __syncthreads();
    // T = U1 rows x Z: one 16 x 16 tile per warp (kBM / 16 row tiles x 2 column tiles)
    if (!P2ROWS && warp < 2 * kBM / 16) {
      const int rt = warp >> 1, ct = warp & 1;
      const double2* u1 = forms + cd.off_u1;  // n1p x r1 col-major
      double p1[2][2][2] = {}, p2[2][2][2] = {}, p3[2][2][2] = {};
      const int row0 = p1lo + rt * 16 + fr;
      const double2* zb = zs + fk * kZS + ct * 16 + fr;
      // all U1 fragments of the tile row block issued up front (<= 7 k-steps: KA <= 28), so the
      // L2 latency is paid once, not once per k-step
      double2 u1f[7][2];
#pragma unroll
      for (int ks = 0; ks < 7; ++ks)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int row = row0 + 8 * i, k = 4 * ks + fk;
          u1f[ks][i] = (row < p1hi && k < r1) ? __ldg(u1 + row + static_cast<int64_t>(n1p) * k) : make_double2(0.0, 0.0);
        }
#pragma unroll
      for (int ks = 0; ks < 7; ++ks) {
        const int k0 = 4 * ks;
        if (k0 >= KA) break;
        const double2 av[2] = {u1f[ks][0], u1f[ks][1]};
        const double2 bv[2] = {zb[k0 * kZS], zb[k0 * kZS + 8]};
        const double as[2] = {av[0].x + av[0].y, av[1].x + av[1].y};
        const double bs[2] = {bv[0].x + bv[0].y, bv[1].x + bv[1].y};
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            mma_f64(p1[i][j][0], p1[i][j][1], av[i].x, bv[j].x);
            mma_f64(p2[i][j][0], p2[i][j][1], av[i].y, bv[j].y);
            mma_f64(p3[i][j][0], p3[i][j][1], as[i], bs[j]);
          }
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
    for (int b = b0; b < b1; ++b) {
      if (b > b0) {  // restage U3 for the next parity (T stays)
        __syncthreads();
        stage_u3(b);
        cp_wait_all();
        __syncthreads();
      }
      const int NB = nb3(n3, b);
      // S^ = T U3^T: 16 x 16 warp tiles over (kBM / 16) x (NP3 / 16)
      const int nrt = (min(kBM, p1hi - p1lo) + 15) / 16, nct = NP3 / 16;
      for (int t = warp; t < nrt * nct; t += NT / 32) {
        const int rt = t / nct, ct = t - rt * nct;
        double p1[2][2][2] = {}, p2[2][2][2] = {}, p3[2][2][2] = {};
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
            for (int j = 0; j < 2; ++j) mma_f64(p1[i][j][0], p1[i][j][1], av[i].x, bv[j].x);
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) mma_f64(p2[i][j][0], p2[i][j][1], av[i].y, bv[j].y);
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) mma_f64(p3[i][j][0], p3[i][j][1], as[i], bs[j]);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int prow = rt * 16 + i * 8 + fr;
          if (p1lo + prow >= p1hi) continue;
          double2* dst = out + prow * rs + static_cast<int64_t>(c) * n3p + (b ? E : 0);
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int col = ct * 16 + j * 8 + 2 * fk;
#pragma unroll
            for (int h = 0; h < 2; ++h)
              if (col + h < NB) {
                const double2 v = make_double2(p1[i][j][h] - p2[i][j][h], p3[i][j][h] - p1[i][j][h] - p2[i][j][h]);
                if (KEEP_L2) st_hint(dst + col + h, v, pol);
                else dst[col + h] = v;
              }
          }
        }
      }
    }
  }
}

}  // namespace dtile
}  // namespace vie
