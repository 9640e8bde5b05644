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
#include <utility>

#include "fft.cuh"
#include "kernels.cuh"

namespace vie {

namespace {

__host__ __device__ __forceinline__ int line_stride(int n) { return n + 1; }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

template <int KIND, int BASIS>
struct Tab {
  static constexpr Table<KIND, BASIS> value = make_table<KIND, BASIS>();
};

// First block of component c (of block B) whose target lies in this half.
template <int KIND, int BASIS>
constexpr bool first_in_half(int B, int TH, int HALF) {
  const auto& tb = Tab<KIND, BASIS>::value;
  const int c = tb.blocks[B].c;
  for (int b = B - 1; b >= 0 && tb.blocks[b].c == c; --b)
    if (tb.blocks[b].t / TH == HALF) return false;
  return true;
}

// Block B of the table, all indices compile-time constants; only blocks whose
// target is in [HALF*TH, HALF*TH + TH) (target split across two threads).
template <int KIND, int BASIS, int B, int S, int TH, int HALF>
__device__ __forceinline__ void had_block(double2 (&yh)[TH], const double2 (&xh)[S], double2& sh,
                                          const double2* sh_base, int cstride, uint64_t active, int m1flag,
                                          int m2flag, int mir) {
  constexpr BlockT blk = Tab<KIND, BASIS>::value.blocks[B];
  if constexpr (blk.t / TH == HALF) {
    constexpr bool first = first_in_half<KIND, BASIS>(B, TH, HALF);
    constexpr CompT cp = Tab<KIND, BASIS>::value.comps[blk.c];
    if (!((active >> blk.c) & 1ull)) return;
    if (first) {
      sh = sh_base[blk.c * cstride];
      const int flip = (cp.p0 < 0 ? m1flag : 0) ^ (cp.p1 < 0 ? m2flag : 0) ^ (cp.p2 < 0 ? mir : 0);
      if (flip) sh = make_double2(-sh.x, -sh.y);
    }
    if (blk.coef > 0) cfma(yh[blk.t - HALF * TH], sh, xh[blk.s]);
    else cfms(yh[blk.t - HALF * TH], sh, xh[blk.s]);
  }
}

template <int KIND, int BASIS, int S, int TH, int HALF, int... Bs>
__device__ __forceinline__ void had_all(std::integer_sequence<int, Bs...>, double2 (&yh)[TH], const double2 (&xh)[S],
                                        const double2* sh_base, int cstride, uint64_t active, int m1flag, int m2flag,
                                        int mir) {
  double2 sh = make_double2(0.0, 0.0);
  (had_block<KIND, BASIS, Bs, S, TH, HALF>(yh, xh, sh, sh_base, cstride, active, m1flag, m2flag, mir), ...);
}

struct PencilArgs {
  const double2* Bin;
  double2* Bout;
  const double2* Shat;
  const double2* twm3;  // w_m3^e, e < m3 (full-length plan table)
  Geom g;
  FftPlan PH;           // n3-point plan (branch transforms)
  int P1P;              // axis-1 mirror pairs per CTA
  int CF;               // octant frequencies per spectrum chunk
  uint64_t active;
};

constexpr int kPencilThreads = 512;  // 16 warps: the CTA owns the SM (smem), so it must hide latency itself

template <int KIND, int BASIS>
__global__ void __launch_bounds__(kPencilThreads, 1) k_pencil(PencilArgs a) {
  constexpr int S = TableDims<KIND, BASIS>::S;
  constexpr int NB = TableDims<KIND, BASIS>::NB;
  constexpr int NC = TableDims<KIND, BASIS>::NC;
  constexpr int TS = S >= 12 ? 2 : 1;  // target split: 2 threads per spectral point (register budget)
  constexpr int TH = S / TS;
  extern __shared__ double2 sm[];
  const Geom& g = a.g;
  const int n1 = g.n1, n2 = g.n2, n3 = g.n3, m1 = g.m1, m2 = g.m2, m3 = g.m3;
  const int P1P = a.P1P, CF = a.CF;
  const int NP = 4 * P1P;  // pencils: [p2sel][w], w < 2*P1P
  const int W = 2 * P1P;
  const int ls = line_stride(n3);
  const SmemPlan SP = load_plan(sm, a.PH);
  double2* twb = sm + plan_smem_elems(n3);  // w_m3^k, k < n3
  double2* shb = twb + n3;                  // 2 x [P1P][NC][CF]
  const int chunk_elems = P1P * NC * CF;
  double2* buf = shb + 2 * chunk_elems;     // [S][NP] lines of ls
  for (int e = threadIdx.x; e < n3; e += blockDim.x) twb[e] = a.twm3[e];

  const int c0 = blockIdx.x * W;  // first axis-1 position
  const int q0 = c0 >> 1;         // tile octant row of axis 1
  const int j = blockIdx.y;       // axis-2 position pair (2j, 2j+1)
  const int f2t = freq_of_pos(2 * j, n2);
  const int p2o_tile = f2t > n2 ? m2 - f2t : f2t;
  const int n3p = n3 + 1;
  const int E = n3 / 2 + 1;            // even octant frequencies 0,2,..
  const int O = (n3 + 1) / 2;          // odd octant frequencies 1,3,..
  const int64_t kstride = static_cast<int64_t>(m2) * m1;
  const int64_t sstride = kstride * n3;

  for (int b = 0; b < 2; ++b) {
    // ---- prefetch spectrum chunk 0 of this branch (lands during the FFT)
    const int nbo = b ? O : E;
    const int nchunks = (nbo + CF - 1) / CF;
    auto issue_chunk = [&](int ci) {
      double2* dst = shb + (ci & 1) * chunk_elems;
      const int u0 = ci * CF;
      for (int e = threadIdx.x; e < chunk_elems; e += blockDim.x) {
        const int ul = e % CF;
        const int rc = e / CF;
        const int c = rc % NC, tr = rc / NC;
        const int p1o = q0 + tr;
        if (p1o <= n1 && u0 + ul < nbo)
          cp_async16(dst + e, a.Shat + ((static_cast<int64_t>(p2o_tile) * (n1 + 1) + p1o) * NC + c) * n3p +
                                  b * E + u0 + ul);
      }
      cp_async_commit();
    };
    issue_chunk(0);

    // ---- load the pencils (k < n3) with cp.async (no register staging)
    for (int e = threadIdx.x; e < S * n3 * NP; e += blockDim.x) {
      const int w = e % W;
      const int r = e / W;
      const int p2sel = r & 1;
      const int sk = r >> 1;
      const int s = sk / n3, k = sk - s * n3;
      const int pos1 = c0 + w, pos2 = 2 * j + p2sel;
      double2* dst = buf + (s * NP + p2sel * W + w) * ls + k;
      if (pos1 < m1) cp_async16(dst, a.Bin + s * sstride + k * kstride + static_cast<int64_t>(pos2) * m1 + pos1);
      else *dst = make_double2(0.0, 0.0);
    }
    cp_async_commit();
    cp_async_wait_all();  // also lands spectrum chunk 0 (committed earlier)
    __syncthreads();
    if (b) {  // branch twiddle w_m3^{k} (odd frequencies)
      for (int e = threadIdx.x; e < S * NP * n3; e += blockDim.x) {
        const int line = e / n3, k = e - line * n3;
        buf[line * ls + k] = cmul(buf[line * ls + k], twb[k]);
      }
    }
    __syncthreads();
    fft_forward(buf, S * NP, ls, SP, false);

    // ---- Hadamard over the branch's octant frequencies, chunk by chunk
    for (int ci = 0; ci < nchunks; ++ci) {
      cp_async_wait_all();
      __syncthreads();  // chunk ci visible; chunk ci-1 consumers done
      if (ci + 1 < nchunks) issue_chunk(ci + 1);
      const double2* shc = shb + (ci & 1) * chunk_elems;
      // work unit = (spectral point, target half); threads [0, items) take
      // half 0, [items, 2 items) half 1 (warp-uniform halves)
      const int items = CF * NP * 2;
      const int units = items * TS;
      for (int u0 = 0; u0 < units; u0 += blockDim.x) {
        const int unit = u0 + threadIdx.x;
        const int half = unit >= items ? 1 : 0;
        const int it = unit - half * items;
        // lanes: mirror pair (mir) x pencil x frequency, frequency slowest
        const int mir = it & 1;
        const int rest = it >> 1;
        const int p = rest % NP;
        const int ul = rest / NP;
        const int u = ci * CF + ul;
        const int f3o = 2 * u + b;
        const int w = p % W, p2sel = p / W;
        const int pos1 = c0 + w;
        const bool valid = unit < units && u < nbo && !(mir && (f3o == 0 || f3o == n3)) && pos1 < m1;
        double2 xh[S];
        double2* pl = buf;
        int m1flag = 0, m2flag = 0, p1o = 0, p2o = 0;
        if (valid) {
          const int f1 = freq_of_pos(pos1, n1);
          m1flag = f1 > n1;
          p1o = m1flag ? m1 - f1 : f1;
          const int f2 = freq_of_pos(2 * j + p2sel, n2);
          m2flag = f2 > n2;
          p2o = m2flag ? m2 - f2 : f2;
          const int f3 = mir ? m3 - f3o : f3o;
          pl = buf + p * ls + SP.slot[(f3 - b) >> 1];
#pragma unroll
          for (int s = 0; s < S; ++s) xh[s] = pl[s * NP * ls];
        }
        if (TS > 1) __syncthreads();  // both halves read x^ before either overwrites it
        if (valid) {
          const double2* sh_base;
          int cstride;
          const int tr = p1o - q0;
          if (p2o == p2o_tile && tr >= 0 && tr < P1P) {
            sh_base = shc + (tr * NC) * CF + ul;
            cstride = CF;
          } else {  // boundary pencils (frequencies 0 / n of a pair) outside the tile
            sh_base = a.Shat + ((static_cast<int64_t>(p2o) * (n1 + 1) + p1o) * NC) * n3p + b * E + u;
            cstride = n3p;
          }
          double2 yh[TH];
#pragma unroll
          for (int t = 0; t < TH; ++t) yh[t] = make_double2(0.0, 0.0);
          if (half == 0) {
            had_all<KIND, BASIS, S, TH, 0>(std::make_integer_sequence<int, NB>{}, yh, xh, sh_base, cstride, a.active,
                                           m1flag, m2flag, mir);
          } else if constexpr (TS > 1) {
            had_all<KIND, BASIS, S, TH, 1>(std::make_integer_sequence<int, NB>{}, yh, xh, sh_base, cstride, a.active,
                                           m1flag, m2flag, mir);
          }
#pragma unroll
          for (int t = 0; t < TH; ++t) pl[(half * TH + t) * NP * ls] = yh[t];
        }
      }
    }
    __syncthreads();
    fft_inverse(buf, S * NP, ls, SP, false);

    // ---- store / accumulate the cropped output pencils
    for (int e = threadIdx.x; e < S * n3 * NP; e += blockDim.x) {
      const int w = e % W;
      const int r = e / W;
      const int p2sel = r & 1;
      const int sk = r >> 1;
      const int s = sk / n3, k = sk - s * n3;
      const int pos1 = c0 + w, pos2 = 2 * j + p2sel;
      if (pos1 >= m1) continue;
      double2* out = a.Bout + s * sstride + k * kstride + static_cast<int64_t>(pos2) * m1 + pos1;
      const double2 v = buf[(s * NP + p2sel * W + w) * ls + k];
      if (b == 0) *out = v;
      else *out = cadd(*out, cmulc(v, twb[k]));
    }
    __syncthreads();
  }
}

int pencil_p1pairs(int S) { return S >= 12 ? 1 : (S >= 6 ? 2 : 4); }

size_t pencil_smem_cf(int n3, int S, int NC, int CF) {
  const int P1P = pencil_p1pairs(S);
  const size_t e = static_cast<size_t>(plan_smem_elems(n3)) + n3 + 2ull * P1P * NC * CF +
                   static_cast<size_t>(S) * 4 * P1P * line_stride(n3);
  return e * sizeof(double2);
}

int pencil_cf(int n3, int S, int NC) {
  for (int cf : {32, 16, 8})
    if (pencil_smem_cf(n3, S, NC, cf) <= kMaxSmem) return cf;
  return 0;
}

template <int KIND, int BASIS>
void launch_pencil_t(const double2* Bin, double2* Bout, const double2* Shat, const Geom& g, const FftPlan& PH,
                     const double2* twm3, uint64_t active, cudaStream_t st) {
  constexpr int S = TableDims<KIND, BASIS>::S;
  constexpr int NC = TableDims<KIND, BASIS>::NC;
  PencilArgs a{Bin, Bout, Shat, twm3, g, PH, pencil_p1pairs(S), pencil_cf(g.n3, S, NC), active};
  const size_t sm = pencil_smem_cf(g.n3, S, NC, a.CF);
  auto fn = k_pencil<KIND, BASIS>;
  VIE_CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
  dim3 grid((g.n1 + a.P1P - 1) / a.P1P, g.n2);
  fn<<<grid, kPencilThreads, sm, st>>>(a);
  VIE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace

size_t pencil_smem(int n3, int S, int NC) {
  const int cf = pencil_cf(n3, S, NC);
  return cf ? pencil_smem_cf(n3, S, NC, cf) : static_cast<size_t>(-1);
}

void launch_pencil(int kind, int basis, const double2* Bin, double2* Bout, const double2* Shat, const Geom& g,
                   const FftPlan& PH, const double2* twm3, uint64_t active, cudaStream_t st) {
  if (kind == 0 && basis == 0) launch_pencil_t<0, 0>(Bin, Bout, Shat, g, PH, twm3, active, st);
  else if (kind == 1 && basis == 0) launch_pencil_t<1, 0>(Bin, Bout, Shat, g, PH, twm3, active, st);
  else if (kind == 0 && basis == 1) launch_pencil_t<0, 1>(Bin, Bout, Shat, g, PH, twm3, active, st);
  else launch_pencil_t<1, 1>(Bin, Bout, Shat, g, PH, twm3, active, st);
}

}  // namespace vie
