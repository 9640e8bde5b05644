// kernels_pencil.cu -- fused axis-3 FFT + Tucker-spectrum Hadamard + IFFT.
//
// One CTA owns W consecutive mirror-paired axis-1 positions of one axis-2
// position, for all S source currents, along the whole axis 3:
//   load x^ pencils (n3 values; the pad to m3 is never materialised)
//   -> in-smem DIF FFT along axis 3 (digit-reversed slots)
//   -> per spectral point: y^_t = sum_blocks coef * sign * S^_c(octant) * x^_s
//      (apply_operator's component loop + mac_elementwise, operator.hpp:303-364,
//       fused over all components; x^ read once, y^ written once)
//   -> adjoint IFFT along axis 3, crop to n3, store in place.
// The decompressed spectrum S^_c is read at its octant representative
// (|p| <= n per axis) and mirrored with the component parity: with U_q(m-p) =
// sign_q U_q(p) (embed_column, operator.hpp:64-70) every component satisfies
// S^(m1-p1, p2, p3) = sign_1 S^(p1, p2, p3) and likewise per axis.
#include <utility>

#include "fft.cuh"
#include "kernels.cuh"

namespace vie {

namespace {

__host__ __device__ __forceinline__ int line_stride(int n) { return n + 1; }

template <int KIND, int BASIS>
struct Tab {
  static constexpr Table<KIND, BASIS> value = make_table<KIND, BASIS>();
};

// Block B of the table, all indices compile-time constants.
template <int KIND, int BASIS, int B, int S>
__device__ __forceinline__ void had_block(double2 (&yh)[S], const double2 (&xh)[S], double2& sh,
                                          const double2* sh_base, int64_t cstride, uint64_t active, int m1flag,
                                          int m2flag, int mir) {
  constexpr BlockT blk = Tab<KIND, BASIS>::value.blocks[B];
  constexpr bool first = (B == 0) || (Tab<KIND, BASIS>::value.blocks[B == 0 ? 0 : B - 1].c != blk.c);
  constexpr CompT cp = Tab<KIND, BASIS>::value.comps[blk.c];
  if (!((active >> blk.c) & 1ull)) return;
  if (first) {
    sh = __ldg(sh_base + static_cast<int64_t>(blk.c) * cstride);
    const int flip = (cp.p0 < 0 ? m1flag : 0) ^ (cp.p1 < 0 ? m2flag : 0) ^ (cp.p2 < 0 ? mir : 0);
    if (flip) sh = make_double2(-sh.x, -sh.y);
  }
  if (blk.coef > 0) cfma(yh[blk.t], sh, xh[blk.s]);
  else cfms(yh[blk.t], sh, xh[blk.s]);
}

template <int KIND, int BASIS, int S, int... Bs>
__device__ __forceinline__ void had_all(std::integer_sequence<int, Bs...>, double2 (&yh)[S], const double2 (&xh)[S],
                                        const double2* sh_base, int64_t cstride, uint64_t active, int m1flag,
                                        int m2flag, int mir) {
  double2 sh = make_double2(0.0, 0.0);
  (had_block<KIND, BASIS, Bs, S>(yh, xh, sh, sh_base, cstride, active, m1flag, m2flag, mir), ...);
}

template <int KIND, int BASIS>
__global__ void __launch_bounds__(kThreads) k_pencil(double2* __restrict__ B, const double2* __restrict__ Shat,
                                                     Geom g, FftPlan P, int W, uint64_t active) {
  constexpr int S = TableDims<KIND, BASIS>::S;
  constexpr int NB = TableDims<KIND, BASIS>::NB;
  constexpr int NC = TableDims<KIND, BASIS>::NC;
  extern __shared__ double2 sm[];
  const int m3 = P.n;
  const SmemPlan SP = load_plan(sm, P);
  double2* buf = sm + plan_smem_elems(m3);
  const int ls = line_stride(m3);
  const int n1 = g.n1, n2 = g.n2, n3 = g.n3, m1 = g.m1, m2 = g.m2;
  const int pos2 = blockIdx.y;
  const int c0 = blockIdx.x * W;
  const int wc = min(W, m1 - c0);
  const int64_t kstride = static_cast<int64_t>(m2) * m1;  // between consecutive k
  const int64_t sstride = kstride * n3;                   // between current components
  double2* col = B + static_cast<int64_t>(pos2) * m1 + c0;

  // ---- load the S * wc pencils (k < n3)
  for (int e = threadIdx.x; e < S * n3 * W; e += blockDim.x) {
    const int w = e % W;
    const int sk = e / W;
    const int s = sk / n3, k = sk - s * n3;
    if (w < wc) buf[(s * W + w) * ls + k] = col[s * sstride + k * kstride + w];
  }
  __syncthreads();
  fft_forward(buf, S * W, ls, SP, true);

  // ---- Hadamard with the octant-mirrored decompressed spectrum
  const int f2 = freq_of_pos(pos2, n2);
  const int m2flag = f2 > n2;
  const int p2o = m2flag ? m2 - f2 : f2;
  const int n3p = n3 + 1;
  const int items = wc * 2 * n3p;
  for (int u = threadIdx.x; u < items; u += blockDim.x) {
    const int w = u % wc;
    const int rest = u / wc;
    const int mir = rest & 1;
    const int f3o = rest >> 1;
    if (mir && (f3o == 0 || f3o == n3)) continue;  // self-mirror frequency
    const int f1 = freq_of_pos(c0 + w, n1);
    const int m1flag = f1 > n1;
    const int p1o = m1flag ? m1 - f1 : f1;
    const int f3 = mir ? m3 - f3o : f3o;
    const int slot = SP.slot[f3];
    double2 xh[S], yh[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
      xh[s] = buf[(s * W + w) * ls + slot];
      yh[s] = make_double2(0.0, 0.0);
    }
    const double2* sh_base = Shat + ((static_cast<int64_t>(p2o) * (n1 + 1) + p1o) * NC) * n3p + f3o;
    had_all<KIND, BASIS, S>(std::make_integer_sequence<int, NB>{}, yh, xh, sh_base, n3p, active, m1flag, m2flag,
                            mir);
#pragma unroll
    for (int s = 0; s < S; ++s) buf[(s * W + w) * ls + slot] = yh[s];
  }
  __syncthreads();
  fft_inverse(buf, S * W, ls, SP, true);

  // ---- store the cropped y^ pencils in place
  for (int e = threadIdx.x; e < S * n3 * W; e += blockDim.x) {
    const int w = e % W;
    const int sk = e / W;
    const int s = sk / n3, k = sk - s * n3;
    if (w < wc) col[s * sstride + k * kstride + w] = buf[(s * W + w) * ls + k];
  }
}

int pencil_width(int S) {
  int W = kPencilLines / S;
  if (W < 2) W = 2;
  return W & ~1;  // keep mirror pairs (positions 2q, 2q+1) together
}

template <int KIND, int BASIS>
void launch_pencil_t(double2* B, const double2* Shat, const Geom& g, const FftPlan& P3, uint64_t active,
                     cudaStream_t st) {
  constexpr int S = TableDims<KIND, BASIS>::S;
  const int W = pencil_width(S);
  const size_t sm = pencil_smem(g.m3, S);
  auto fn = k_pencil<KIND, BASIS>;
  VIE_CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
  dim3 grid((g.m1 + W - 1) / W, g.m2);
  fn<<<grid, kThreads, sm, st>>>(B, Shat, g, P3, W, active);
  VIE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace

size_t pencil_smem(int m3, int S) {
  const int W = pencil_width(S);
  return sizeof(double2) * (static_cast<size_t>(plan_smem_elems(m3)) + static_cast<size_t>(S) * W * line_stride(m3));
}

void launch_pencil(int kind, int basis, double2* B, const double2* Shat, const Geom& g, const FftPlan& P3,
                   uint64_t active, cudaStream_t st) {
  if (kind == 0 && basis == 0) launch_pencil_t<0, 0>(B, Shat, g, P3, active, st);
  else if (kind == 1 && basis == 0) launch_pencil_t<1, 0>(B, Shat, g, P3, active, st);
  else if (kind == 0 && basis == 1) launch_pencil_t<0, 1>(B, Shat, g, P3, active, st);
  else launch_pencil_t<1, 1>(B, Shat, g, P3, active, st);
}

}  // namespace vie
