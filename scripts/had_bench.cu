// Microbenchmark: the PWL Hadamard block table (kernels_pencil.cu had_all) in
// isolation, data in smem, full occupancy -> achievable FP64 rate of that code.
#include <cstdio>
#include <utility>
#include "../paper_1811_00484_b200/csrc/common.cuh"
namespace vie {
template <int KIND, int BASIS> struct Tab { static constexpr Table<KIND, BASIS> value = make_table<KIND, BASIS>(); };
template <int KIND, int BASIS>
constexpr bool first_in_half(int B, int TH, int HALF) {
  const auto& tb = Tab<KIND, BASIS>::value;
  const int c = tb.blocks[B].c;
  for (int b = B - 1; b >= 0 && tb.blocks[b].c == c; --b)
    if (tb.blocks[b].t / TH == HALF) return false;
  return true;
}
__device__ __forceinline__ double2 flip_sign(double2 v, unsigned long long sbit) {
  return make_double2(__longlong_as_double(__double_as_longlong(v.x) ^ static_cast<long long>(sbit)),
                      __longlong_as_double(__double_as_longlong(v.y) ^ static_cast<long long>(sbit)));
}
template <int KIND, int BASIS, int B, int S, int TH, int HALF>
__device__ __forceinline__ void had_block(double2 (&yh)[TH], const double2 (&xh)[S], double2& sh,
                                          const double2* sh_base, int cstride, unsigned long long f1,
                                          unsigned long long f2, unsigned long long f3) {
  constexpr BlockT blk = Tab<KIND, BASIS>::value.blocks[B];
  if constexpr (blk.t / TH == HALF) {
    constexpr bool first = first_in_half<KIND, BASIS>(B, TH, HALF);
    constexpr CompT cp = Tab<KIND, BASIS>::value.comps[blk.c];
    if (first) {
      const unsigned long long sbit = (cp.p0 < 0 ? f1 : 0ull) ^ (cp.p1 < 0 ? f2 : 0ull) ^ (cp.p2 < 0 ? f3 : 0ull);
      sh = flip_sign(sh_base[blk.c * cstride], sbit);
    }
    if (blk.coef > 0) cfma(yh[blk.t - HALF * TH], sh, xh[blk.s]);
    else cfms(yh[blk.t - HALF * TH], sh, xh[blk.s]);
  }
}
template <int KIND, int BASIS, int S, int TH, int HALF, int... Bs>
__device__ __forceinline__ void had_all(std::integer_sequence<int, Bs...>, double2 (&yh)[TH], const double2 (&xh)[S],
                                        const double2* sh_base, int cstride, int m1flag, int m2flag, int mir) {
  double2 sh = make_double2(0.0, 0.0);
  const unsigned long long f1 = static_cast<unsigned long long>(m1flag) << 63;
  const unsigned long long f2 = static_cast<unsigned long long>(m2flag) << 63;
  const unsigned long long f3 = static_cast<unsigned long long>(mir) << 63;
  (had_block<KIND, BASIS, Bs, S, TH, HALF>(yh, xh, sh, sh_base, cstride, f1, f2, f3), ...);
}
}  // namespace vie
using namespace vie;
template <int THREADS>
__global__ void __launch_bounds__(THREADS, 2) k(double2* out, int iters) {
  extern __shared__ double2 sm[];  // x: 12 x THREADS ; S: 60 x 32
  for (int e = threadIdx.x; e < 12 * THREADS + 60 * 32; e += blockDim.x) sm[e] = make_double2(1e-3 * e, 2e-3);
  __syncthreads();
  const int half = (threadIdx.x / 32) & 1;
  double2 acc = make_double2(0, 0);
  for (int it = 0; it < iters; ++it) {
    double2 xh[12], yh[6];
#pragma unroll
    for (int s = 0; s < 12; ++s) xh[s] = sm[threadIdx.x + THREADS * s];
#pragma unroll
    for (int t = 0; t < 6; ++t) yh[t] = make_double2(0, 0);
    const double2* shb = sm + 12 * THREADS + ((threadIdx.x >> 3) & 31);
    if (half == 0)
      had_all<0, 1, 12, 6, 0>(std::make_integer_sequence<int, 144>{}, yh, xh, shb, 32, it & 1, 0, threadIdx.x & 1);
    else
      had_all<0, 1, 12, 6, 1>(std::make_integer_sequence<int, 144>{}, yh, xh, shb, 32, it & 1, 0, threadIdx.x & 1);
#pragma unroll
    for (int t = 0; t < 6; ++t) acc = cadd(acc, yh[t]);
  }
  if (acc.x == 1234.5) out[0] = acc;
}
int main() {
  double2* out;
  cudaMalloc(&out, 16);
  constexpr int T = 256;
  const size_t smem = sizeof(double2) * (12 * T + 60 * 32);
  cudaFuncSetAttribute(k<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 200, blocks = 148 * 2;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    k<T><<<blocks, T, smem>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double dfma = 288.0 * iters * blocks * T;  // DFMA per thread per point
    printf("Hadamard (PWL, 2x256 thr/SM): %.2f TFLOP/s (%.1f%% of 36.3)\n", 2 * dfma / ms / 1e9,
           100 * 2 * dfma / ms / 1e9 / 36.3);
  }
  return 0;
}
