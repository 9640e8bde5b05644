// common.cuh -- shared device helpers for the B200 VIE matvec (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <array>

namespace vie {

// ---------------------------------------------------------------- complex fp64
__host__ __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__host__ __device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // a * conj(b)
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__host__ __device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// acc += a * b
__host__ __device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
// acc -= a * b
__host__ __device__ __forceinline__ void cfms(double2& acc, double2 a, double2 b) {
  acc.x = fma(-a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(-a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}
// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ double2 mul_mi(double2 a) {
  return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

// ---------------------------------------------------------------- fast divmod
// Division by a runtime-invariant divisor (x < 2^31), CUTLASS-style.
struct FastDiv {
  uint32_t d, mul, shr;
  __host__ void init(uint32_t den) {
    d = den;
    if (den <= 1) {
      mul = 0;
      shr = 0;
      return;
    }
    uint32_t l = 0;
    while ((1u << l) < den) ++l;
    const uint32_t p = 31 + l;
    mul = static_cast<uint32_t>(((1ull << p) + den - 1) / den);
    shr = p - 32;
  }
  __device__ __forceinline__ uint32_t div(uint32_t x) const {
    return d <= 1 ? x : (__umulhi(x, mul) >> shr);
  }
};

// ---------------------------------------------------------------- FFT plans
// In-place mixed-radix DIF forward transform (digit-reversed output slots)
// and its adjoint (digit-reversed input -> natural output), see fft.cuh.
constexpr int kMaxStages = 12;
struct StageDesc {
  int radix;
  int L;    // block length entering the stage
  int M;    // L / radix
  int tws;  // twiddle stride n / L
  FastDiv div_nbf;  // n / radix (butterflies per line)
  FastDiv div_M;
};
// Kernel-parameter view of a plan: only fixed-offset fields (dynamic indexing
// into kernel parameters would force a local-memory copy).
struct FftPlan {
  int n;    // transform length (= 2 * grid edge)
  int nst;  // number of stages
  const StageDesc* st;   // device: nst stage descriptors
  const double2* tw;     // device: w[e] = exp(-2 pi i e / n), n entries
  const int* slot;       // device: slot_of_freq[f], n entries
};

// ---------------------------------------------------------------- mirror-paired
// spectral ordering of an axis of length m = 2n: positions (2p, 2p+1) hold
// frequencies (p, m-p) for 1 <= p < n; positions 0, 1 hold frequencies 0, n.
__host__ __device__ __forceinline__ int freq_of_pos(int P, int n) {
  if (P == 0) return 0;
  if (P == 1) return n;
  return (P & 1) ? 2 * n - (P >> 1) : (P >> 1);
}
__host__ __device__ __forceinline__ int pos_of_freq(int f, int n) {
  if (f == 0) return 0;
  if (f == n) return 1;
  return f < n ? 2 * f : 2 * (2 * n - f) + 1;
}

// ---------------------------------------------------------------- tables
// Component tables (product-side implementation; the oracle has its own).
// PWC: components.hpp:71-92 + operator.hpp:205-219.  PWL: DESIGN.md.
struct CompT {
  int q, qp, l, lp, p0, p1, p2;
};
struct BlockT {
  int t, s, c, coef;  // FFT-path coefficient = dense_sign * prod(parity)
};

template <int KIND, int BASIS>
struct TableDims {
  static constexpr int L = BASIS == 0 ? 1 : 4;
  static constexpr int S = 3 * L;
  static constexpr int NQ = KIND == 0 ? 6 : 3;
  static constexpr int NC = NQ * (L * (L + 1) / 2);
  static constexpr int NB = KIND == 0 ? (BASIS == 0 ? 9 : 144) : (BASIS == 0 ? 6 : 96);
};

template <int KIND, int BASIS>
struct Table {
  std::array<CompT, TableDims<KIND, BASIS>::NC> comps{};
  std::array<BlockT, TableDims<KIND, BASIS>::NB> blocks{};
};

template <int KIND, int BASIS>
constexpr Table<KIND, BASIS> make_table() {
  Table<KIND, BASIS> tb{};
  constexpr int L = TableDims<KIND, BASIS>::L;
  int nc = 0, nb = 0;
  for (int q = 0; q < 3; ++q)
    for (int qp = (KIND == 0 ? q : q + 1); qp < 3; ++qp)
      for (int l = 0; l < L; ++l)
        for (int lp = l; lp < L; ++lp) {
          int par[3] = {1, 1, 1};
          for (int a = 0; a < 3; ++a) {
            int odd = (l == a + 1) + (lp == a + 1);
            if (KIND == 0) odd += (q == a) + (qp == a);
            else odd += (a == 3 - q - qp);
            par[a] = (odd % 2) ? -1 : 1;
          }
          tb.comps[nc] = CompT{q, qp, l, lp, par[0], par[1], par[2]};
          const int sigma = par[0] * par[1] * par[2];
          const int kappa = KIND == 0 ? 1 : -1;
          const int t0[4] = {q * L + l, qp * L + l, q * L + lp, qp * L + lp};
          const int s0[4] = {qp * L + lp, q * L + lp, qp * L + l, q * L + l};
          const int ds[4] = {1, kappa, kappa * sigma, sigma};
          const int first = nb;
          for (int k = 0; k < 4; ++k) {
            bool dup = false;
            for (int e = first; e < nb; ++e) dup = dup || (tb.blocks[e].t == t0[k] && tb.blocks[e].s == s0[k]);
            if (!dup) {
              tb.blocks[nb] = BlockT{t0[k], s0[k], nc, ds[k] * sigma};
              ++nb;
            }
          }
          ++nc;
        }
  return tb;
}

}  // namespace vie

#define VIE_CUDA_CHECK(expr)                                                   \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) throw ::vie::CudaError(_e, #expr, __FILE__, __LINE__); \
  } while (0)

#include <stdexcept>
#include <string>
namespace vie {
struct CudaError : std::runtime_error {
  cudaError_t code;
  CudaError(cudaError_t e, const char* expr, const char* file, int line)
      : std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(e) + " at " + file + ":" +
                           std::to_string(line) + " (" + expr + ")"),
        code(e) {}
};
}  // namespace vie
