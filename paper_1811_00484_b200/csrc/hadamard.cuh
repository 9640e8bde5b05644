// hadamard.cuh -- the fused Hadamard of apply_operator (operator.hpp:303-364,
// mac_elementwise over every (target, source, component) block) for one
// spectral point, unrolled at compile time from the block table (common.cuh
// make_table): x^ of all sources in registers, y^ of one target half in
// registers, octant spectrum values read once per component and sign-flipped
// for the mirrored point.
#pragma once
#include <utility>

#include "common.cuh"

namespace vie {
namespace had {

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
__device__ __forceinline__ double2 flip_sign(double2 v, unsigned long long sbit) {
  // branch-free negation: xor of the IEEE sign bits (integer pipe)
  return make_double2(__longlong_as_double(__double_as_longlong(v.x) ^ static_cast<long long>(sbit)),
                      __longlong_as_double(__double_as_longlong(v.y) ^ static_cast<long long>(sbit)));
}

// Block B of the table, all indices compile-time constants; only blocks whose
// target is in [HALF*TH, HALF*TH + TH) (target split across two threads).
// ALL = every component active (no per-component branch: lets the compiler
// schedule spectrum loads and FMAs across components).
// Component groups: the spectrum is streamed NG groups of CG components at a
// time (double-buffered cp.async) while y^ stays in registers.
template <int NC>
constexpr int n_groups() {
  return NC >= 16 ? 3 : 1;
}
template <int NC>
constexpr int group_size() {
  return (NC + n_groups<NC>() - 1) / n_groups<NC>();
}

template <int KIND, int BASIS, int B, int S, int TH, int HALF, bool ALL, int GRP, int CG>
__device__ __forceinline__ void had_block(double2 (&yh)[TH], const double2 (&xh)[S], double2& sh,
                                          const double2* sh_base, int cstride, uint64_t active,
                                          unsigned long long f1, unsigned long long f2, unsigned long long f3) {
  constexpr BlockT blk = Tab<KIND, BASIS>::value.blocks[B];
  if constexpr (blk.t / TH == HALF && blk.c / CG == GRP) {
    constexpr bool first = first_in_half<KIND, BASIS>(B, TH, HALF);
    constexpr CompT cp = Tab<KIND, BASIS>::value.comps[blk.c];
    if (!ALL && !((active >> blk.c) & 1ull)) return;
    if (first) {
      // sign of the mirrored point: product of the odd-axis flags (sign bits)
      const unsigned long long sbit = (cp.p0 < 0 ? f1 : 0ull) ^ (cp.p1 < 0 ? f2 : 0ull) ^ (cp.p2 < 0 ? f3 : 0ull);
      sh = flip_sign(sh_base[blk.c * cstride], sbit);
    }
    if (blk.coef > 0) cfma(yh[blk.t - HALF * TH], sh, xh[blk.s]);
    else cfms(yh[blk.t - HALF * TH], sh, xh[blk.s]);
  }
}

template <int KIND, int BASIS, int S, int TH, int HALF, bool ALL, int GRP, int CG, int... Bs>
__device__ __forceinline__ void had_all(std::integer_sequence<int, Bs...>, double2 (&yh)[TH], const double2 (&xh)[S],
                                        const double2* sh_base, int cstride, uint64_t active, int m1flag, int m2flag,
                                        int mir) {
  double2 sh = make_double2(0.0, 0.0);
  const unsigned long long f1 = static_cast<unsigned long long>(m1flag) << 63;
  const unsigned long long f2 = static_cast<unsigned long long>(m2flag) << 63;
  const unsigned long long f3 = static_cast<unsigned long long>(mir) << 63;
  (had_block<KIND, BASIS, Bs, S, TH, HALF, ALL, GRP, CG>(yh, xh, sh, sh_base, cstride, active, f1, f2, f3), ...);
}

// ---- sign factorisation.  The mirrored-point sign of component c is
// prod_a sigma_a^{P_a(c)} (P = odd-axis pattern, sigma = the point's mirror flags).
// For every table the pattern splits over the block's currents:
// P(c) = pi(t) ^ pi(s) ^ G for each block (t, s, c) (N: pi(q,l) = axis of q and of
// the linear direction of l, G = 0; K: the same with G = all axes), so the sign
// moves from every spectrum value (NC flips per point) onto x^_s before and y^_t
// after the block sum (2 S flips per point).  Derived and verified at compile time.
template <int S>
struct SignSplit {
  int pi[S];
  int G;
  bool ok;
};
template <int KIND, int BASIS>
constexpr SignSplit<TableDims<KIND, BASIS>::S> make_sign_split() {
  constexpr int S = TableDims<KIND, BASIS>::S, NB = TableDims<KIND, BASIS>::NB;
  const auto& tb = Tab<KIND, BASIS>::value;
  SignSplit<S> r{};
  for (int G : {0, 7}) {
    for (int s = 0; s < S; ++s) r.pi[s] = -1;
    r.pi[0] = 0;
    for (int it = 0; it < S; ++it)
      for (int b = 0; b < NB; ++b) {
        const BlockT& bk = tb.blocks[b];
        const CompT& cp = tb.comps[bk.c];
        const int P = (cp.p0 < 0 ? 1 : 0) | (cp.p1 < 0 ? 2 : 0) | (cp.p2 < 0 ? 4 : 0);
        if (r.pi[bk.t] >= 0 && r.pi[bk.s] < 0) r.pi[bk.s] = P ^ r.pi[bk.t] ^ G;
        if (r.pi[bk.s] >= 0 && r.pi[bk.t] < 0) r.pi[bk.t] = P ^ r.pi[bk.s] ^ G;
      }
    bool ok = true;
    for (int s = 0; s < S; ++s)
      if (r.pi[s] < 0) r.pi[s] = 0;
    for (int b = 0; b < NB; ++b) {
      const BlockT& bk = tb.blocks[b];
      const CompT& cp = tb.comps[bk.c];
      const int P = (cp.p0 < 0 ? 1 : 0) | (cp.p1 < 0 ? 2 : 0) | (cp.p2 < 0 ? 4 : 0);
      if (P != (r.pi[bk.t] ^ r.pi[bk.s] ^ G)) ok = false;
    }
    if (ok) {
      r.G = G;
      r.ok = true;
      return r;
    }
  }
  r.ok = false;
  return r;
}
template <int KIND, int BASIS>
struct Signs {
  static constexpr SignSplit<TableDims<KIND, BASIS>::S> value = make_sign_split<KIND, BASIS>();
  static_assert(value.ok, "component parities do not factor over the block currents");
};

// sign bit (IEEE bit 63) of pattern v at a point with mirror flags bits = m1 | m2 << 1 | mir << 2
__device__ __forceinline__ unsigned long long pattern_sign(int v, int bits) {
  return static_cast<unsigned long long>(__popc(v & bits) & 1) << 63;
}

// Block sum without per-value signs (x^ pre-signed, y^ post-signed by the caller).
template <int KIND, int BASIS, int B, int S, int TH, int GRP, int CG>
__device__ __forceinline__ void had_block_ns(double2 (&yh)[TH], const double2 (&xh)[S], double2& sh,
                                             const double2* sh_base, int cstride) {
  constexpr BlockT blk = Tab<KIND, BASIS>::value.blocks[B];
  if constexpr (blk.c / CG == GRP) {
    constexpr bool first = first_in_half<KIND, BASIS>(B, TH, 0);
    if (first) sh = sh_base[blk.c * cstride];
    if (blk.coef > 0) cfma(yh[blk.t], sh, xh[blk.s]);
    else cfms(yh[blk.t], sh, xh[blk.s]);
  }
}
template <int KIND, int BASIS, int S, int TH, int GRP, int CG, int... Bs>
__device__ __forceinline__ void had_all_ns(std::integer_sequence<int, Bs...>, double2 (&yh)[TH], const double2 (&xh)[S],
                                           const double2* sh_base, int cstride) {
  static_assert(TH == S, "unsplit targets");
  double2 sh = make_double2(0.0, 0.0);
  (had_block_ns<KIND, BASIS, Bs, S, TH, GRP, CG>(yh, xh, sh, sh_base, cstride), ...);
}

template <int... Is, class F>
__device__ __forceinline__ void sfor_g(std::integer_sequence<int, Is...>, F&& f) {
  (f(std::integral_constant<int, Is>{}), ...);
}

}  // namespace had
}  // namespace vie
