// fft.cuh -- in-shared-memory mixed-radix FP64 FFT passes for sm_100a.
//
// Each stage is one shared-memory pass: a thread loads R elements (stride M),
// runs a radix-R DFT entirely in registers (compile-time factorised, constant
// twiddles), applies the stage twiddles and stores in place.  Plans use 2-3
// stages with radices up to 25, so a length-400 line costs two smem round
// trips instead of four (the v1 radix-4/5 passes were smem-bandwidth bound).
//
// Forward: decimation in frequency, output in digit-reversed slots:
//   stage s (block length L, radix R, M = L/R): for block b and m < M
//   V[k] = DFT_R(x[bL + m + iM])_k * w_L^{k m}  ->  x[bL + m + kM]
// frequency f = k1 + R1 k2 + R1 R2 k3 + ... lands in slot sum_s k_s M_s.
// Inverse: the exact adjoint of the forward stages in reverse order
// (digit-reversed in, natural order out, unnormalised).
// Pruning: `half_in` (forward, first stage) = upper half of every line is
// the circulant zero pad (operator.hpp:290-297) and is never read; `half_out`
// (inverse, last stage) = only the lower half is kept (the crop, :367-375).
#pragma once
#include <type_traits>
#include <utility>

#include "common.cuh"
#include "twiddles_gen.cuh"

namespace vie {

// ----------------------------------------------------------------- register DFTs
// In-place radix-R DFT on the register view v[OFF + ST*i], i < R, fully
// unrolled (compile-time indices).  Composite R = A*B: A-point DFTs over the
// strided subsets, constant twiddles, B-point DFTs; the result X[k] is left
// at register OFF + ST*out_idx<R>(k) (a compile-time permutation, free).
constexpr int first_factor(int R) {
  return (R % 4 == 0 && R > 4) ? 4 : (R % 2 == 0 ? 2 : (R % 3 == 0 ? 3 : (R % 5 == 0 ? 5 : R)));
}
// primes 11..31: direct symmetric-pair DFTs (the Duke head's embedded lengths 186 = 6 x 31 and
// 238 = 14 x 17 need them); only the EXT instantiations of the two-stage passes use them
constexpr bool is_ext_prime(int R) {
  return R == 11 || R == 13 || R == 17 || R == 19 || R == 23 || R == 29 || R == 31;
}
constexpr bool is_base(int R) {
  return R == 1 || R == 2 || R == 3 || R == 4 || R == 5 || R == 7 || is_ext_prime(R);
}
constexpr int out_idx(int R, int k) {
  return is_base(R) ? k
                    : (R / first_factor(R)) * out_idx(first_factor(R), k % first_factor(R)) +
                          out_idx(R / first_factor(R), k / first_factor(R));
}

template <int... Is, class F>
__device__ __forceinline__ void sfor_impl(std::integer_sequence<int, Is...>, F&& f) {
  (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void sfor(F&& f) {
  sfor_impl(std::make_integer_sequence<int, N>{}, f);
}

// x * exp(-+2 pi i e / R), e a compile-time constant
template <int R, bool INV, int E0>
__device__ __forceinline__ double2 twc(double2 x) {
  constexpr int e = E0 % R;
  if constexpr (e == 0) {
    return x;
  } else if constexpr (4 * e == R) {
    return mul_mi<INV>(x);  // -i (fwd) / +i (inv)
  } else if constexpr (2 * e == R) {
    return make_double2(-x.x, -x.y);
  } else if constexpr (4 * e == 3 * R) {
    return mul_mi<!INV>(x);
  } else {
    constexpr double c = tw_re(R, e);
    constexpr double s = INV ? -tw_im(R, e) : tw_im(R, e);
    return make_double2(fma(x.x, c, -x.y * s), fma(x.x, s, x.y * c));
  }
}

constexpr int gcd_c(int a, int b) { return b == 0 ? a : gcd_c(b, a % b); }
constexpr int inv_mod(int a, int m) {  // a^-1 mod m (a, m coprime)
  for (int x = 1; x < m; ++x)
    if ((a * x) % m == 1) return x;
  return 1;
}

template <int R, bool INV, int ST, int OFF>
struct DFTs {
  static constexpr int A = first_factor(R);
  static constexpr int B = R / A;
  __device__ __forceinline__ static void run(double2* v) {
    if constexpr (is_ext_prime(R)) {
      // prime R: pairs a_j = x_j + x_{R-j}, b_j = x_j - x_{R-j} (j <= H); X_0 = x_0 + sum a_j,
      // X_k, X_{R-k} = x_0 + sum_j cos(2 pi j k / R) a_j -+ i sum_j sin(2 pi j k / R) b_j
      // (signs swapped for the inverse), ~R^2 real FMAs instead of 2 R^2 complex ones
      constexpr int H = (R - 1) / 2;
      double2 a[H], b[H];
      const double2 x0 = v[OFF];
      sfor<H>([&](auto jc) {
        constexpr int j = decltype(jc)::value + 1;
        a[j - 1] = cadd(v[OFF + ST * j], v[OFF + ST * (R - j)]);
        b[j - 1] = csub(v[OFF + ST * j], v[OFF + ST * (R - j)]);
      });
      double2 s0 = x0;
      sfor<H>([&](auto jc) { s0 = cadd(s0, a[decltype(jc)::value]); });
      sfor<H>([&](auto kc) {
        constexpr int kk = decltype(kc)::value + 1;
        double2 re = x0, im = make_double2(0.0, 0.0);
        sfor<H>([&](auto jc) {
          constexpr int j = decltype(jc)::value + 1;
          constexpr double c = tw_re(R, (j * kk) % R);
          constexpr double s = -tw_im(R, (j * kk) % R);  // sin(2 pi j k / R)
          re = make_double2(fma(c, a[j - 1].x, re.x), fma(c, a[j - 1].y, re.y));
          im = make_double2(fma(s, b[j - 1].x, im.x), fma(s, b[j - 1].y, im.y));
        });
        const double2 t = mul_mi<INV>(im);
        v[OFF + ST * kk] = cadd(re, t);
        v[OFF + ST * (R - kk)] = csub(re, t);
      });
      v[OFF] = s0;
      return;
    } else if constexpr (gcd_c(A, B) == 1 && B > 1) {
      // Good-Thomas prime-factor algorithm (A, B coprime): no inner twiddles.  Input index
      // n = (B n1 + A n2) mod R; output k = k1 (mod A), k2 (mod B).  All index maps are
      // compile-time register renamings; X[k] lands at the same register as in the
      // Cooley-Tukey form below (out_idx), so callers see one contract.
      double2 t[R];
      sfor<A>([&](auto n1c) {
        sfor<B>([&](auto n2c) {
          constexpr int n1 = decltype(n1c)::value, n2 = decltype(n2c)::value;
          t[n2 * A + n1] = v[OFF + ST * ((B * n1 + A * n2) % R)];
        });
      });
      sfor<B>([&](auto n2c) { DFTs<A, INV, 1, decltype(n2c)::value * A>::run(t); });
      sfor<A>([&](auto k1c) { DFTs<B, INV, A, out_idx(A, decltype(k1c)::value)>::run(t); });
      // W^(n k) = W_A^(n1 k) W_B^(n2 k): the A-point stage gives k mod A, the B-point stage
      // k mod B, so t[out_idx(B, k2) A + out_idx(A, k1)] = X[k] with k = CRT(k1, k2)
      sfor<A>([&](auto k1c) {
        sfor<B>([&](auto k2c) {
          constexpr int k1 = decltype(k1c)::value, k2 = decltype(k2c)::value;
          constexpr int k = (k1 * B * inv_mod(B % A, A) + k2 * A * inv_mod(A % B, B)) % R;
          v[OFF + ST * out_idx(R, k)] = t[out_idx(B, k2) * A + out_idx(A, k1)];
        });
      });
      return;
    } else {
    sfor<B>([&](auto n2c) {
      constexpr int n2 = decltype(n2c)::value;
      DFTs<A, INV, ST * B, OFF + ST * n2>::run(v);
      sfor<A>([&](auto k1c) {
        constexpr int k1 = decltype(k1c)::value;
        constexpr int pos = OFF + ST * (B * out_idx(A, k1) + n2);
        v[pos] = twc<R, INV, n2 * k1>(v[pos]);
      });
    });
    sfor<A>([&](auto k1c) {
      constexpr int k1 = decltype(k1c)::value;
      DFTs<B, INV, ST, OFF + ST * B * out_idx(A, k1)>::run(v);
    });
    }
  }
};

template <bool INV, int ST, int OFF>
struct DFTs<1, INV, ST, OFF> {
  __device__ __forceinline__ static void run(double2*) {}
};

template <bool INV, int ST, int OFF>
struct DFTs<2, INV, ST, OFF> {
  __device__ __forceinline__ static void run(double2* v) {
    const double2 a = v[OFF], b = v[OFF + ST];
    v[OFF] = cadd(a, b);
    v[OFF + ST] = csub(a, b);
  }
};

template <bool INV, int ST, int OFF>
struct DFTs<3, INV, ST, OFF> {
  __device__ __forceinline__ static void run(double2* v) {
    const double s3 = 0.86602540378443864676372317075294;
    const double2 x0 = v[OFF], x1 = v[OFF + ST], x2 = v[OFF + 2 * ST];
    const double2 t1 = cadd(x1, x2);
    const double2 t2 = make_double2(fma(-0.5, t1.x, x0.x), fma(-0.5, t1.y, x0.y));
    const double2 d = csub(x1, x2);
    const double2 t3 = mul_mi<INV>(make_double2(s3 * d.x, s3 * d.y));
    v[OFF] = cadd(x0, t1);
    v[OFF + ST] = cadd(t2, t3);
    v[OFF + 2 * ST] = csub(t2, t3);
  }
};

template <bool INV, int ST, int OFF>
struct DFTs<4, INV, ST, OFF> {
  __device__ __forceinline__ static void run(double2* v) {
    const double2 x0 = v[OFF], x1 = v[OFF + ST], x2 = v[OFF + 2 * ST], x3 = v[OFF + 3 * ST];
    const double2 s02 = cadd(x0, x2), d02 = csub(x0, x2);
    const double2 s13 = cadd(x1, x3), d13 = mul_mi<INV>(csub(x1, x3));
    v[OFF] = cadd(s02, s13);
    v[OFF + ST] = cadd(d02, d13);
    v[OFF + 2 * ST] = csub(s02, s13);
    v[OFF + 3 * ST] = csub(d02, d13);
  }
};

template <bool INV, int ST, int OFF>
struct DFTs<5, INV, ST, OFF> {
  __device__ __forceinline__ static void run(double2* v) {
    const double c1 = 0.30901699437494742410229341718282;   // cos(2pi/5)
    const double c2 = -0.80901699437494742410229341718282;  // cos(4pi/5)
    const double s1 = 0.95105651629515357211643933337938;   // sin(2pi/5)
    const double s2 = 0.58778525229247312916870595463907;   // sin(4pi/5)
    const double2 x0 = v[OFF];
    const double2 t1 = cadd(v[OFF + ST], v[OFF + 4 * ST]), t2 = cadd(v[OFF + 2 * ST], v[OFF + 3 * ST]);
    const double2 t3 = csub(v[OFF + ST], v[OFF + 4 * ST]), t4 = csub(v[OFF + 2 * ST], v[OFF + 3 * ST]);
    const double2 a1 = make_double2(fma(c2, t2.x, fma(c1, t1.x, x0.x)), fma(c2, t2.y, fma(c1, t1.y, x0.y)));
    const double2 a2 = make_double2(fma(c1, t2.x, fma(c2, t1.x, x0.x)), fma(c1, t2.y, fma(c2, t1.y, x0.y)));
    const double2 b1 = mul_mi<INV>(make_double2(fma(s2, t4.x, s1 * t3.x), fma(s2, t4.y, s1 * t3.y)));
    const double2 b2 = mul_mi<INV>(make_double2(fma(-s1, t4.x, s2 * t3.x), fma(-s1, t4.y, s2 * t3.y)));
    v[OFF] = cadd(x0, cadd(t1, t2));
    v[OFF + ST] = cadd(a1, b1);
    v[OFF + 4 * ST] = csub(a1, b1);
    v[OFF + 2 * ST] = cadd(a2, b2);
    v[OFF + 3 * ST] = csub(a2, b2);
  }
};

template <bool INV, int ST, int OFF>
struct DFTs<7, INV, ST, OFF> {  // direct form with constant twiddles
  __device__ __forceinline__ static void run(double2* v) {
    double2 x[7], o[7];
    sfor<7>([&](auto jc) { x[decltype(jc)::value] = v[OFF + ST * decltype(jc)::value]; });
    sfor<7>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      double2 acc = x[0];
      sfor<6>([&](auto jc) {
        constexpr int j = decltype(jc)::value + 1;
        acc = cadd(acc, twc<7, INV, j * k>(x[j]));
      });
      o[k] = acc;
    });
    sfor<7>([&](auto kc) { v[OFF + ST * decltype(kc)::value] = o[decltype(kc)::value]; });
  }
};

// ----------------------------------------------------------------- stages
// Stage twiddles w_L^{k m} = tw[k m tws]: w^1 from the table, higher powers by
// recurrence (error ~k eps, k < 25).
template <int R>
__device__ __forceinline__ void dif_stage(double2* buf, int nlines, int ls, int n, const StageDesc& sd,
                                          const double2* tw, bool half_in, int tid, int nth) {
  const int M = sd.M, L = sd.L, tws = sd.tws;
  const int nbf = n / R;
  const int total = nlines * nbf;
  for (int u = tid; u < total; u += nth) {
    const int line = sd.div_nbf.div(u);
    const int bm = u - line * nbf;
    const int b = sd.div_M.div(bm);
    const int m = bm - b * M;
    double2* base = buf + line * ls + b * L + m;
    double2 v[R];
    if (half_in) {
#pragma unroll
      for (int i = 0; i < R; ++i) v[i] = (i < R / 2) ? base[i * M] : make_double2(0.0, 0.0);
    } else {
#pragma unroll
      for (int i = 0; i < R; ++i) v[i] = base[i * M];
    }
    DFTs<R, false, 1, 0>::run(v);
    base[0] = v[out_idx(R, 0)];
    if (m == 0) {
      sfor<R - 1>([&](auto kc) {
        constexpr int k = decltype(kc)::value + 1;
        base[k * M] = v[out_idx(R, k)];
      });
    } else {
      const double2 w1 = tw[m * tws];
      double2 w = w1;
      sfor<R - 1>([&](auto kc) {
        constexpr int k = decltype(kc)::value + 1;
        base[k * M] = cmul(v[out_idx(R, k)], w);
        if (k + 1 < R) w = cmul(w, w1);
      });
    }
  }
}

template <int R>
__device__ __forceinline__ void dit_stage_adj(double2* buf, int nlines, int ls, int n, const StageDesc& sd,
                                              const double2* tw, bool half_out, int tid, int nth) {
  const int M = sd.M, L = sd.L, tws = sd.tws;
  const int nbf = n / R;
  const int total = nlines * nbf;
  for (int u = tid; u < total; u += nth) {
    const int line = sd.div_nbf.div(u);
    const int bm = u - line * nbf;
    const int b = sd.div_M.div(bm);
    const int m = bm - b * M;
    double2* base = buf + line * ls + b * L + m;
    double2 v[R];
    v[0] = base[0];
    if (m == 0) {
#pragma unroll
      for (int k = 1; k < R; ++k) v[k] = base[k * M];
    } else {
      const double2 w1 = tw[m * tws];
      double2 w = w1;
#pragma unroll
      for (int k = 1; k < R; ++k) {
        v[k] = cmulc(base[k * M], w);
        if (k + 1 < R) w = cmul(w, w1);
      }
    }
    DFTs<R, true, 1, 0>::run(v);
    if (half_out) {
      sfor<R / 2>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        base[i * M] = v[out_idx(R, i)];
      });
    } else {
      sfor<R>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        base[i * M] = v[out_idx(R, i)];
      });
    }
  }
}

// Radices the plans may use (api.cu get_plan chooses among these).  Small set
// (<= 10, low register pressure) for the occupancy-bound row/column passes;
// wide set (two-stage plans, fewer smem passes) for the pencil kernel, which
// owns its SM and has 128 registers per thread.
#define VIE_FFT_RADICES(X) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(10)
#define VIE_FFT_RADICES_WIDE(X) VIE_FFT_RADICES(X) X(12) X(15) X(16) X(20) X(24)
// radices with a prime factor 11..31 (two-stage row / column passes only, EXT instantiation)
#define VIE_FFT_RADICES_EXT_EVEN(X) X(14) X(22) X(26) X(34)
#define VIE_FFT_RADICES_EXT(X) VIE_FFT_RADICES_EXT_EVEN(X) X(11) X(13) X(17) X(19) X(23) X(29) X(31)

template <bool INV, bool WIDE = false>
__device__ __forceinline__ void run_stage(double2* buf, int nlines, int ls, int n, const StageDesc& sd,
                                          const double2* tw, bool prune, int tid, int nth) {
  switch (sd.radix) {
#define VIE_CASE(R)                                                          \
  case R:                                                                    \
    if (INV) dit_stage_adj<R>(buf, nlines, ls, n, sd, tw, prune, tid, nth);  \
    else dif_stage<R>(buf, nlines, ls, n, sd, tw, prune, tid, nth);          \
    break;
    VIE_FFT_RADICES(VIE_CASE)
#undef VIE_CASE
    default:
      if constexpr (WIDE) {
        switch (sd.radix) {
#define VIE_CASE(R)                                                          \
  case R:                                                                    \
    if (INV) dit_stage_adj<R>(buf, nlines, ls, n, sd, tw, prune, tid, nth);  \
    else dif_stage<R>(buf, nlines, ls, n, sd, tw, prune, tid, nth);          \
    break;
          VIE_CASE(12)
          VIE_CASE(15)
          VIE_CASE(16)
          VIE_CASE(20)
          VIE_CASE(24)
#undef VIE_CASE
          default:
            break;
        }
      }
      break;  // plan creation rejects other radices
  }
}

// Per-CTA shared copy of a plan: twiddles, digit-reversal slots, stages.
struct SmemPlan {
  int n, nst;
  double2* tw;
  int* slot;
  StageDesc* st;
};

// smem footprint (in double2 units) of the tables of an n-point plan
__host__ __device__ __forceinline__ int plan_smem_elems(int n) {
  return n + (n + 3) / 4 + (static_cast<int>(sizeof(StageDesc)) * kMaxStages + 15) / 16;
}

// Carve the tables out of `sm` and fill them (caller syncs before use).
__device__ __forceinline__ SmemPlan load_plan(double2* sm, const FftPlan& P) {
  SmemPlan s;
  s.n = P.n;
  s.nst = P.nst;
  s.tw = sm;
  s.slot = reinterpret_cast<int*>(sm + P.n);
  s.st = reinterpret_cast<StageDesc*>(sm + P.n + (P.n + 3) / 4);
  for (int e = threadIdx.x; e < P.n; e += blockDim.x) {
    s.tw[e] = P.tw[e];
    s.slot[e] = P.slot[e];
  }
  if (threadIdx.x < P.nst) s.st[threadIdx.x] = P.st[threadIdx.x];
  return s;
}

// Full forward transform of `nlines` lines in smem (digit-reversed output).
template <bool WIDE = false>
__device__ __forceinline__ void fft_forward(double2* buf, int nlines, int ls, const SmemPlan& P, bool half_in) {
  const int tid = threadIdx.x, nth = blockDim.x;
  for (int s = 0; s < P.nst; ++s) {
    run_stage<false, WIDE>(buf, nlines, ls, P.n, P.st[s], P.tw, half_in && s == 0, tid, nth);
    __syncthreads();
  }
}

// Full inverse transform (digit-reversed input, natural unnormalised output).
template <bool WIDE = false>
__device__ __forceinline__ void fft_inverse(double2* buf, int nlines, int ls, const SmemPlan& P, bool half_out) {
  const int tid = threadIdx.x, nth = blockDim.x;
  for (int s = P.nst - 1; s >= 0; --s) {
    run_stage<true, WIDE>(buf, nlines, ls, P.n, P.st[s], P.tw, half_out && s == 0, tid, nth);
    __syncthreads();
  }
}

}  // namespace vie
