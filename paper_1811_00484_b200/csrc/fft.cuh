// fft.cuh -- in-shared-memory mixed-radix FP64 FFT stages for sm_100a.
//
// Forward: decimation-in-frequency, in place, output in digit-reversed slots:
//   stage s (block length L, radix r, M = L/r): for each block b and m < M
//   V[k] = DFT_r(x[bL + m + iM])_k * w_L^{k m}  -> x[bL + m + kM].
// The frequency f = k1 + r1 k2 + r1 r2 k3 + ... lands in slot sum_s k_s M_s.
// Inverse: the exact adjoint of the forward stages applied in reverse order,
// consuming digit-reversed slots and producing natural order (unnormalised).
//
// Pruning: `half_in` (forward) means the upper half of every line is zero
// (the circulant pad, operator.hpp:290-297) and is never read; `half_out`
// (inverse) means only the lower half is needed (the crop, :367-375).  Both
// need an even first radix.
#pragma once
#include "common.cuh"

namespace vie {

template <int R, bool INV>
struct Bfly {
  // generic prime radix via the twiddle table (w_R^{jk} = w_N^{(jk mod R) N/R})
  __device__ __forceinline__ static void run(double2* v, const double2* tw, int n_over_r) {
    double2 o[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      double2 acc = v[0];
#pragma unroll
      for (int j = 1; j < R; ++j) {
        double2 w = tw[((j * k) % R) * n_over_r];
        if (INV) w.y = -w.y;
        cfma(acc, v[j], w);
      }
      o[k] = acc;
    }
#pragma unroll
    for (int k = 0; k < R; ++k) v[k] = o[k];
  }
};

template <bool INV>
struct Bfly<2, INV> {
  __device__ __forceinline__ static void run(double2* v, const double2*, int) {
    const double2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  }
};

template <bool INV>
struct Bfly<3, INV> {
  __device__ __forceinline__ static void run(double2* v, const double2*, int) {
    const double s3 = 0.86602540378443864676372317075294;
    const double2 t1 = cadd(v[1], v[2]);
    const double2 t2 = make_double2(fma(-0.5, t1.x, v[0].x), fma(-0.5, t1.y, v[0].y));
    const double2 d = csub(v[1], v[2]);
    const double2 t3 = mul_mi<INV>(make_double2(s3 * d.x, s3 * d.y));
    v[0] = cadd(v[0], t1);
    v[1] = cadd(t2, t3);
    v[2] = csub(t2, t3);
  }
};

template <bool INV>
struct Bfly<4, INV> {
  __device__ __forceinline__ static void run(double2* v, const double2*, int) {
    const double2 s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
    const double2 s13 = cadd(v[1], v[3]), d13 = mul_mi<INV>(csub(v[1], v[3]));
    v[0] = cadd(s02, s13);
    v[1] = cadd(d02, d13);
    v[2] = csub(s02, s13);
    v[3] = csub(d02, d13);
  }
};

template <bool INV>
struct Bfly<5, INV> {
  __device__ __forceinline__ static void run(double2* v, const double2*, int) {
    const double c1 = 0.30901699437494742410229341718282;   // cos(2pi/5)
    const double c2 = -0.80901699437494742410229341718282;  // cos(4pi/5)
    const double s1 = 0.95105651629515357211643933337938;   // sin(2pi/5)
    const double s2 = 0.58778525229247312916870595463907;   // sin(4pi/5)
    const double2 t1 = cadd(v[1], v[4]), t2 = cadd(v[2], v[3]);
    const double2 t3 = csub(v[1], v[4]), t4 = csub(v[2], v[3]);
    const double2 a1 = make_double2(fma(c2, t2.x, fma(c1, t1.x, v[0].x)), fma(c2, t2.y, fma(c1, t1.y, v[0].y)));
    const double2 a2 = make_double2(fma(c1, t2.x, fma(c2, t1.x, v[0].x)), fma(c1, t2.y, fma(c2, t1.y, v[0].y)));
    const double2 b1 = mul_mi<INV>(make_double2(fma(s2, t4.x, s1 * t3.x), fma(s2, t4.y, s1 * t3.y)));
    const double2 b2 = mul_mi<INV>(make_double2(fma(-s1, t4.x, s2 * t3.x), fma(-s1, t4.y, s2 * t3.y)));
    v[0] = cadd(v[0], cadd(t1, t2));
    v[1] = cadd(a1, b1);
    v[4] = csub(a1, b1);
    v[2] = cadd(a2, b2);
    v[3] = csub(a2, b2);
  }
};

template <bool INV>
struct Bfly<8, INV> {
  __device__ __forceinline__ static void run(double2* v, const double2* tw, int n_over_r) {
    const double h = 0.70710678118654752440084436210485;
    // radix-2 x 4: even/odd split
    double2 e[4] = {v[0], v[2], v[4], v[6]};
    double2 o[4] = {v[1], v[3], v[5], v[7]};
    Bfly<4, INV>::run(e, tw, n_over_r);
    Bfly<4, INV>::run(o, tw, n_over_r);
    // o[k] *= w8^k
    const double2 o1 = o[1], o2 = o[2], o3 = o[3];
    o[1] = INV ? make_double2(h * (o1.x - o1.y), h * (o1.x + o1.y)) : make_double2(h * (o1.x + o1.y), h * (o1.y - o1.x));
    o[2] = mul_mi<INV>(o2);
    o[3] = INV ? make_double2(-h * (o3.x + o3.y), h * (o3.x - o3.y)) : make_double2(h * (o3.y - o3.x), -h * (o3.x + o3.y));
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[k] = cadd(e[k], o[k]);
      v[k + 4] = csub(e[k], o[k]);
    }
  }
};

// One forward DIF stage over `nlines` lines (line stride `ls` elements).
template <int R>
__device__ __forceinline__ void dif_stage(double2* buf, int nlines, int ls, int n, const StageDesc& sd,
                                          const double2* tw, bool half_in, int tid, int nth) {
  const int M = sd.M, L = sd.L, tws = sd.tws;
  const int nbf = n / R;
  const int total = nlines * nbf;
  const int nr = n / R;
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
    Bfly<R, false>::run(v, tw, nr);
    base[0] = v[0];
#pragma unroll
    for (int k = 1; k < R; ++k) base[k * M] = (m == 0) ? v[k] : cmul(v[k], tw[k * m * tws]);
  }
}

// One inverse (adjoint) stage.
template <int R>
__device__ __forceinline__ void dit_stage_adj(double2* buf, int nlines, int ls, int n, const StageDesc& sd,
                                              const double2* tw, bool half_out, int tid, int nth) {
  const int M = sd.M, L = sd.L, tws = sd.tws;
  const int nbf = n / R;
  const int total = nlines * nbf;
  const int nr = n / R;
  for (int u = tid; u < total; u += nth) {
    const int line = sd.div_nbf.div(u);
    const int bm = u - line * nbf;
    const int b = sd.div_M.div(bm);
    const int m = bm - b * M;
    double2* base = buf + line * ls + b * L + m;
    double2 v[R];
    v[0] = base[0];
#pragma unroll
    for (int k = 1; k < R; ++k) v[k] = (m == 0) ? base[k * M] : cmulc(base[k * M], tw[k * m * tws]);
    Bfly<R, true>::run(v, tw, nr);
    if (half_out) {
#pragma unroll
      for (int i = 0; i < R / 2; ++i) base[i * M] = v[i];
    } else {
#pragma unroll
      for (int i = 0; i < R; ++i) base[i * M] = v[i];
    }
  }
}

template <bool INV>
__device__ __forceinline__ void run_stage(double2* buf, int nlines, int ls, int n, const StageDesc& sd,
                                          const double2* tw, bool prune, int tid, int nth) {
  switch (sd.radix) {
#define VIE_CASE(R)                                                          \
  case R:                                                                    \
    if (INV) dit_stage_adj<R>(buf, nlines, ls, n, sd, tw, prune, tid, nth);  \
    else dif_stage<R>(buf, nlines, ls, n, sd, tw, prune, tid, nth);          \
    break;
    VIE_CASE(2)
    VIE_CASE(3)
    VIE_CASE(4)
    VIE_CASE(5)
    VIE_CASE(7)
    VIE_CASE(8)
#undef VIE_CASE
    default:
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
__device__ __forceinline__ void fft_forward(double2* buf, int nlines, int ls, const SmemPlan& P, bool half_in) {
  const int tid = threadIdx.x, nth = blockDim.x;
  for (int s = 0; s < P.nst; ++s) {
    run_stage<false>(buf, nlines, ls, P.n, P.st[s], P.tw, half_in && s == 0, tid, nth);
    __syncthreads();
  }
}

// Full inverse transform (digit-reversed input, natural unnormalised output).
__device__ __forceinline__ void fft_inverse(double2* buf, int nlines, int ls, const SmemPlan& P, bool half_out) {
  const int tid = threadIdx.x, nth = blockDim.x;
  for (int s = P.nst - 1; s >= 0; --s) {
    run_stage<true>(buf, nlines, ls, P.n, P.st[s], P.tw, half_out && s == 0, tid, nth);
    __syncthreads();
  }
}

}  // namespace vie
