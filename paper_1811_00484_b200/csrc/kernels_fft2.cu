// kernels_fft2.cu -- register-staged row / column FFT passes (two-stage plans).
//
// For an embedded length m = R0 * R1 (both radices in the wide register-DFT
// set) the pass needs exactly ONE shared-memory round trip:
//   forward:  global (n = m/2 real inputs, pad pruned) -> registers -> radix-R0
//             DIF stage + twiddles -> smem -> radix-R1 stage -> global at the
//             mirror-paired position of each frequency f = b + R0 k
//   inverse:  global (mirror-paired) -> registers -> adjoint radix-R1 stage ->
//             smem -> conj twiddles + adjoint radix-R0 stage -> global (crop:
//             only n of the m outputs are written)
// versus the generic multi-stage passes (kernels_fft.cu), which stage the
// whole line through smem on load, in every stage and on store.  Single-stage
// plans (m <= 24) skip shared memory entirely.
//
// Smem layout of a line: element j = k R1 + i (k < R0, i < R1) sits at
// k * R1p + i with R1p = R1 rounded up to odd, so both access patterns --
// lanes over i (first stage) and lanes over blocks k (second stage) -- are
// bank-conflict free; the line stride is odd for the column passes (lanes
// over lines).
#include "fft.cuh"
#include "kernels.cuh"

namespace vie {

namespace {

// EXT = false: the wide register-DFT set (7-smooth lengths; every production grid).
// EXT = true: the wide set plus the radices with a prime factor 11..31 (VIE_FFT_RADICES_EXT),
// a separate instantiation so the large prime DFTs never raise the register count of the
// 7-smooth passes.
template <bool EXT, class F>
__device__ __forceinline__ void radix_dispatch(int R, F&& f) {
  switch (R) {
#define VIE_CASE(RR)                          \
  case RR:                                    \
    f(std::integral_constant<int, RR>{});     \
    break;
    VIE_FFT_RADICES_WIDE(VIE_CASE)
    default:
      if constexpr (EXT) {
        switch (R) {
          VIE_FFT_RADICES_EXT(VIE_CASE)
          default:
            break;
        }
      }
      break;  // host plan selection only produces radices of the instantiated set
#undef VIE_CASE
  }
}

// first (pruned) stage: even radices only
template <bool EXT, class F>
__device__ __forceinline__ void even_dispatch(int R, F&& f) {
  switch (R) {
#define VIE_CASE(RR)                          \
  case RR:                                    \
    f(std::integral_constant<int, RR>{});     \
    break;
    VIE_CASE(2) VIE_CASE(4) VIE_CASE(6) VIE_CASE(8) VIE_CASE(10) VIE_CASE(12) VIE_CASE(16) VIE_CASE(20) VIE_CASE(24)
    default:
      if constexpr (EXT) {
        switch (R) {
          VIE_FFT_RADICES_EXT_EVEN(VIE_CASE)
          default:
            break;
        }
      }
      break;
#undef VIE_CASE
  }
}

// Forward DIF first stage of a pruned (zero-padded) line, butterfly mp:
// v_i = x[mp + i M0] (i < R/2, upper half is the pad), X_k = DFT_R(v)_k w_m^{k mp}.
template <int R, class LD, class ST>
__device__ __forceinline__ void fwd_first(int mp, const double2* __restrict__ tw, LD&& ld, ST&& st) {
  static_assert(R % 2 == 0, "pruned first stage needs an even radix");
  double2 v[R];
#pragma unroll
  for (int i = 0; i < R; ++i) v[i] = (i < R / 2) ? ld(i) : make_double2(0.0, 0.0);
  DFTs<R, false, 1, 0>::run(v);
  st(0, v[out_idx(R, 0)]);
  if (mp == 0) {
    sfor<R - 1>([&](auto kc) {
      constexpr int k = decltype(kc)::value + 1;
      st(k, v[out_idx(R, k)]);
    });
  } else {
    const double2 w1 = __ldg(tw + mp);
    double2 w = w1;
    sfor<R - 1>([&](auto kc) {
      constexpr int k = decltype(kc)::value + 1;
      st(k, cmul(v[out_idx(R, k)], w));
      if (k + 1 < R) w = cmul(w, w1);
    });
  }
}

// Plain radix-R DFT (no twiddles): the last forward stage (INV = false) or
// its adjoint, the first inverse stage (INV = true).
template <int R, bool INV, class LD, class ST>
__device__ __forceinline__ void plain_stage(LD&& ld, ST&& st) {
  double2 v[R];
#pragma unroll
  for (int i = 0; i < R; ++i) v[i] = ld(i);
  DFTs<R, INV, 1, 0>::run(v);
  sfor<R>([&](auto kc) {
    constexpr int k = decltype(kc)::value;
    st(k, v[out_idx(R, k)]);
  });
}

// Adjoint of fwd_first (last inverse stage) with the crop: v_k = X_k conj(w_m^{k mp}),
// y[mp + i M0] = IDFT_R(v)_i for i < R/2 only.
template <int R, class LD, class ST>
__device__ __forceinline__ void inv_last(int mp, const double2* __restrict__ tw, LD&& ld, ST&& st) {
  static_assert(R % 2 == 0, "pruned last stage needs an even radix");
  double2 v[R];
  v[0] = ld(0);
  if (mp == 0) {
#pragma unroll
    for (int k = 1; k < R; ++k) v[k] = ld(k);
  } else {
    const double2 w1 = __ldg(tw + mp);
    double2 w = w1;
#pragma unroll
    for (int k = 1; k < R; ++k) {
      v[k] = cmulc(ld(k), w);
      if (k + 1 < R) w = cmul(w, w1);
    }
  }
  DFTs<R, true, 1, 0>::run(v);
  sfor<R / 2>([&](auto ic) {
    constexpr int i = decltype(ic)::value;
    st(i, v[out_idx(R, i)]);
  });
}

// -------------------------------------------------------------------- rows
// Offset of (row, axis-1 position pos) in the spectral row slab A: rows of m on one GPU;
// blocked by the pencil rank q = pos / W for the slab-decomposed matvec (Geom):
// [q][row][pos - q W], blocks of nrows * W.
template <bool BLOCKED>
__device__ __forceinline__ int64_t arow(int row, int pos, int m, const FastDiv& dW, int64_t blk) {
  if constexpr (!BLOCKED) {
    return static_cast<int64_t>(row) * m + pos;
  } else {
    const int q = static_cast<int>(dW.div(static_cast<uint32_t>(pos)));
    const int W = static_cast<int>(dW.d);
    return q * blk + static_cast<int64_t>(row) * W + (pos - q * W);
  }
}

// x: rows of n (voxel order) -> A: rows of m, mirror-paired spectral positions.
template <bool BLOCKED, bool EXT>
__global__ void __launch_bounds__(256, EXT ? 1 : 2) k_row_fwd2(const double2* __restrict__ x, double2* __restrict__ A,
                                                     int nrows, Pass2 P, FastDiv dW, int64_t blk) {
  extern __shared__ double2 buf[];
  const int n = P.n, m = P.m, R0 = P.R0, R1 = P.R1;
  const int row0 = blockIdx.x * P.lines;
  const int nr = min(P.lines, nrows - row0);
  const double2* src = x + static_cast<int64_t>(row0) * n;
  if (R1 == 1) {  // single stage: no shared memory
    for (int r = threadIdx.x; r < nr; r += blockDim.x)
      even_dispatch<EXT>(R0, [&](auto rc) {
        fwd_first<decltype(rc)::value>(
            0, P.tw, [&](int i) { return src[r * n + i]; },
            [&](int k, double2 v) { A[arow<BLOCKED>(row0 + r, pos_of_freq(k, n), m, dW, blk)] = v; });
      });
    return;
  }
  const int R1p = P.R1p, ls = P.ls;
  for (int u = threadIdx.x; u < nr * R1; u += blockDim.x) {
    const int r = static_cast<int>(P.dR1.div(u)), mp = u - r * R1;
    const double2* s = src + r * n + mp;
    double2* b = buf + r * ls + mp;
    even_dispatch<EXT>(R0, [&](auto rc) {
      fwd_first<decltype(rc)::value>(
          mp, P.tw, [&](int i) { return s[i * R1]; }, [&](int k, double2 v) { b[k * R1p] = v; });
    });
  }
  __syncthreads();
  for (int u = threadIdx.x; u < nr * R0; u += blockDim.x) {
    const int r = static_cast<int>(P.dR0.div(u)), bk = u - r * R0;
    const double2* b = buf + r * ls + bk * R1p;
    radix_dispatch<EXT>(R1, [&](auto rc) {
      plain_stage<decltype(rc)::value, false>(
          [&](int i) { return b[i]; },
          [&](int k, double2 v) { A[arow<BLOCKED>(row0 + r, pos_of_freq(bk + R0 * k, n), m, dW, blk)] = v; });
    });
  }
}

// A (mirror-paired) -> y rows of n, scaled, with the apply_system epilogue.
struct RowEpi {
  double scale;
  const double2* eps;  // nullptr: plain scaled output
  const double2* xin;
  double inv_v;
  int lin, diag, rows_per_comp;
  int64_t nv;
  FastDiv drpc;
  // solver.hpp:191-198: y = eps*g*x - (eps-1)*inv_v*(N x)
  __device__ __forceinline__ double2 operator()(double2 v, int row, int i, int n) const {
    v = cscale(v, scale);
    if (eps == nullptr) return v;
    const int t = static_cast<int>(drpc.div(row));
    const int64_t vox = static_cast<int64_t>(row - t * rows_per_comp) * n + i;
    const double2 ep = eps[vox];
    const double2 chv = make_double2((ep.x - 1.0) * inv_v, ep.y * inv_v);
    double2 out = make_double2(0.0, 0.0);
    if (diag) {
      const double g = (lin && (t & 3)) ? (1.0 / 12.0) : 1.0;
      out = cmul(lin ? cscale(ep, g) : ep, xin[static_cast<int64_t>(t) * nv + vox]);
    }
    return csub(out, cmul(chv, v));
  }
};

template <bool BLOCKED, bool EXT>
__global__ void __launch_bounds__(256, EXT ? 1 : 2) k_row_inv2(const double2* __restrict__ A, double2* __restrict__ y,
                                                     int nrows, Pass2 P, RowEpi epi, FastDiv dW, int64_t blk) {
  extern __shared__ double2 buf[];
  const int n = P.n, m = P.m, R0 = P.R0, R1 = P.R1;
  const int row0 = blockIdx.x * P.lines;
  const int nr = min(P.lines, nrows - row0);
  double2* dst = y + static_cast<int64_t>(row0) * n;
  if (R1 == 1) {
    for (int r = threadIdx.x; r < nr; r += blockDim.x)
      even_dispatch<EXT>(R0, [&](auto rc) {
        inv_last<decltype(rc)::value>(
            0, P.tw, [&](int k) { return A[arow<BLOCKED>(row0 + r, pos_of_freq(k, n), m, dW, blk)]; },
            [&](int i, double2 v) { dst[r * n + i] = epi(v, row0 + r, i, n); });
      });
    return;
  }
  const int R1p = P.R1p, ls = P.ls;
  for (int u = threadIdx.x; u < nr * R0; u += blockDim.x) {
    const int r = static_cast<int>(P.dR0.div(u)), bk = u - r * R0;
    double2* b = buf + r * ls + bk * R1p;
    radix_dispatch<EXT>(R1, [&](auto rc) {
      plain_stage<decltype(rc)::value, true>(
          [&](int k) { return A[arow<BLOCKED>(row0 + r, pos_of_freq(bk + R0 * k, n), m, dW, blk)]; },
          [&](int i, double2 v) { b[i] = v; });
    });
  }
  __syncthreads();
  for (int u = threadIdx.x; u < nr * R1; u += blockDim.x) {
    const int r = static_cast<int>(P.dR1.div(u)), mp = u - r * R1;
    const double2* b = buf + r * ls + mp;
    double2* d = dst + r * n + mp;
    even_dispatch<EXT>(R0, [&](auto rc) {
      inv_last<decltype(rc)::value>(
          mp, P.tw, [&](int k) { return b[k * R1p]; },
          [&](int i, double2 v) { d[i * R1] = epi(v, row0 + r, mp + i * R1, n); });
    });
  }
}

// -------------------------------------------------------------------- columns
// A: planes of n2 rows x m1 -> B: planes of m2 rows x m1 (mirror-paired rows);
// kColsPerCta consecutive columns per CTA, lanes over columns (128 B segments).
constexpr int kCW = kColsPerCta;
static_assert((kCW & (kCW - 1)) == 0, "column tile must be a power of two");
constexpr int kLgCW = kCW == 8 ? 3 : (kCW == 4 ? 2 : (kCW == 16 ? 4 : 0));

template <bool EXT>
__global__ void __launch_bounds__(256, EXT ? 1 : 2) k_col_fwd2(const double2* __restrict__ A, double2* __restrict__ B, int m1,
                                                     Pass2 P, int64_t bps, PlaneMap pm) {
  extern __shared__ double2 buf[];
  const int n = P.n, R0 = P.R0, R1 = P.R1;
  const int c0 = blockIdx.x * kCW;
  const int wc = min(kCW, m1 - c0);
  const int64_t plane = blockIdx.y;
  const double2* src = A + plane * n * m1 + c0;
  double2* dst = B + pm(static_cast<int>(plane)) * bps + c0;
  if (R1 == 1) {
    const int w = threadIdx.x;
    if (w < wc)
      even_dispatch<EXT>(R0, [&](auto rc) {
        fwd_first<decltype(rc)::value>(
            0, P.tw, [&](int i) { return src[static_cast<int64_t>(i) * m1 + w]; },
            [&](int k, double2 v) { dst[static_cast<int64_t>(pos_of_freq(k, n)) * m1 + w] = v; });
      });
    return;
  }
  const int R1p = P.R1p, ls = P.ls;
  for (int u = threadIdx.x; u < kCW * R1; u += blockDim.x) {
    const int w = u & (kCW - 1), mp = u >> kLgCW;
    if (w >= wc) continue;
    const double2* s = src + static_cast<int64_t>(mp) * m1 + w;
    double2* b = buf + w * ls + mp;
    const int64_t step = static_cast<int64_t>(R1) * m1;
    even_dispatch<EXT>(R0, [&](auto rc) {
      fwd_first<decltype(rc)::value>(
          mp, P.tw, [&](int i) { return s[i * step]; }, [&](int k, double2 v) { b[k * R1p] = v; });
    });
  }
  __syncthreads();
  for (int u = threadIdx.x; u < kCW * R0; u += blockDim.x) {
    const int w = u & (kCW - 1), bk = u >> kLgCW;
    if (w >= wc) continue;
    const double2* b = buf + w * ls + bk * R1p;
    double2* d = dst + w;
    radix_dispatch<EXT>(R1, [&](auto rc) {
      plain_stage<decltype(rc)::value, false>(
          [&](int i) { return b[i]; },
          [&](int k, double2 v) { d[static_cast<int64_t>(pos_of_freq(bk + R0 * k, n)) * m1] = v; });
    });
  }
}

template <bool EXT>
__global__ void __launch_bounds__(256, EXT ? 1 : 2) k_col_inv2(const double2* __restrict__ B, double2* __restrict__ A, int m1,
                                                     Pass2 P, int64_t bps, PlaneMap pm) {
  extern __shared__ double2 buf[];
  const int n = P.n, R0 = P.R0, R1 = P.R1;
  const int c0 = blockIdx.x * kCW;
  const int wc = min(kCW, m1 - c0);
  const int64_t plane = blockIdx.y;
  const double2* src = B + pm(static_cast<int>(plane)) * bps + c0;
  double2* dst = A + plane * n * m1 + c0;
  if (R1 == 1) {
    const int w = threadIdx.x;
    if (w < wc)
      even_dispatch<EXT>(R0, [&](auto rc) {
        inv_last<decltype(rc)::value>(
            0, P.tw, [&](int k) { return src[static_cast<int64_t>(pos_of_freq(k, n)) * m1 + w]; },
            [&](int i, double2 v) { dst[static_cast<int64_t>(i) * m1 + w] = v; });
      });
    return;
  }
  const int R1p = P.R1p, ls = P.ls;
  for (int u = threadIdx.x; u < kCW * R0; u += blockDim.x) {
    const int w = u & (kCW - 1), bk = u >> kLgCW;
    if (w >= wc) continue;
    const double2* s = src + w;
    double2* b = buf + w * ls + bk * R1p;
    radix_dispatch<EXT>(R1, [&](auto rc) {
      plain_stage<decltype(rc)::value, true>(
          [&](int k) { return s[static_cast<int64_t>(pos_of_freq(bk + R0 * k, n)) * m1]; },
          [&](int i, double2 v) { b[i] = v; });
    });
  }
  __syncthreads();
  for (int u = threadIdx.x; u < kCW * R1; u += blockDim.x) {
    const int w = u & (kCW - 1), mp = u >> kLgCW;
    if (w >= wc) continue;
    const double2* b = buf + w * ls + mp;
    double2* d = dst + static_cast<int64_t>(mp) * m1 + w;
    const int64_t step = static_cast<int64_t>(R1) * m1;
    even_dispatch<EXT>(R0, [&](auto rc) {
      inv_last<decltype(rc)::value>(
          mp, P.tw, [&](int k) { return b[k * R1p]; }, [&](int i, double2 v) { d[i * step] = v; });
    });
  }
}

int round_threads(int t) { return std::max(32, std::min(256, (t + 31) / 32 * 32)); }

size_t pass2_smem(const Pass2& P, int lines) {
  return P.R1 == 1 ? 0 : sizeof(double2) * static_cast<size_t>(lines) * P.ls;
}

void set_smem2(const void* fn, size_t bytes) {
  VIE_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
}

}  // namespace

bool pass2_init(Pass2& P, int m, const int* radices, int nst, const double2* tw, int row_lines) {
  if (nst < 1 || nst > 2 || (m & 1)) return false;
  const int R0 = radices[0], R1 = nst == 2 ? radices[1] : 1;
  if (R0 & 1) return false;  // pad / crop pruning needs an even first radix
  P.m = m;
  P.n = m / 2;
  P.R0 = R0;
  P.R1 = R1;
  P.R1p = R1 | 1;
  auto wide = [](int r) {
    switch (r) {
#define VIE_CASE(RR) case RR:
      VIE_FFT_RADICES_WIDE(VIE_CASE)
#undef VIE_CASE
      return true;
      default:
        return r == 1;
    }
  };
  P.ext = !(wide(R0) && wide(R1));
  P.ls = (R0 * P.R1p) | 1;
  P.tw = tw;
  P.dR0.init(static_cast<uint32_t>(R0));
  P.dR1.init(static_cast<uint32_t>(R1));
  const int widest = std::max(R0, R1);
  P.lines = R1 == 1 ? 64 : std::max(1, (row_lines > 0 ? row_lines : 120 / widest));  // 6 rows at m = 400 (measured best)
  return true;
}

template <bool BLOCKED, bool EXT>
void row_fwd2_t(const double2* x, double2* A, int nrows, const Pass2& P, const FastDiv& dW, int64_t blk, size_t sm,
                int threads, cudaStream_t st) {
  if (sm) set_smem2(reinterpret_cast<const void*>(k_row_fwd2<BLOCKED, EXT>), sm);
  k_row_fwd2<BLOCKED, EXT><<<(nrows + P.lines - 1) / P.lines, threads, sm, st>>>(x, A, nrows, P, dW, blk);
}

template <bool BLOCKED, bool EXT>
void row_inv2_t(const double2* A, double2* y, int nrows, const Pass2& P, const RowEpi& epi, const FastDiv& dW,
                int64_t blk, size_t sm, int threads, cudaStream_t st) {
  if (sm) set_smem2(reinterpret_cast<const void*>(k_row_inv2<BLOCKED, EXT>), sm);
  k_row_inv2<BLOCKED, EXT><<<(nrows + P.lines - 1) / P.lines, threads, sm, st>>>(A, y, nrows, P, epi, dW, blk);
}

void launch_row_fwd2(const double2* x, double2* A, const Geom& g, const Pass2& P, cudaStream_t st) {
  const int nrows = g.S * g.n2 * g.n3;
  const size_t sm = pass2_smem(P, P.lines);
  const int threads = round_threads(P.R1 == 1 ? P.lines : P.lines * std::max(P.R0, P.R1));
  FastDiv dW;
  dW.init(static_cast<uint32_t>(g.W));
  const int64_t blk = static_cast<int64_t>(nrows) * g.W;
  const bool blocked = g.W != g.m1;
  if (P.ext) {
    if (blocked) row_fwd2_t<true, true>(x, A, nrows, P, dW, blk, sm, threads, st);
    else row_fwd2_t<false, true>(x, A, nrows, P, dW, blk, sm, threads, st);
  } else {
    if (blocked) row_fwd2_t<true, false>(x, A, nrows, P, dW, blk, sm, threads, st);
    else row_fwd2_t<false, false>(x, A, nrows, P, dW, blk, sm, threads, st);
  }
  VIE_CUDA_CHECK(cudaGetLastError());
}

void launch_row_inv2(const double2* A, double2* y, const Geom& g, const Pass2& P, double scale, const double2* eps,
                     const double2* xin, double inv_v, int basis, int diag, cudaStream_t st) {
  const int nrows = g.S * g.n2 * g.n3;
  const size_t sm = pass2_smem(P, P.lines);
  RowEpi epi{scale, eps, xin, inv_v, basis == 1 ? 1 : 0, diag, g.n2 * g.n3,
             static_cast<int64_t>(g.n1) * g.n2 * g.n3, {}};
  epi.drpc.init(static_cast<uint32_t>(g.n2 * g.n3));
  const int threads = round_threads(P.R1 == 1 ? P.lines : P.lines * std::max(P.R0, P.R1));
  FastDiv dW;
  dW.init(static_cast<uint32_t>(g.W));
  const int64_t blk = static_cast<int64_t>(nrows) * g.W;
  const bool blocked = g.W != g.m1;
  if (P.ext) {
    if (blocked) row_inv2_t<true, true>(A, y, nrows, P, epi, dW, blk, sm, threads, st);
    else row_inv2_t<false, true>(A, y, nrows, P, epi, dW, blk, sm, threads, st);
  } else {
    if (blocked) row_inv2_t<true, false>(A, y, nrows, P, epi, dW, blk, sm, threads, st);
    else row_inv2_t<false, false>(A, y, nrows, P, epi, dW, blk, sm, threads, st);
  }
  VIE_CUDA_CHECK(cudaGetLastError());
}

// Column passes over the S * nk planes of a Geom, rows of length W (= m1 on one GPU;
// the rank's axis-1 positions in the slab-decomposed pencil stage).
void launch_col_fwd2(const double2* A, double2* B, const Geom& g, const Pass2& P, cudaStream_t st, PlaneMap pm) {
  const size_t sm = pass2_smem(P, kCW);
  dim3 grid((g.W + kCW - 1) / kCW, g.S * g.nk);
  const int threads = round_threads(P.R1 == 1 ? kCW : kCW * std::max(P.R0, P.R1));
  auto fn = P.ext ? k_col_fwd2<true> : k_col_fwd2<false>;
  if (sm) set_smem2(reinterpret_cast<const void*>(fn), sm);
  fn<<<grid, threads, sm, st>>>(A, B, g.W, P, g.bps, pm);
  VIE_CUDA_CHECK(cudaGetLastError());
}

void launch_col_inv2(const double2* B, double2* A, const Geom& g, const Pass2& P, cudaStream_t st, PlaneMap pm) {
  const size_t sm = pass2_smem(P, kCW);
  dim3 grid((g.W + kCW - 1) / kCW, g.S * g.nk);
  const int threads = round_threads(P.R1 == 1 ? kCW : kCW * std::max(P.R0, P.R1));
  auto fn = P.ext ? k_col_inv2<true> : k_col_inv2<false>;
  if (sm) set_smem2(reinterpret_cast<const void*>(fn), sm);
  fn<<<grid, threads, sm, st>>>(B, A, g.W, P, g.bps, pm);
  VIE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace vie
