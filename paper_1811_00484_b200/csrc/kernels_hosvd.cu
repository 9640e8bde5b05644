// kernels_hosvd.cu -- device parts of tucker_compress (hosvd, decomp.hpp:160-176):
// unfolding Gram matrices G_q = M_q M_q^H (tensor.hpp:81-98 unfoldings) and the
// core projection core = t x1 U1^H x2 U2^H x3 U3^H (decomp.hpp:171-174).
#include "kernels.cuh"

namespace vie {

namespace {

// element (i, col) of the mode-q unfolding, reference column order
__device__ __forceinline__ int64_t unfold_index(int mode, int64_t i, int64_t col, int64_t n1, int64_t n2) {
  if (mode == 1) return i + n1 * col;                       // M(i, j + n2 k)
  if (mode == 2) return (col % n1) + n1 * (i + n2 * (col / n1));  // M(j, i + n1 k)
  return col + n1 * n2 * i;                                  // M(k, i + n1 j)
}

constexpr int kGT = 16;  // Gram tile
constexpr int kGC = 32;  // columns per smem chunk

__global__ void __launch_bounds__(kGT* kGT) k_gram(const double2* __restrict__ t, int64_t n1, int64_t n2,
                                                   int64_t n3, int mode, int nq, double2* __restrict__ G) {
  __shared__ double2 ma[kGT][kGC + 1], mb[kGT][kGC + 1];
  const int64_t ncols = n1 * n2 * n3 / nq;
  const int i0 = blockIdx.x * kGT, j0 = blockIdx.y * kGT;
  const int ti = threadIdx.x / kGT, tj = threadIdx.x % kGT;
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t c0 = 0; c0 < ncols; c0 += kGC) {
    for (int e = threadIdx.x; e < kGT * kGC; e += blockDim.x) {
      const int r = e / kGC, c = e % kGC;
      const int64_t col = c0 + c;
      const bool okc = col < ncols;
      ma[r][c] = (okc && i0 + r < nq) ? t[unfold_index(mode, i0 + r, col, n1, n2)] : make_double2(0.0, 0.0);
      mb[r][c] = (okc && j0 + r < nq) ? t[unfold_index(mode, j0 + r, col, n1, n2)] : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll 8
    for (int c = 0; c < kGC; ++c) {
      const double2 x = ma[ti][c], y = mb[tj][c];  // x * conj(y)
      acc.x = fma(x.x, y.x, fma(x.y, y.y, acc.x));
      acc.y = fma(x.y, y.x, fma(-x.x, y.y, acc.y));
    }
    __syncthreads();
  }
  if (i0 + ti < nq && j0 + tj < nq) G[(i0 + ti) + static_cast<int64_t>(nq) * (j0 + tj)] = acc;
}

// out = in x_q U^H : dims d (in) -> d with d_q replaced by r; U is n_q x r col-major
__global__ void k_mode_product_h(const double2* __restrict__ in, int64_t d1, int64_t d2, int64_t d3, int mode,
                                 const double2* __restrict__ U, int r, double2* __restrict__ out) {
  const int64_t o1 = mode == 1 ? r : d1, o2 = mode == 2 ? r : d2, o3 = mode == 3 ? r : d3;
  const int64_t total = o1 * o2 * o3;
  const int64_t nq = mode == 1 ? d1 : (mode == 2 ? d2 : d3);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t a = e % o1, rest = e / o1, b = rest % o2, c = rest / o2;
    const int64_t oq = mode == 1 ? a : (mode == 2 ? b : c);
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t i = 0; i < nq; ++i) {
      const int64_t ia = mode == 1 ? i : a, ib = mode == 2 ? i : b, ic = mode == 3 ? i : c;
      const double2 v = in[ia + d1 * (ib + d2 * ic)];
      const double2 u = U[i + nq * oq];  // conj(u) * v
      acc.x = fma(u.x, v.x, fma(u.y, v.y, acc.x));
      acc.y = fma(u.x, v.y, fma(-u.y, v.x, acc.y));
    }
    out[e] = acc;
  }
}

// sum |a - b|^2 (b may be null) into *acc (one double, zeroed by the caller)
__global__ void k_diff_norm2(const double2* __restrict__ a, const double2* __restrict__ b, int64_t n,
                             double* __restrict__ acc) {
  double s = 0.0;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double2 v = a[e];
    if (b) {
      v.x -= b[e].x;
      v.y -= b[e].y;
    }
    s = fma(v.x, v.x, fma(v.y, v.y, s));
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ double ws[8];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += ws[w];
    atomicAdd(acc, t);
  }
}

// sum |t - cp(W1, W2, W3)|^2, cp(i,j,k) = sum_l W1(i,l) W2(j,l) W3(k,l) (tensor.hpp:157-168)
__global__ void k_cp_residual2(const double2* __restrict__ t, int64_t n1, int64_t n2, int64_t n3,
                               const double2* __restrict__ w1, const double2* __restrict__ w2,
                               const double2* __restrict__ w3, int R, double* __restrict__ acc) {
  double s = 0.0;
  const int64_t n = n1 * n2 * n3;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e % n1, j = (e / n1) % n2, k = e / (n1 * n2);
    double2 rec = make_double2(0.0, 0.0);
    for (int l = 0; l < R; ++l) {
      const double2 p = cmul(w1[i + n1 * l], w2[j + n2 * l]);
      rec = cadd(rec, cmul(p, w3[k + n3 * l]));
    }
    const double dx = t[e].x - rec.x, dy = t[e].y - rec.y;
    s = fma(dx, dx, fma(dy, dy, s));
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ double ws[8];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tt = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) tt += ws[w];
    atomicAdd(acc, tt);
  }
}

}  // namespace

void launch_gram(const double2* t, const int64_t dims[3], int mode, double2* G, cudaStream_t st) {
  const int nq = static_cast<int>(dims[mode - 1]);
  dim3 grid((nq + kGT - 1) / kGT, (nq + kGT - 1) / kGT);
  k_gram<<<grid, kGT * kGT, 0, st>>>(t, dims[0], dims[1], dims[2], mode, nq, G);
  VIE_CUDA_CHECK(cudaGetLastError());
}

void launch_mode_product_h(const double2* in, const int64_t dims[3], int mode, const double2* U, int r,
                           double2* out, cudaStream_t st) {
  const int64_t total = (mode == 1 ? r : dims[0]) * (mode == 2 ? r : dims[1]) * (mode == 3 ? r : dims[2]);
  const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  k_mode_product_h<<<std::max(blocks, 1), 256, 0, st>>>(in, dims[0], dims[1], dims[2], mode, U, r, out);
  VIE_CUDA_CHECK(cudaGetLastError());
}

void launch_diff_norm2(const double2* a, const double2* b, int64_t n, double* acc, cudaStream_t st) {
  const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 8));
  k_diff_norm2<<<std::max(blocks, 1), 256, 0, st>>>(a, b, n, acc);
  VIE_CUDA_CHECK(cudaGetLastError());
}

void launch_cp_residual2(const double2* t, const int64_t dims[3], const double2* w1, const double2* w2,
                         const double2* w3, int R, double* acc, cudaStream_t st) {
  const int64_t n = dims[0] * dims[1] * dims[2];
  const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 8));
  k_cp_residual2<<<std::max(blocks, 1), 256, 0, st>>>(t, dims[0], dims[1], dims[2], w1, w2, w3, R, acc);
  VIE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace vie
