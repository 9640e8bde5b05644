// kernels_blas.cu -- GMRES BLAS-1 (solver.hpp:75-80, 120, 130) as streaming
// kernels with deterministic two-level reductions: each CTA writes a partial,
// the last CTA to finish (atomic ticket) sums the partials in index order.
// The modified Gram-Schmidt step is fused: w -= h_i v_i and the next
// coefficient h_{i+1} = <v_{i+1}, w> (or ||w||^2) in one pass over w.
#include "kernels.cuh"

namespace vie {

namespace {

__device__ __forceinline__ double2 warp_sum(double2 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// Block reduction + last-block finalisation into out[0].
__device__ __forceinline__ void reduce_finish(double2 v, RedBuf rb, double2* out) {
  __shared__ double2 ws[kThreads / 32];
  __shared__ bool last;
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) ws[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double2 s = lane < (int)(blockDim.x / 32) ? ws[lane] : make_double2(0.0, 0.0);
    s = warp_sum(s);
    if (lane == 0) {
      rb.partials[blockIdx.x] = s;
      __threadfence();
      const unsigned int ticket = atomicAdd(rb.counter, 1u);
      last = (ticket == gridDim.x - 1);
    }
  }
  __syncthreads();
  if (last && wid == 0) {
    __threadfence();
    double2 s = make_double2(0.0, 0.0);
    for (int i = lane; i < (int)gridDim.x; i += 32) {
      const volatile double* p = reinterpret_cast<volatile double*>(&rb.partials[i]);
      s.x += p[0];
      s.y += p[1];
    }
    s = warp_sum(s);
    if (lane == 0) {
      out[0] = s;
      *rb.counter = 0u;
    }
  }
}

__global__ void __launch_bounds__(kThreads) k_dot(const double2* __restrict__ a, const double2* __restrict__ b,
                                                  int64_t n, double2* out, RedBuf rb) {
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 x = a[i], y = b[i];
    acc.x = fma(x.x, y.x, fma(x.y, y.y, acc.x));
    acc.y = fma(x.x, y.y, fma(-x.y, y.x, acc.y));
  }
  reduce_finish(acc, rb, out);
}

__global__ void __launch_bounds__(kThreads) k_nrm2sq(const double2* __restrict__ a, int64_t n, double2* out,
                                                     RedBuf rb) {
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 x = a[i];
    acc.x = fma(x.x, x.x, fma(x.y, x.y, acc.x));
  }
  reduce_finish(acc, rb, out);
}

__global__ void __launch_bounds__(kThreads) k_mgs_step(double2* __restrict__ w, const double2* __restrict__ v,
                                                       const double2* __restrict__ h,
                                                       const double2* __restrict__ vnext, int64_t n, double2* out,
                                                       RedBuf rb) {
  const double2 hh = h[0];
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 x = w[i];
    cfms(x, hh, v[i]);
    w[i] = x;
    if (vnext) {
      const double2 y = vnext[i];  // conj(y) * x
      acc.x = fma(y.x, x.x, fma(y.y, x.y, acc.x));
      acc.y = fma(y.x, x.y, fma(-y.y, x.x, acc.y));
    } else {
      acc.x = fma(x.x, x.x, fma(x.y, x.y, acc.x));
    }
  }
  reduce_finish(acc, rb, out);
}

__global__ void __launch_bounds__(kThreads) k_residual(const double2* __restrict__ rhs, const double2* __restrict__ ax,
                                                       double2* __restrict__ r, int64_t n, double2* out, RedBuf rb) {
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 x = csub(rhs[i], ax[i]);
    if (r) r[i] = x;
    acc.x = fma(x.x, x.x, fma(x.y, x.y, acc.x));
  }
  reduce_finish(acc, rb, out);
}

__global__ void k_scale_inv(const double2* __restrict__ x, double2* __restrict__ y, const double2* __restrict__ s,
                            double divisor, int64_t n) {
  // reference divides (basis.col(0) = r / beta; w / wnorm), solver.hpp:67, :120
  const double d = s ? s[0].x : divisor;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = x[i];
    y[i] = make_double2(v.x / d, v.y / d);
  }
}

__global__ void k_basis_update(double2* __restrict__ x, const double2* __restrict__ V, int64_t ldv,
                               const double2* __restrict__ coef, int j, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int l = 0; l < j; ++l) cfma(acc, V[l * ldv + i], coef[l]);
    x[i] = cadd(x[i], acc);
  }
}

__global__ void k_axpy1(double2* __restrict__ x, const double2* __restrict__ z, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = cadd(x[i], z[i]);
}

__global__ void k_cmul_elem(const double2* __restrict__ d, const double2* __restrict__ in, double2* __restrict__ out,
                            int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = cmul(d[i], in[i]);
}

}  // namespace

void launch_axpy1(double2* x, const double2* z, int64_t n, cudaStream_t st) {
  k_axpy1<<<kRedBlocks, kThreads, 0, st>>>(x, z, n);
  VIE_CUDA_CHECK(cudaGetLastError());
}
void launch_cmul_elem(const double2* d, const double2* in, double2* out, int64_t n, cudaStream_t st) {
  k_cmul_elem<<<kRedBlocks, kThreads, 0, st>>>(d, in, out, n);
  VIE_CUDA_CHECK(cudaGetLastError());
}

void launch_dot(const double2* a, const double2* b, int64_t n, double2* out, RedBuf rb, cudaStream_t st) {
  k_dot<<<kRedBlocks, kThreads, 0, st>>>(a, b, n, out, rb);
  VIE_CUDA_CHECK(cudaGetLastError());
}
void launch_nrm2sq(const double2* a, int64_t n, double2* out, RedBuf rb, cudaStream_t st) {
  k_nrm2sq<<<kRedBlocks, kThreads, 0, st>>>(a, n, out, rb);
  VIE_CUDA_CHECK(cudaGetLastError());
}
void launch_mgs_step(double2* w, const double2* v, const double2* h, const double2* vnext, int64_t n, double2* out,
                     RedBuf rb, cudaStream_t st) {
  k_mgs_step<<<kRedBlocks, kThreads, 0, st>>>(w, v, h, vnext, n, out, rb);
  VIE_CUDA_CHECK(cudaGetLastError());
}
void launch_residual(const double2* rhs, const double2* ax, double2* r, int64_t n, double2* out, RedBuf rb,
                     cudaStream_t st) {
  k_residual<<<kRedBlocks, kThreads, 0, st>>>(rhs, ax, r, n, out, rb);
  VIE_CUDA_CHECK(cudaGetLastError());
}
void launch_scale_inv(const double2* x, double2* y, const double2* s, double scalar, int64_t n, cudaStream_t st) {
  k_scale_inv<<<kRedBlocks, kThreads, 0, st>>>(x, y, s, scalar, n);
  VIE_CUDA_CHECK(cudaGetLastError());
}
void launch_basis_update(double2* x, const double2* V, int64_t ldv, const double2* coef, int j, int64_t n,
                         cudaStream_t st) {
  k_basis_update<<<kRedBlocks, kThreads, 0, st>>>(x, V, ldv, coef, j, n);
  VIE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace vie
