// kernels_fft.cu -- padded/cropped FFT passes of the matvec pipeline.
//
// Data flow: x --row FFT (axis 1, pad)--> A --column FFT (axis 2,
// pad)--> B --pencil kernel (axis 3 FFT, Hadamard, IFFT, crop)--> B --column
// IFFT (axis 2, crop)--> A --row IFFT (axis 1, crop, 1/N_e, system epilogue)--> y.
// Spectral axes 1 and 2 are stored in mirror-paired order (common.cuh) so that
// the octant partners p and m-p sit next to each other for the pencil kernel.
#include "fft.cuh"
#include "kernels.cuh"

namespace vie {

namespace {

// smem carve-up: [plan tables][lines]
__host__ __device__ __forceinline__ int line_stride(int n) { return n + 1; }

// global -> shared 16-byte copies without register staging (full MLP)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// -------------------------------------------------------------------- rows
__global__ void __launch_bounds__(kThreads, 2) k_row_fwd(const double2* __restrict__ x, double2* __restrict__ A,
                                                      int n1, int nrows, FftPlan P, FastDiv dn1, FastDiv dm) {
  extern __shared__ double2 sm[];
  const int m = P.n;
  const SmemPlan SP = load_plan(sm, P);
  const int* slot_s = SP.slot;
  double2* buf = sm + plan_smem_elems(m);
  const int ls = line_stride(m);
  const int row0 = blockIdx.x * kRowsPerCta;
  const int nr = min(kRowsPerCta, nrows - row0);
  const double2* src = x + static_cast<int64_t>(row0) * n1;
  for (int e = threadIdx.x; e < nr * n1; e += blockDim.x) {
    const int r = static_cast<int>(dn1.div(e)), i = e - r * n1;
    cp_async16(buf + r * ls + i, src + e);
  }
  cp_async_wait();
  __syncthreads();
  fft_forward<true>(buf, nr, ls, SP, true);
  double2* dst = A + static_cast<int64_t>(row0) * m;
  for (int e = threadIdx.x; e < nr * m; e += blockDim.x) {
    const int r = static_cast<int>(dm.div(e)), pos = e - r * m;
    dst[e] = buf[r * ls + slot_s[freq_of_pos(pos, n1)]];
  }
}

__global__ void __launch_bounds__(kThreads, 2) k_row_inv(const double2* __restrict__ A, double2* __restrict__ y,
                                                      int n1, int nrows, int rows_per_comp, int64_t nv, FftPlan P,
                                                      double scale, const double2* __restrict__ eps,
                                                      const double2* __restrict__ xin, double inv_v, int lin,
                                                      int diag, FastDiv dn1, FastDiv dm, FastDiv drpc) {
  extern __shared__ double2 sm[];
  const int m = P.n;
  const SmemPlan SP = load_plan(sm, P);
  const int* slot_s = SP.slot;
  double2* buf = sm + plan_smem_elems(m);
  const int ls = line_stride(m);
  __syncthreads();
  const int row0 = blockIdx.x * kRowsPerCta;
  const int nr = min(kRowsPerCta, nrows - row0);
  const double2* src = A + static_cast<int64_t>(row0) * m;
  for (int e = threadIdx.x; e < nr * m; e += blockDim.x) {
    const int r = static_cast<int>(dm.div(e)), pos = e - r * m;
    cp_async16(buf + r * ls + slot_s[freq_of_pos(pos, n1)], src + e);
  }
  cp_async_wait();
  __syncthreads();
  fft_inverse<true>(buf, nr, ls, SP, true);
  double2* dst = y + static_cast<int64_t>(row0) * n1;
  for (int e = threadIdx.x; e < nr * n1; e += blockDim.x) {
    const int r = static_cast<int>(dn1.div(e)), i = e - r * n1;
    const double2 v = cscale(buf[r * ls + i], scale);
    if (eps == nullptr) {
      dst[e] = v;
    } else {
      // apply_system (solver.hpp:191-198): y = eps*x - chi*inv_v*nx
      const int row = row0 + r;
      const int t = static_cast<int>(drpc.div(row));
      const int64_t vox = static_cast<int64_t>(row - t * rows_per_comp) * n1 + i;
      const double2 ep = eps[vox];
      const double2 chv = make_double2((ep.x - 1.0) * inv_v, ep.y * inv_v);
      double2 out = make_double2(0.0, 0.0);
      if (diag) {
        const double g = (lin && (t & 3)) ? (1.0 / 12.0) : 1.0;
        const double2 eg = lin ? cscale(ep, g) : ep;
        out = cmul(eg, xin[static_cast<int64_t>(t) * nv + vox]);
      }
      dst[e] = csub(out, cmul(chv, v));
    }
  }
}

// -------------------------------------------------------------------- columns
// A: planes of n2 rows x m1 (row-major, column index fastest) -> B: planes of
// m2 rows x m1; W consecutive columns per CTA.
__global__ void __launch_bounds__(kThreads, 3) k_col_fwd(const double2* __restrict__ A, double2* __restrict__ B,
                                                      int n2, int m1, FftPlan P, int64_t bps) {
  extern __shared__ double2 sm[];
  const int m = P.n;
  const SmemPlan SP = load_plan(sm, P);
  const int* slot_s = SP.slot;
  double2* buf = sm + plan_smem_elems(m);
  const int ls = line_stride(m);
  const int c0 = blockIdx.x * kColsPerCta;
  const int wc = min(kColsPerCta, m1 - c0);
  const int64_t plane = blockIdx.y;
  const double2* src = A + plane * n2 * m1 + c0;
  for (int e = threadIdx.x; e < n2 * kColsPerCta; e += blockDim.x) {
    const int j = e / kColsPerCta, w = e - j * kColsPerCta;
    if (w < wc) cp_async16(buf + w * ls + j, src + static_cast<int64_t>(j) * m1 + w);
  }
  cp_async_wait();
  __syncthreads();
  fft_forward(buf, wc, ls, SP, true);
  double2* dst = B + plane * bps + c0;
  for (int e = threadIdx.x; e < m * kColsPerCta; e += blockDim.x) {
    const int pos = e / kColsPerCta, w = e - pos * kColsPerCta;
    if (w < wc) dst[static_cast<int64_t>(pos) * m1 + w] = buf[w * ls + slot_s[freq_of_pos(pos, n2)]];
  }
}

__global__ void __launch_bounds__(kThreads, 3) k_col_inv(const double2* __restrict__ B,
                                                         const double2* __restrict__ B1, double2* __restrict__ A,
                                                         int n2, int m1, FftPlan P, int64_t bps) {
  extern __shared__ double2 sm[];
  const int m = P.n;
  const SmemPlan SP = load_plan(sm, P);
  const int* slot_s = SP.slot;
  double2* buf = sm + plan_smem_elems(m);
  const int ls = line_stride(m);
  __syncthreads();
  const int c0 = blockIdx.x * kColsPerCta;
  const int wc = min(kColsPerCta, m1 - c0);
  const int64_t plane = blockIdx.y;
  const double2* src = B + plane * bps + c0;
  for (int e = threadIdx.x; e < m * kColsPerCta; e += blockDim.x) {
    const int pos = e / kColsPerCta, w = e - pos * kColsPerCta;
    if (w < wc) cp_async16(buf + w * ls + slot_s[freq_of_pos(pos, n2)], src + static_cast<int64_t>(pos) * m1 + w);
  }
  cp_async_wait();
  if (B1) {  // add the second slab (same element mapping: each thread owns its cp.async targets)
    const double2* src1 = B1 + plane * bps + c0;
    for (int e = threadIdx.x; e < m * kColsPerCta; e += blockDim.x) {
      const int pos = e / kColsPerCta, w = e - pos * kColsPerCta;
      if (w < wc) {
        double2* d = buf + w * ls + slot_s[freq_of_pos(pos, n2)];
        *d = cadd(*d, src1[static_cast<int64_t>(pos) * m1 + w]);
      }
    }
  }
  __syncthreads();
  fft_inverse(buf, wc, ls, SP, true);
  double2* dst = A + plane * n2 * m1 + c0;
  for (int e = threadIdx.x; e < n2 * kColsPerCta; e += blockDim.x) {
    const int j = e / kColsPerCta, w = e - j * kColsPerCta;
    if (w < wc) dst[static_cast<int64_t>(j) * m1 + w] = buf[w * ls + j];
  }
}

}  // namespace

size_t row_smem(int m) {
  return sizeof(double2) * (static_cast<size_t>(plan_smem_elems(m)) + static_cast<size_t>(kRowsPerCta) * line_stride(m));
}
size_t col_smem(int m) {
  return sizeof(double2) * (static_cast<size_t>(plan_smem_elems(m)) + static_cast<size_t>(kColsPerCta) * line_stride(m));
}

static void set_smem(const void* fn, size_t bytes) {
  VIE_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
}

void launch_row_fwd(const double2* x, double2* A, const Geom& g, const FftPlan& P1, cudaStream_t st) {
  const int nrows = g.S * g.n2 * g.n3;
  const size_t sm = row_smem(g.m1);
  set_smem(reinterpret_cast<const void*>(k_row_fwd), sm);
  FastDiv dn1, dm;
  dn1.init(static_cast<uint32_t>(g.n1));
  dm.init(static_cast<uint32_t>(g.m1));
  k_row_fwd<<<(nrows + kRowsPerCta - 1) / kRowsPerCta, kThreads, sm, st>>>(x, A, g.n1, nrows, P1, dn1, dm);
  VIE_CUDA_CHECK(cudaGetLastError());
}

void launch_row_inv(const double2* A, double2* y, const Geom& g, const FftPlan& P1, double scale,
                    const double2* eps, const double2* xin, double inv_v, int basis, int diag, cudaStream_t st) {
  const int nrows = g.S * g.n2 * g.n3;
  const size_t sm = row_smem(g.m1);
  set_smem(reinterpret_cast<const void*>(k_row_inv), sm);
  const int64_t nv = static_cast<int64_t>(g.n1) * g.n2 * g.n3;
  FastDiv dn1, dm, drpc;
  dn1.init(static_cast<uint32_t>(g.n1));
  dm.init(static_cast<uint32_t>(g.m1));
  drpc.init(static_cast<uint32_t>(g.n2 * g.n3));
  k_row_inv<<<(nrows + kRowsPerCta - 1) / kRowsPerCta, kThreads, sm, st>>>(
      A, y, g.n1, nrows, g.n2 * g.n3, nv, P1, scale, eps, xin, inv_v, basis == 1 ? 1 : 0, diag, dn1, dm, drpc);
  VIE_CUDA_CHECK(cudaGetLastError());
}

void launch_col_fwd(const double2* A, double2* B, const Geom& g, const FftPlan& P2, cudaStream_t st) {
  const size_t sm = col_smem(g.m2);
  set_smem(reinterpret_cast<const void*>(k_col_fwd), sm);
  dim3 grid((g.m1 + kColsPerCta - 1) / kColsPerCta, g.S * g.n3);
  k_col_fwd<<<grid, kThreads, sm, st>>>(A, B, g.n2, g.m1, P2, g.bps);
  VIE_CUDA_CHECK(cudaGetLastError());
}

void launch_col_inv(const double2* B, const double2* B1, double2* A, const Geom& g, const FftPlan& P2,
                    cudaStream_t st) {
  const size_t sm = col_smem(g.m2);
  set_smem(reinterpret_cast<const void*>(k_col_inv), sm);
  dim3 grid((g.m1 + kColsPerCta - 1) / kColsPerCta, g.S * g.n3);
  k_col_inv<<<grid, kThreads, sm, st>>>(B, B1, A, g.n2, g.m1, P2, g.bps);
  VIE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace vie
