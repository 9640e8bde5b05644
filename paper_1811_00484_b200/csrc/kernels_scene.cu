// kernels_scene.cu -- the per-voxel stages of solve_scene around the solve
// (solver.hpp:148-285): build_rhs, the e / h recovery of recover_fields and
// postprocess.  Each is one streaming pass over the voxels (HBM-bound, no
// reuse); the incident plane wave is evaluated in registers, never stored.
// The absorbed-power sum is deterministic: one partial per CTA, then a single
// warp adds the partials in index order.
#include "kernels.cuh"

namespace vie {

namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// 1 / z with the scaling of std::complex division (no overflow for |z| ~ 1e300)
__device__ __forceinline__ double2 cinv(double2 z) {
  const double s = fabs(z.x) >= fabs(z.y) ? z.x : z.y;
  const double zr = z.x / s, zi = z.y / s;
  const double d = s * (zr * zr + zi * zi);
  return make_double2(zr / d, -zi / d);
}

// PlaneWave phase e^{-i k0 dir.r} (grid.hpp:90-99)
__device__ __forceinline__ double2 phase_at(const SceneDev& sc, double rx, double ry, double rz) {
  const double a = sc.k0 * (sc.dir[0] * rx + sc.dir[1] * ry + sc.dir[2] * rz);
  double s, c;
  sincos(a, &s, &c);
  return make_double2(c, -s);
}

__device__ __forceinline__ void voxel_center(const SceneDev& sc, int64_t v, double& x, double& y, double& z) {
  const int64_t i = v % sc.n[0];
  const int64_t r = v / sc.n[0];
  const int64_t j = r % sc.n[1];
  const int64_t k = r / sc.n[1];
  x = sc.org[0] + (static_cast<double>(i) + 0.5) * sc.res[0];  // grid.hpp:42-46
  y = sc.org[1] + (static_cast<double>(j) + 0.5) * sc.res[1];
  z = sc.org[2] + (static_cast<double>(k) + 0.5) * sc.res[2];
}

__global__ void __launch_bounds__(kThreads) k_build_rhs(SceneDev sc, const double2* __restrict__ eps,
                                                        double2* __restrict__ rhs) {
  const int64_t nv = sc.n[0] * sc.n[1] * sc.n[2];
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    const double2 e = eps[v];
    const double2 chi = make_double2(e.x - 1.0, e.y);
    if (chi.x == 0.0 && chi.y == 0.0) {  // solver.hpp:161: no current outside the scatterer
      for (int q = 0; q < 3; ++q) rhs[q * nv + v] = make_double2(0.0, 0.0);
      continue;
    }
    double cx, cy, cz;
    voxel_center(sc, v, cx, cy, cz);
    double2 ph;
    if (sc.quad == 1) {
      ph = phase_at(sc, cx, cy, cz);
    } else {  // tensor Gauss over the voxel (solver.hpp:165-172)
      ph = make_double2(0.0, 0.0);
      for (int a = 0; a < sc.quad; ++a)
        for (int b = 0; b < sc.quad; ++b)
          for (int d = 0; d < sc.quad; ++d) {
            const double w = sc.qw[a] * sc.qw[b] * sc.qw[d];
            const double2 p = phase_at(sc, cx + sc.res[0] * (sc.qn[a] - 0.5), cy + sc.res[1] * (sc.qn[b] - 0.5),
                                       cz + sc.res[2] * (sc.qn[d] - 0.5));
            ph.x += w * p.x;
            ph.y += w * p.y;
          }
    }
    const double2 cc = cmul(sc.ce, chi);
    for (int q = 0; q < 3; ++q) {
      const double2 eq = make_double2(sc.pol[q] * sc.amp * ph.x, sc.pol[q] * sc.amp * ph.y);
      rhs[q * nv + v] = cmul(cc, eq);
    }
  }
}

__global__ void __launch_bounds__(kThreads) k_recover_e(SceneDev sc, const double2* __restrict__ eps,
                                                        const double2* __restrict__ j, double2* __restrict__ e) {
  const int64_t nv = sc.n[0] * sc.n[1] * sc.n[2];
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    const double2 ep = eps[v];
    const double2 chi = make_double2(ep.x - 1.0, ep.y);
    if (chi.x == 0.0 && chi.y == 0.0) {  // solver.hpp:222-224: incident field, never divided
      double cx, cy, cz;
      voxel_center(sc, v, cx, cy, cz);
      const double2 ph = phase_at(sc, cx, cy, cz);
      for (int q = 0; q < 3; ++q) e[q * nv + v] = make_double2(sc.pol[q] * sc.amp * ph.x, sc.pol[q] * sc.amp * ph.y);
    } else {  // solver.hpp:225-227
      const double2 inv = cinv(cmul(sc.ce, chi));
      for (int q = 0; q < 3; ++q) e[q * nv + v] = cmul(inv, j[q * nv + v]);
    }
  }
}

// h = h_inc + inv_v * kj, in place over kj (solver.hpp:233-243)
__global__ void __launch_bounds__(kThreads) k_add_hinc(SceneDev sc, double inv_v, double2* __restrict__ h) {
  const int64_t nv = sc.n[0] * sc.n[1] * sc.n[2];
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    double cx, cy, cz;
    voxel_center(sc, v, cx, cy, cz);
    const double2 ph = phase_at(sc, cx, cy, cz);
    for (int q = 0; q < 3; ++q) {
      const double2 kj = h[q * nv + v];
      const double s = sc.hdir[q] * sc.hamp;
      h[q * nv + v] = make_double2(s * ph.x + inv_v * kj.x, s * ph.y + inv_v * kj.y);
    }
  }
}

// postprocess (solver.hpp:258-284): p_abs, b1_plus, per-CTA partial of sum p_abs
__global__ void __launch_bounds__(kThreads) k_postprocess(SceneDev sc, const double2* __restrict__ eps,
                                                          const double2* __restrict__ e,
                                                          const double2* __restrict__ h, double* __restrict__ p_abs,
                                                          double* __restrict__ b1, double* __restrict__ partials) {
  __shared__ double ws[kThreads / 32];
  const int64_t nv = sc.n[0] * sc.n[1] * sc.n[2];
  double acc = 0.0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    double e2 = 0.0;
    for (int q = 0; q < 3; ++q) {
      const double2 x = e[q * nv + v];
      e2 += x.x * x.x + x.y * x.y;  // std::norm
    }
    const double sigma = -eps[v].y * kEpsilon0 * sc.omega;  // grid.hpp:68-70
    const double p = 0.5 * sigma * e2;
    p_abs[v] = p;
    acc += p;
    if (h) {
      const double2 hx = h[v], hy = h[nv + v];
      b1[v] = kMu0 * hypot(hx.x - hy.y, hx.y + hy.x);  // |h_x + i h_y|
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) s += ws[w];
    partials[blockIdx.x] = s;
  }
}

// one warp, partials summed in index order -> out[0]
__global__ void k_sum_partials(const double* __restrict__ partials, int n, double scale, double* out) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += 32) s += partials[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) out[0] = s * scale;
}

int grid_for(int64_t n) {
  const int64_t b = (n + kThreads - 1) / kThreads;
  return static_cast<int>(b < kRedBlocks ? (b < 1 ? 1 : b) : kRedBlocks);
}

}  // namespace

void launch_build_rhs(const SceneDev& sc, const double2* eps, double2* rhs, cudaStream_t st) {
  k_build_rhs<<<grid_for(sc.n[0] * sc.n[1] * sc.n[2]), kThreads, 0, st>>>(sc, eps, rhs);
  VIE_CUDA_CHECK(cudaGetLastError());
}

void launch_recover_e(const SceneDev& sc, const double2* eps, const double2* j, double2* e, cudaStream_t st) {
  k_recover_e<<<grid_for(sc.n[0] * sc.n[1] * sc.n[2]), kThreads, 0, st>>>(sc, eps, j, e);
  VIE_CUDA_CHECK(cudaGetLastError());
}

void launch_add_hinc(const SceneDev& sc, double inv_v, double2* h, cudaStream_t st) {
  k_add_hinc<<<grid_for(sc.n[0] * sc.n[1] * sc.n[2]), kThreads, 0, st>>>(sc, inv_v, h);
  VIE_CUDA_CHECK(cudaGetLastError());
}

void launch_postprocess(const SceneDev& sc, const double2* eps, const double2* e, const double2* h, double* p_abs,
                        double* b1, double* partials, double* total, double scale, cudaStream_t st) {
  const int g = grid_for(sc.n[0] * sc.n[1] * sc.n[2]);
  k_postprocess<<<g, kThreads, 0, st>>>(sc, eps, e, h, p_abs, b1, partials);
  VIE_CUDA_CHECK(cudaGetLastError());
  k_sum_partials<<<1, 32, 0, st>>>(partials, g, scale, total);
  VIE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace vie
