// kernels.cuh -- host-side launch interface of the matvec kernels.
#pragma once
#include <vector>

#include "common.cuh"

namespace vie {

// Per-component device descriptor of a Fourier-domain Tucker form, octant rows
// only: U_q^o has (n_q + 1) rows (the rest follow from U(m - p) = sign U(p)).
struct CompDev {
  int r1, r2, r3;
  int active;
  int64_t off_core;  // r1*r2*r3, core(a,b,g) at a + r1*(b + r2*g)   (decomp.hpp:124)
  int64_t off_u1;    // (n1+1) x r1 column-major
  int64_t off_u2;    // (n2+1) x r2
  int64_t off_u3;    // (n3+1) x r3
  int64_t off_z;     // Z[p2o][a][g]  (n2+1) x r1 x r3
  int64_t off_u3i;   // U3 shared-memory image of the tile decomposition: [b][NP3][Kp] (decomp_tile.cuh)
};

struct Geom {
  int n1, n2, n3;  // grid
  int m1, m2, m3;  // embedded (2n)
  int S;           // current components (sources = targets)
  int NC;          // canonical component count
  // Slab decomposition (multi-GPU): rank r of R owns the z-planes
  // [r nk, (r+1) nk) for the axis-1 passes and the axis-1 positions [p1off, p1off + W) for
  // the axis-2 passes, the decomposition rows and the pencil stage.  The exchanged slabs
  // (after the axis-1 FFT) are blocked [rank][s][k in block][j][w < W]; the spectral slabs
  // B, Bo of the pencil stage are [r][s][k in block][pos2][w < W] (block r = k / nk).
  // One GPU: nk = n3, W = m1, p1off = 0, a single block.
  int nk;          // k-planes per block
  int W;           // axis-1 positions per rank (row length of the exchanged / spectral slabs)
  int p1off;       // first global axis-1 position of this rank's W
  int64_t bps;     // plane stride of B, Bo = m2 * W
  // Octant-spectrum row layout read by the edge pencil kernels: 0 = the full (n2+1) x (n1+1)
  // rows; 1 = the compact EDGE buffer of the fused path (only rows p2o in {0, n2} and p1o in
  // {0, n1} exist, shat_row)
  int ecompact;
};

// Row of octant row (p2o, p1o) in the spectrum buffer (Geom::ecompact)
__host__ __device__ __forceinline__ int64_t shat_row(int p2o, int p1o, int n1, int n2, int compact) {
  if (!compact) return static_cast<int64_t>(p2o) * (n1 + 1) + p1o;
  if (p2o == 0) return p1o;
  if (p2o == n2) return n1 + 1 + p1o;
  return 2 * (n1 + 1) + 2 * (p2o - 1) + (p1o == 0 ? 0 : 1);  // p1o in {0, n1}
}
__host__ __device__ __forceinline__ int64_t shat_rows(int n1, int n2, int compact) {
  return compact ? 2 * static_cast<int64_t>(n1 + 1) + 2 * static_cast<int64_t>(n2 - 1)
                 : static_cast<int64_t>(n1 + 1) * (n2 + 1);
}

// Tuning constants.
constexpr int kRowsPerCta = 8;     // row FFT kernels
constexpr int kColsPerCta = 8;     // column FFT kernels (128 B segments)
constexpr int kPencilLines = 24;   // pencil kernel: S * W lines in smem
constexpr int kThreads = 256;
constexpr size_t kMaxSmem = 227 * 1024;  // per-CTA dynamic shared memory limit (sm_100a)

size_t row_smem(int m);
size_t col_smem(int m);
size_t pencil_smem(int n3, int S, int NC);  // (size_t)-1 if it does not fit
size_t decomp_smem(int n3, int rmax);
// U3 images of the tile decomposition (decomp_tile.cuh), one per active component
int64_t u3_image_elems(int n3, int r3);
void launch_u3_image(const double2* forms, const CompDev* comps_host, int NC, int n3, double2* img, cudaStream_t st);
size_t decomp_mma_smem(int n1, int n3, int rmax);

void launch_row_fwd(const double2* x, double2* A, const Geom& g, const FftPlan& P1, cudaStream_t st);
void launch_col_fwd(const double2* A, double2* B, const Geom& g, const FftPlan& P2, cudaStream_t st);
// Bin: forward slab (after axes 1-2); Bout: output slab (before the axis-2/1
// inverses); PH: n3-point plan; twm3: w_m3^e table of the m3-point plan.
void launch_pencil(int kind, int basis, const double2* Bin, double2* Bout, double2* Bout1, const double2* Shat,
                   const Geom& g, const FftPlan& PH, const double2* twm3, uint64_t active_mask, cudaStream_t st,
                   int groups = 0);  // groups > 0: only the first `groups` axis-1 pair groups (edge pencils)
// Compile-time-shaped pencil kernel (kernels_pencil2.cu) for n3 = R0 * R1 in
// its shape list and all components active; handles every axis-1 group but
// the first (frequencies 0 and n1 pair differently), which launch_pencil
// covers with groups = 1.  Returns false (nothing launched) if unsupported.
bool pencil2_supported(int kind, int basis, int n3, uint64_t active_mask, int NC);

// pos2 range [pos2lo, pos2hi) of axis-2 positions (pos2hi < 0: all m2)
void launch_pencil2(int kind, int basis, const double2* Bin, double2* Bout, const double2* Shat, const Geom& g,
                    const double2* twm3, cudaStream_t st, int pos2lo = 0, int pos2hi = -1);
// PWL pencil kernel with the Hadamard on the FP64 tensor cores (kernels_pencil3.cu): one
// 2-CTA cluster per interior mirror group (axis-1 pair group >= 1, axis-2 pair >= 1), all
// four pencils; the axis-1 edge group (launch_pencil groups = 1) and the axis-2 edge
// positions 0, 1 (launch_pencil2 with pos2 in [0, 2)) complete the grid.
bool pencil3_supported(int kind, int basis, int n3, uint64_t active_mask, int NC);
void launch_pencil3(int kind, const double2* Bin, double2* Bout, const double2* Shat, const Geom& g,
                    const double2* twm3, cudaStream_t st);
// Same interior mirror groups, half a group (one axis-2 position) per 2-CTA cluster and two
// clusters per SM pair (kernels_pencil4.cu); preferred over pencil3 where supported.
bool pencil4_supported(int kind, int basis, int n3, uint64_t active_mask, int NC);
void launch_pencil4(int kind, const double2* Bin, double2* Bout, const double2* Shat, const Geom& g,
                    const double2* twm3, cudaStream_t st);
// Fused decompression x pencil (kernels_fused.cu): the interior octant rows are decompressed
// tile by tile into an L2-resident ring and consumed by the pencil items of one persistent kernel.
struct FusedPlan {
  const double2* forms = nullptr;
  const double2* u3img = nullptr;
  const CompDev* comps = nullptr;
  const double2* Z = nullptr;
  double2* ring = nullptr;       // [RING * BM][NC][n3 + 1]
  const int4* items = nullptr;   // work queue (fused_plan_items)
  int nitems = 0;
  unsigned* counters = nullptr;  // queue head, done[ntiles][2], consumed[ntiles]
  int ntiles = 0, CG = 4, NG = 0, RING = 0, BM = 0, NB = 0, rmax = 0;
};
bool fused_supported(int kind, int basis, const Geom& g, uint64_t active_mask, int rmax);
void fused_plan_items(FusedPlan& fp, const Geom& g, std::vector<int4>& items);
void launch_fused(int kind, const FusedPlan& fp, const double2* Bin, double2* Bout, const Geom& g,
                  const double2* twm3, cudaStream_t st);
// edge rows (p2o in {0, n2}, p1o in {0, n1}) into the compact edge buffer (Geom::ecompact = 1)
void launch_decomp_edges(const FusedPlan& fp, double2* Sedge, const Geom& g, cudaStream_t st);
// Z = core x2 U2 only (the fused path's decompression prologue)
void launch_decomp_z(const double2* forms, const CompDev* comps_dev, double2* Z, const Geom& g, int rmax,
                     cudaStream_t st);
// B1 (optional): second slab added to B on load (the pencil kernel's odd branch)
void launch_col_inv(const double2* B, const double2* B1, double2* A, const Geom& g, const FftPlan& P2,
                    cudaStream_t st);
// Register-staged passes (kernels_fft2.cu) for axes with m = R0 * R1 (or
// m = R0), R0 even: one shared-memory round trip per pass.
struct Pass2 {
  int m, n;     // embedded / grid length
  int R0, R1;   // radices (R1 == 1: single stage)
  int R1p, ls;  // padded block length (odd) and smem line stride (odd)
  int lines;    // rows per CTA (row passes)
  int ext;      // a radix has a prime factor 11..31: the EXT instantiation of the passes
  const double2* tw;  // w_m^e
  FastDiv dR0, dR1;
};
bool pass2_init(Pass2& P, int m, const int* radices, int nst, const double2* tw, int row_lines);
void launch_row_fwd2(const double2* x, double2* A, const Geom& g, const Pass2& P, cudaStream_t st);
// Plane remap of the slab-blocked column passes (current groups of the overlapped multi-GPU
// exchange): plane p of the group-local side <-> plane (p / in_per_r) out_per_r + off + p % in_per_r
// of the full spectral slab.  Default: identity.
struct PlaneMap {
  int in_per_r = 1 << 30, out_per_r = 1 << 30, off = 0;
  __host__ __device__ int64_t operator()(int p) const {
    return static_cast<int64_t>(p / in_per_r) * out_per_r + off + p % in_per_r;
  }
};
void launch_col_fwd2(const double2* A, double2* B, const Geom& g, const Pass2& P, cudaStream_t st, PlaneMap pm = {});
void launch_col_inv2(const double2* B, double2* A, const Geom& g, const Pass2& P, cudaStream_t st, PlaneMap pm = {});
void launch_row_inv2(const double2* A, double2* y, const Geom& g, const Pass2& P, double scale, const double2* eps,
                     const double2* xin, double inv_v, int basis, int diag, cudaStream_t st);

// Epilogue: y = scale * (IDFT) or the system form (eps != nullptr):
//   y = (diag ? eps*g_l*xin : 0) - (eps - 1) * inv_v * scale * (IDFT)
void launch_row_inv(const double2* A, double2* y, const Geom& g, const FftPlan& P1, double scale,
                    const double2* eps, const double2* xin, double inv_v, int basis, int diag, cudaStream_t st);

// Octant spectra rows p2o in [p2lo, p2hi) x p1o in [p1lo, p1hi) (hi < 0: all rows);
// with_z: also Z = core x2 U2
void launch_decomp(const double2* forms, const CompDev* comps_dev, const CompDev* comps_host, double2* Z,
                   double2* Shat, const Geom& g, int rmax, cudaStream_t st, int p2lo = 0, int p2hi = -1,
                   bool with_z = true, int p1lo = 0, int p1hi = -1, const double2* u3img = nullptr);

// transform_factors on device: spatial factor (n x r, col-major) -> octant rows
// (n+1) x r of the DFT of the parity embedding (operator.hpp:64-90).
void launch_factor_transform(const double2* u, int n, int r, int sign, const double2* tw2n, double2* out,
                             cudaStream_t st);

// ---- tucker_compress (hosvd) device parts
// G (nq x nq, col-major) = M_q M_q^H of the mode-q unfolding (mode 1..3)
void launch_gram(const double2* t, const int64_t dims[3], int mode, double2* G, cudaStream_t st);
// out = in x_mode U^H (U: n_mode x r col-major)
void launch_mode_product_h(const double2* in, const int64_t dims[3], int mode, const double2* U, int r,
                           double2* out, cudaStream_t st);
// *acc += sum |a - b|^2 (b null: sum |a|^2); acc is a device double the caller zeroes
void launch_diff_norm2(const double2* a, const double2* b, int64_t n, double* acc, cudaStream_t st);
// *acc += sum |t - cp(W1, W2, W3)|^2 (W_q: dims[q] x R col-major, device)
void launch_cp_residual2(const double2* t, const int64_t dims[3], const double2* w1, const double2* w2,
                         const double2* w3, int R, double* acc, cudaStream_t st);

// ---- cp_als (decomp.hpp:237-298) on a host tensor (the HOSVD core: r1 r2 r3 <= a few
// 10^4 entries, setup work like the r x r eigenproblems of the HOSVD); cp_als.cu
struct CpAlsHost {
  std::vector<double2> f[3];  // d_q x r col-major
  std::vector<double> trace;  // relative error per sweep
  bool converged = false, ill_posed = false;
};
CpAlsHost cp_als_host(const double2* t, const int64_t d[3], int64_t r, int max_iters, double stall_tol,
                      uint64_t seed);

// ---- Green's-tensor assembly (kernels_assembly.cu; assembly.hpp:159-233)
struct AssemblyDesc {
  int64_t dims[3];
  double res[3];  // voxel edges (m)
  double k0;      // wavenumber (1/m)
  int op;         // 0 N, 1 K, 2 scalar g
  int q, qp;      // row / column axis
  int far, near, near_radius, surface, volume;  // QuadratureSpec (assembly.hpp:24-36)
};
constexpr int kAsmRuleElems = 160;  // Gauss tables: at most 5 point counts <= 31
// t (device, n1 n2 n3 complex) = the defining tensor; t == nullptr: only the static self
// term (dyad_out[3] diagonal, err_out the refinement change), both device pointers or null.
// self_scratch: 1 complex, rules_scratch: 2 kAsmRuleElems + 4 doubles (device).
void launch_assemble(const AssemblyDesc& ad, double2* t, double2* self_scratch, double* rules_scratch,
                     cudaStream_t st, double* dyad_out, double* err_out);

// detail::correlation_entry (assembly.hpp:49-79) of kernel op (0 N, 1 K, 2 g, 3 N self
// remainder) at displacement d, voxel delta (x-edge units), one thread (test hook)
void launch_correlation_entry(int op, double k, int q, int qp, const double d[3], const double delta[3], int points,
                              int duffy, double* rules_scratch, double2* out, cudaStream_t st);

// ---- BLAS-1 for GMRES (deterministic two-level reductions) ----
struct RedBuf {
  double2* partials;       // kRedBlocks entries
  unsigned int* counter;   // zero-initialised
};
constexpr int kRedBlocks = 592;  // 4 x 148 SMs
// out[0] = sum conj(a) * b
void launch_dot(const double2* a, const double2* b, int64_t n, double2* out, RedBuf rb, cudaStream_t st);
// out[0].x = sum |a|^2
void launch_nrm2sq(const double2* a, int64_t n, double2* out, RedBuf rb, cudaStream_t st);
// w -= h[0] * v ; then out[0] = sum conj(vnext) * w   (vnext == nullptr: out = |w|^2)
void launch_mgs_step(double2* w, const double2* v, const double2* h, const double2* vnext, int64_t n,
                     double2* out, RedBuf rb, cudaStream_t st);
// r = rhs - ax ; out = |r|^2
void launch_residual(const double2* rhs, const double2* ax, double2* r, int64_t n, double2* out, RedBuf rb,
                     cudaStream_t st);
// y = x / d with d = s[0].x (device) or `divisor` when s == nullptr
void launch_scale_inv(const double2* x, double2* y, const double2* s, double divisor, int64_t n, cudaStream_t st);
// x += z
void launch_axpy1(double2* x, const double2* z, int64_t n, cudaStream_t st);
// out = d * in (element-wise complex product: the diagonal right preconditioner)
void launch_cmul_elem(const double2* d, const double2* in, double2* out, int64_t n, cudaStream_t st);
// x += sum_l V_l * coef[l]
void launch_basis_update(double2* x, const double2* V, int64_t ldv, const double2* coef, int j, int64_t n,
                         cudaStream_t st);

// ---- scene stages around the solve (kernels_scene.cu; solver.hpp:148-285)
constexpr double kEpsilon0 = 8.8541878128e-12;  // grid.hpp:15
constexpr double kMu0 = 1.25663706212e-6;       // grid.hpp:16
constexpr int kMaxQuad = 8;
struct SceneDev {
  int64_t n[3];
  double res[3], org[3];
  double k0, omega;
  double2 ce;             // c_e = i omega eps0 (grid.hpp:64)
  double pol[3], dir[3];  // normalised (grid.hpp:84-86)
  double amp;
  double hdir[3];         // dir x pol (grid.hpp:97)
  double hamp;            // amp / eta0
  int quad;               // build_rhs quadrature points per axis
  double qn[kMaxQuad], qw[kMaxQuad];  // Gauss rule on [0, 1] (quadrature.hpp:23-52)
};
void launch_build_rhs(const SceneDev& sc, const double2* eps, double2* rhs, cudaStream_t st);
void launch_recover_e(const SceneDev& sc, const double2* eps, const double2* j, double2* e, cudaStream_t st);
void launch_add_hinc(const SceneDev& sc, double inv_v, double2* h, cudaStream_t st);
// p_abs, b1 (h != nullptr), total[0] = scale * sum p_abs; partials: kRedBlocks doubles
void launch_postprocess(const SceneDev& sc, const double2* eps, const double2* e, const double2* h, double* p_abs,
                        double* b1, double* partials, double* total, double scale, cudaStream_t st);

}  // namespace vie
