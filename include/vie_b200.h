/*
 * vie_b200.h -- C ABI of the B200-native Tucker-compressed VIE matvec.
 *
 * Drop-in boundary for the reference's operator API (header-only C++ library
 * /root/reference/proj/include/vie).  Each entry point names the reference
 * interface it replaces.  All complex data is interleaved double (re, im),
 * i.e. std::complex<double> / double2, in the reference layouts:
 *   Tensor3:        flat = i + n1*(j + n2*k)                 tensor.hpp:17-21
 *   factor matrix:  column-major, rows x cols                tensor.hpp:15-17
 *   current field:  component-major blocks of N_v            grid.hpp:122-127
 *                   PWC: 3 blocks (q); PWL: 12 blocks (s = 4q + l)
 * Pointers are DEVICE pointers unless the name ends in _host.  `stream` is a
 * cudaStream_t passed as void* (NULL = the context's stream).
 *
 * Every function returns VIE_OK (0) or an error code, and sets a thread-local
 * message readable with vie_last_error().  VIE_EINVAL corresponds to the
 * reference's std::invalid_argument (operator.hpp:277-284, solver.hpp:37-39).
 * GMRES non-convergence is a flag, not an error (solver.hpp:28-33).
 */
#ifndef VIE_B200_H
#define VIE_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VIE_OK 0
#define VIE_EINVAL 1
#define VIE_ENOMEM 2
#define VIE_ECUDA 3
#define VIE_ENCCL 4
#define VIE_EIO 5 /* file I/O (the reference's std::runtime_error of container.hpp) */

#define VIE_KIND_N 0 /* OperatorKind::N  (components.hpp:14) */
#define VIE_KIND_K 1 /* OperatorKind::K                      */
#define VIE_BASIS_PWC 0 /* BasisOrder::PWC (grid.hpp:103)    */
#define VIE_BASIS_PWL 1 /* BasisOrder::PWL (generalised) */
#define VIE_RULE_SIGMA_MAX 0 /* TruncationRule (decomp.hpp:23) */
#define VIE_RULE_ENERGY 1

typedef struct vie_ctx_s* vie_ctx;       /* device, stream, FFT plan cache   (fft.hpp DftService) */
typedef struct vie_tucker_s* vie_tucker; /* device-resident Fourier Tucker form (decomp.hpp:123 + operator.hpp:76) */
typedef struct vie_op_s* vie_op;         /* immutable device operator        (operator.hpp:120 EmbeddedSpectrum) */

const char* vie_last_error(void);
const char* vie_version(void);

/* DftService construction (fft.hpp:13-21): binds a CUDA device. */
int vie_ctx_create(vie_ctx* out, int device);
int vie_ctx_destroy(vie_ctx ctx);
int vie_ctx_sync(vie_ctx ctx);
/* The context's CUDA stream (cudaStream_t as void*), which the calls use when their
 * `stream` argument is NULL; vie_op_stream: the stream of the operator's context.
 * Forms and operators keep their context alive: vie_ctx_destroy releases the
 * caller's reference and the context is freed with its last form / operator.       */
int vie_ctx_stream(vie_ctx ctx, void** stream);
int vie_op_stream(vie_op op, void** stream);

/* tucker_compress = hosvd + transform_factors (decomp.hpp:160-176,
 * operator.hpp:76-90): HOSVD of a spatial Toeplitz-defining tensor (host
 * buffer, n1*n2*n3 complex), then embedding + 1D DFT of every factor column
 * on the device.  sign[3] = component parity (components.hpp:51-65).
 * rule: VIE_RULE_*.  ranks_out receives (r1, r2, r3).                        */
int vie_tucker_compress(vie_ctx ctx, const int64_t dims[3], const double* t_host, const int sign[3],
                        double tol, int rule, vie_tucker* out, int64_t ranks_out[3]);

/* The same with a DEVICE tensor (e.g. straight from vie_assemble), ordered after
 * `stream` (NULL: the context stream); returns after the form is built.          */
int vie_tucker_compress_device(vie_ctx ctx, const int64_t dims[3], const double* t_dev, const int sign[3],
                               double tol, int rule, vie_tucker* out, int64_t ranks_out[3], void* stream);

/* tucker_cp (decomp.hpp:336-373): hosvd on the device (as vie_tucker_compress_device), CP-ALS
 * on the r1 x r2 x r3 core (cp_als, decomp.hpp:237-298: SVD-initialised factors, seed 0x5eed,
 * cp_iters sweeps at most, stop when the error decrease < stall_tol), merged factors
 * W_q = U_q V_q.  t: n1 n2 n3 complex, a DEVICE buffer when t_on_device (ordered after
 * `stream`, NULL = the context stream) else a host buffer.  CP rank = cp_rank if >= 0 else
 * min(r1, r2, r3).  Every output is optional (NULL): out = the device form of
 * transform_factors(TuckerCPForm) (as vie_tucker_from_cp); rank_out; w1..w3 = the spatial
 * W_q on the host (n_q x w_cap column-major capacity each, VIE_EINVAL if rank > w_cap);
 * errs = {hosvd_relative_error, core_cp_relative_error, stats.achieved_relative_error};
 * trace = the CP error per sweep (up to trace_cap), ntrace = the number of sweeps.       */
int vie_tucker_cp(vie_ctx ctx, const int64_t dims[3], const double* t, int t_on_device, const int sign[3],
                  double tol, int rule, int cp_iters, int64_t cp_rank, double stall_tol, vie_tucker* out,
                  int64_t* rank_out, double* w1, double* w2, double* w3, int64_t w_cap, double errs[3],
                  double* trace, int trace_cap, int* ntrace, void* stream);
/* cp_als (decomp.hpp:237-298) of a host tensor (dims[0] x dims[1] x dims[2], the reference
 * layout) at rank r: factors f_q (dims[q] x r, host, optional), the relative error per sweep
 * (trace, up to trace_cap; ntrace = sweeps run), flags = {converged, ill_posed_rank}.
 * Host computation (meant for Tucker cores; no device needed).                          */
int vie_cp_als(const int64_t dims[3], const double* t_host, int64_t r, int max_iters, double stall_tol,
               uint64_t seed, double* f1, double* f2, double* f3, double* trace, int trace_cap, int* ntrace,
               int flags[2]);

/* ---- Green's-tensor assembly (assembly.hpp:159-246, kernels.hpp, quadrature.hpp) ----
 * QuadratureSpec (assembly.hpp:24-36); NULL = the defaults {5, 10, 1, 12, 6}.          */
typedef struct {
  int far_points_per_axis;
  int near_points_per_axis;
  int near_radius; /* Chebyshev voxel distance using the near rule */
  int surface_points_per_axis; /* self term: static nabla-nabla dyad (face pairs) */
  int volume_points_per_axis;  /* self term: dynamic remainder (Duffy boxes) */
} vie_quadrature;
#define VIE_KIND_G 2 /* OperatorKind::ScalarG (components.hpp:14) */

/* assemble_defining_tensor (assembly.hpp:159-233) on the device: the PWC Galerkin
 * Toeplitz-defining tensor of component (kind, row_axis, col_axis) of the grid with
 * voxel edges resolution[3] (m) at wavenumber k0 (1/m), written to t (device,
 * n1 n2 n3 complex, reference layout, SI units).  basis must be VIE_BASIS_PWC
 * (VIE_EINVAL otherwise, as the reference throws); zero quadrature budgets are
 * VIE_EINVAL.  Runs on `stream` (NULL: the context stream); returns when done.   */
int vie_assemble(vie_ctx ctx, const int64_t dims[3], const double resolution[3], double k0, int kind,
                 int row_axis, int col_axis, int basis, const vie_quadrature* quad, double* t, void* stream);
/* detail::correlation_entry (assembly.hpp:49-79) on the device, one entry: kernel op
 * (0 N, 1 K, 2 scalar g, 3 the N self remainder of kernels.hpp:113-119) at wavenumber k,
 * displacement d and voxel delta in x-edge units, `points` per axis, Duffy at d when
 * duffy != 0; out_host = complex result.  (A test hook for the quadrature parity.)   */
int vie_correlation_entry(vie_ctx ctx, int op, double k, int q, int qp, const double d[3], const double delta[3],
                          int points, int duffy, double* out_host);
/* self_static_term (assembly.hpp:127-150): diagonal of the static nabla-nabla dyad of a
 * delta[0] x delta[1] x delta[2] voxel (off-diagonals vanish), the Gram term (volume),
 * the surface-rule refinement change and converged = change < 1e-7.               */
int vie_self_static_term(vie_ctx ctx, const double delta[3], const vie_quadrature* quad, double dyad_diag[3],
                         double* gram, double* error_indicator, int* converged);

/* Tucker form from given factors (the synthetic-input path, no SVD).
 * domain 0: spatial factors U_q (n_q x r_q, host) -> transform_factors on device
 * domain 1: Fourier factors (2n_q x r_q, host) as returned by transform_factors
 * core_host: r1*r2*r3.  Rows that the parity forces to zero (row 0 of an odd
 * axis) must be zero to 1e-12 relative; VIE_EINVAL otherwise.               */
int vie_tucker_from_factors(vie_ctx ctx, const int64_t dims[3], const int64_t ranks[3],
                            const double* core_host, const double* u1_host, const double* u2_host,
                            const double* u3_host, const int sign[3], int domain, vie_tucker* out);
/* Tucker+CP form (decomp.hpp:143-148, merged factors W_q = U_q V_q, n_q x rank):
 * S = sum_l W1(:,l) o W2(:,l) o W3(:,l), held as a Tucker form with the
 * superdiagonal rank^3 core, so the fused decompress x Hadamard matvec serves the
 * reference's TuckerCpLoop / decompress_cp strategies (operator.hpp:248-261,
 * 346-362).  domain as for vie_tucker_from_factors (1 = transform_factors(
 * TuckerCPForm) output, operator.hpp:92-106).                                   */
int vie_tucker_from_cp(vie_ctx ctx, const int64_t dims[3], int64_t rank, const double* w1_host,
                       const double* w2_host, const double* w3_host, const int sign[3], int domain,
                       vie_tucker* out);
int vie_tucker_ranks(vie_tucker t, int64_t ranks_out[3]);
int vie_tucker_destroy(vie_tucker t);

/* ---- VIET container (container.hpp:15-159): the reference's binary file of dense tensors
 * and compressed forms, byte for byte ("VIET", version 1, kind 0 dense / 1 tucker / 2
 * tucker_cp, rule, tol, dims, ranks, then (re, im) f64 payload: dense n1 n2 n3 axis-1 fastest;
 * tucker U1, U2, U3 column-major then the core; tucker_cp W1, W2, W3).  I/O errors (cannot
 * open, bad magic, unsupported version, truncated, unknown kind) return VIE_EIO.
 * vie_container_info / _read / _write work on host buffers (no device needed).
 * vie_tucker_save writes a device form created from spatial factors (domain 0, including
 * vie_tucker_compress* and vie_tucker_from_cp); vie_tucker_load builds the device form
 * (transform_factors on the device) from a tucker or tucker_cp file; `sign` is the
 * component's parity (not stored in the file).                                          */
int vie_container_info(const char* path, int* kind, int* rule, double* tol, int64_t dims[3], int64_t ranks[3]);
int vie_container_read(const char* path, double* payload, int64_t capacity_complex);
int vie_container_write(const char* path, int kind, int rule, double tol, const int64_t dims[3],
                        const int64_t ranks[3], const double* payload);
int vie_tucker_save(vie_tucker t, const char* path);
int vie_tucker_load(vie_ctx ctx, const char* path, const int sign[3], vie_tucker* out);

/* Canonical component table of (kind, basis): components.hpp:71-92 for PWC,
 * its PWL generalisation otherwise.  comps: ncomp x 4 ints (q, q', l, l');
 * parity: ncomp x 3; blocks: nblock x 4 (target, source, comp, dense_sign).
 * Any output pointer may be NULL (counts only).                             */
int vie_component_table(int kind, int basis, int* ncomp, int* comps, int* parity, int* nblock,
                        int* blocks);

/* build_operator_spectra (operator.hpp:144-177) from compressed forms.
 * comp: ncomp x 4 ints (q, q', l, l') naming which canonical component each
 * form holds (any order, each at most once; absent components are zero, which
 * is how components are sharded over GPUs).  Forms are copied.               */
int vie_op_create(vie_ctx ctx, int kind, int basis, const int64_t grid[3], int ncomp,
                  const int* comp, const vie_tucker* forms, vie_op* out);
int vie_op_destroy(vie_op op);
/* sizes: n_cur (= current components S), n_vox (= N_v), bytes of workspace   */
int vie_op_info(vie_op op, int64_t* n_cur, int64_t* n_vox, int64_t* workspace_bytes);

/* MatvecStrategy of every later apply on this operator (operator.hpp:17-31; the strategy
 * argument of apply_operator, operator.hpp:273-276, and of the solve closure):
 *   VIE_STRATEGY_HOSVD_DECOMPRESS: all components' octant spectra are decompressed into one
 *     HBM buffer, then read by the fused axis-3 FFT x Hadamard pass (default);
 *   VIE_STRATEGY_HOSVD_LOOP: the reference's buffer-free HosvdLoop -- one persistent kernel
 *     decompresses 64-row spectrum tiles into an L2-resident ring and consumes them in the same
 *     launch; only the edge rows (p2o in {0, n2}, p1o in {0, n1}) are stored.  PWL operators
 *     with ranks <= 28 and a compiled axis-3 shape; VIE_EINVAL otherwise or when partitioned.
 * Spectrum storage of a strategy is allocated on its first use (vie_op_info reports it).
 * The TuckerCp strategies map to these two (CP forms are held as Tucker forms).          */
#define VIE_STRATEGY_HOSVD_DECOMPRESS 1
#define VIE_STRATEGY_HOSVD_LOOP 2
int vie_op_set_strategy(vie_op op, int strategy);
int vie_op_get_strategy(vie_op op, int* strategy);

/* apply_operator (operator.hpp:273-382) with the operator's strategy (vie_op_set_strategy):
 * y = A x for device vectors of n_cur * n_vox complex values.                */
int vie_matvec(vie_op op, const double* x, double* y, void* stream);
/* apply_operator with ApplyTimings (operator.hpp:189-192): the stages run serialised with
 * CUDA events between them; fft_ms = the row / column FFT passes (pad, axes 1-2, their
 * inverses, crop), product_ms = decompression + the fused axis-3 FFT x Hadamard x IFFT
 * pass.  Device buffers, context stream, returns after completion.                   */
int vie_matvec_timed(vie_op op, const double* x, double* y, double* fft_ms, double* product_ms);
/* ---- multi-GPU exchange inside the library (one process per GPU) ----
 * vie_comm: an NCCL communicator over the ranks of a slab-partitioned operator.  Rank 0
 * creates the unique id and the caller broadcasts its bytes (MPI, torch.distributed, ...).
 * vie_op_set_comm attaches it to the operator (same rank / size as vie_op_set_partition);
 * then vie_slab_matvec runs this rank's whole matvec -- axis-1 FFTs of the z-slab, the
 * all-to-all (grouped ncclSend / ncclRecv), axis-2 FFTs + pencil stage on the rank's axis-1
 * positions, the all-to-all back, inverse axis-1 FFTs (+ apply_system epilogue when eps_local
 * is given) -- with the x-independent decomposition on a side stream concurrent with the
 * forward FFTs and exchange; and vie_gmres_solve on the partitioned operator solves with
 * distributed vectors (this rank's z-slabs), every dot and norm summed by ncclAllReduce
 * (solver.hpp:75-79).  Replaces the caller-driven vie_slab_* + external all-to-all loop. */
#define VIE_COMM_ID_BYTES 128
typedef struct vie_comm_s* vie_comm;
int vie_comm_unique_id(unsigned char id[VIE_COMM_ID_BYTES]);
int vie_comm_create(vie_ctx ctx, int nranks, int rank, const unsigned char id[VIE_COMM_ID_BYTES], vie_comm* out);
int vie_comm_destroy(vie_comm comm);
/* Loopback transport for tests: R ranks of ONE process (one host thread per rank, e.g. all on
 * one GPU) exchanging by device copies between host barriers; every call that exchanges or
 * all-reduces must be made by all R threads.                                              */
typedef struct vie_loopback_s* vie_loopback;
int vie_loopback_create(int nranks, vie_loopback* out);
int vie_loopback_destroy(vie_loopback lb);
int vie_comm_create_loopback(vie_ctx ctx, vie_loopback lb, int rank, vie_comm* out);
int vie_op_set_comm(vie_op op, vie_comm comm);
int vie_slab_matvec(vie_op op, const double* x_local, double* y_local, const double* eps_local, double inv_v,
                    int diag_term, void* stream);

/* Same call with HOST buffers (H2D, matvec, D2H) -- the reference-facing call. */
int vie_matvec_host(vie_op op, const double* x_host, double* y_host);
/* `count` independent applications with HOST buffers, pipelined: the H2D copy of
 * x_host[i+1] and the D2H copy of y_host[i-1] overlap the matvec of x_host[i]
 * (copy streams + two device slots per direction).  Pinned host buffers are
 * needed for the overlap.  Results are those of count vie_matvec_host calls. */
int vie_matvec_host_batch(vie_op op, int64_t count, const double* const* x_host, double* const* y_host);

/* apply_system (solver.hpp:183-200): y = eps_r*g*x - (eps_r - 1)*inv_v*(N x)
 * with g = 1 (PWC; PWL constant) or 1/12 (PWL linear), eps_r: n_vox complex.
 * diag_term = 0 omits eps_r*g*x (component-sharded ranks other than 0).      */
int vie_system_matvec(vie_op op, const double* eps_r, double inv_v, const double* x, double* y,
                      int diag_term, void* stream);

/* A device linear map y = f(x) on vectors of n complex values (the reference's
 * LinearMap, solver.hpp:26), run on `stream` (the solve's stream).                  */
typedef void (*vie_linear_map_fn)(void* user, const double* x, double* y, void* stream);

/* Right preconditioner M (solver.hpp:34-36, :74, :131): w = A M v_j, x += M V y.
 * Either `diag` (device, n complex: M = diag(diag)) or `apply`/`user` (a callback).  */
typedef struct {
  const double* diag;
  vie_linear_map_fn apply;
  void* user;
} vie_precond;

/* gmres (solver.hpp:34-142) on apply_system, device resident: restarted
 * GMRES(inner), modified Gram-Schmidt, complex Givens rotations.  x0 may be
 * NULL (zero start); precond may be NULL (none).  history_host receives
 * |g_{j+1}|/||b|| per iteration (up to history_cap values; *history_len = total
 * count).  The solve runs on the context's stream, ordered after all work queued on
 * `stream` (NULL: the caller must have completed the producers of eps_r / rhs / x0);
 * `stream` then waits for the solve.  Returns after the result is on the host.
 * On a slab-partitioned operator with a communicator (vie_op_set_comm) every vector is
 * this rank's z-slab (vie_slab_info x_elems) and all ranks call it together.           */
int vie_gmres_solve(vie_op op, const double* eps_r, double inv_v, const double* rhs,
                    const double* x0, double tol, int inner, int outer, const vie_precond* precond,
                    double* x, int* iterations, double* final_rel_res, double* history_host,
                    int history_cap, int* history_len, int* converged, void* stream);

/* The same device GMRES on any linear map of n complex values: gmres(apply, rhs, cfg,
 * x0, precond) of solver.hpp:34 with the closure as a C callback.                   */
int vie_gmres(vie_ctx ctx, int64_t n, vie_linear_map_fn apply, void* apply_user, const double* rhs,
              const double* x0, double tol, int inner, int outer, const vie_precond* precond,
              double* x, int* iterations, double* final_rel_res, double* history_host,
              int history_cap, int* history_len, int* converged, void* stream);

/* ---- scene pipeline around the solve (solve_scene, solver.hpp:148-285) ----
 * PWC fields (3 component blocks of n_vox, grid.hpp:107-136).  The scene is the
 * reference's VoxelGrid (grid.hpp:24-46) + DielectricMap frequency (grid.hpp:52-75)
 * + PlaneWave (grid.hpp:78-100); polarization / direction are normalised here and
 * VIE_EINVAL is returned when they are not orthogonal (|p.d| > 1e-12, grid.hpp:86-87)
 * or when a resolution is not > 0 / a dim < 1 (grid.hpp:33-36).  ctx may be NULL:
 * the caller's current device and `stream` (NULL = legacy default stream).      */
typedef struct {
  int64_t dims[3];
  double resolution[3]; /* meters */
  double origin[3];     /* minimum corner */
  double frequency;     /* Hz */
  double polarization[3];
  double direction[3];
  double amplitude; /* V/m */
} vie_scene;

/* build_rhs (solver.hpp:148-179): rhs_q = c_e chi_e e_inc,q at the voxel centre
 * (quad_points_per_axis = 1) or the Gauss-integrated voxel average (> 1;
 * quadrature.hpp:23-52); voxels with chi_e = 0 get 0.  eps_r: n_vox complex
 * (device); rhs: 3 n_vox complex (device).                                       */
int vie_build_rhs(vie_ctx ctx, const vie_scene* scene, const double* eps_r, int quad_points_per_axis,
                  double* rhs, void* stream);

/* recover_fields (solver.hpp:211-249): e = j / (c_e chi_e) where chi_e != 0, else
 * e_inc(centre); when op_k != NULL (a VIE_KIND_K PWC operator on the same grid),
 * h = h_inc + (K j) / V through vie_matvec, else h is untouched (may be NULL).    */
int vie_recover_fields(vie_ctx ctx, const vie_scene* scene, const double* eps_r, const double* j,
                       vie_op op_k, double* e, double* h, void* stream);

/* postprocess (solver.hpp:258-284): p_abs = sigma_e |e|^2 / 2 (real, n_vox),
 * *total_absorbed_power_host = V sum p_abs (deterministic order-fixed sum);
 * when h != NULL, b1_plus = mu0 |h_x + i h_y| (real, n_vox).                    */
int vie_postprocess(vie_ctx ctx, const vie_scene* scene, const double* eps_r, const double* e,
                    const double* h, double* p_abs, double* b1_plus, double* total_absorbed_power_host,
                    void* stream);

/* Timing helpers for the bench: number of kernels the last vie_matvec
 * launched, and per-stage device times (ms) of the last vie_matvec when
 * profiling was enabled with vie_op_set_profiling(op, 1).                   */
/* ---- slab-decomposed matvec (multi-GPU) ----
 * Rank r of R owns the z-planes [r nk, (r+1) nk) of x and y (nk = n3 / R) and the
 * axis-1 spectral positions [r W, (r+1) W) (W = 2 n1 / R, whole pencil groups) of the
 * axis-2 / axis-3 stages.  One matvec = slab_forward (axis-1 FFTs) -> all-to-all (equal
 * chunks of slab_elems / R) -> slab_pencil (axis-2 FFTs, decompression of the rank's
 * octant rows, fused axis-3 FFT / Hadamard / IFFT, inverse axis-2 FFTs) -> all-to-all ->
 * slab_inverse (inverse axis-1 FFTs).  The exchanged buffers are blocked
 * [rank][s][k in block][j][w < W] so the chunk for rank q is contiguous (the caller runs
 * the collective, e.g. NCCL all_to_all).  With R = 1 the stages are vie_matvec in three. */
int vie_op_set_partition(vie_op op, int nranks, int rank);
/* x_elems = S n1 n2 nk (local x / y), slab_elems = S nk n2 2n1 (each exchange buffer),
 * k0 = first z-plane of this rank, nk = z-planes per rank                         */
int vie_slab_info(vie_op op, int64_t* x_elems, int64_t* slab_elems, int64_t* k0, int64_t* nk);
/* axis-1 FFTs of the local z-slab x_local -> send (blocked by destination rank)      */
int vie_slab_forward(vie_op op, const double* x_local, double* send, void* stream);
/* axis-2 FFTs of the rank's positions, decompression of its octant rows, fused
 * axis-3 FFT / Hadamard / IFFT, inverse axis-2 FFTs: recv -> out (blocked by rank)   */
int vie_slab_pencil(vie_op op, const double* recv, double* out, void* stream);
/* inverse axis-1 FFTs, crop, 1/N_e -> y_local; with eps_local the apply_system
 * epilogue y = eps g x - (eps - 1) inv_v (N x) (x_local needed when diag_term)       */
int vie_slab_inverse(vie_op op, const double* back, double* y_local, const double* eps_local, double inv_v,
                     const double* x_local, int diag_term, void* stream);

int vie_op_set_profiling(vie_op op, int enable);
int vie_op_last_stats(vie_op op, int* launches, double* stage_ms /* [8] */);

#ifdef __cplusplus
}
#endif
#endif
