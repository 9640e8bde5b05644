/*
 * vie_oracle.h -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * B200 product (paper_1811_00484_b200/).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * never links or calls it.
 *
 * It restates, function by function, the reference C++ library under
 * /root/reference/proj/include/vie (header-only, Eigen3 + FFTW3, neither of
 * which exists in this image, so the reference itself cannot be compiled).
 * Every entry point cites the reference file:line it follows.
 *
 * Conventions (all from the reference):
 *   - complex data is interleaved double (re, im) == std::complex<double>
 *   - Tensor3 layout: flat = i + n1*(j + n2*k)               tensor.hpp:20
 *   - factor matrices are column-major rows x cols             tensor.hpp:15-17
 *   - fields are component-major (block q, then q+1, ...)      grid.hpp:122-127
 *   - forward DFT: e^{-2 pi i pm/N}, unnormalised; inverse e^{+}, divided by N
 *                                                              fft.hpp:19-21,32-37
 * Errors: every function returns 0 on success, 1 for the reference's
 * std::invalid_argument cases; orc_last_error() holds the message.
 */
#ifndef VIE_ORACLE_H
#define VIE_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);
void orc_set_threads(int nthreads);

/* ---- seeded inputs (tests/test_util.hpp:9-31) -------------------------- */
int orc_random_tensor(int64_t n1, int64_t n2, int64_t n3, uint64_t seed, double* out);
int orc_random_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out);
/* generic stream: `count` complex values cplx(gauss(rng), gauss(rng)) */
int orc_gauss_stream(uint64_t seed, int64_t count, double* out);

/* ---- DFT service (fft.hpp:22-96) --------------------------------------- */
int orc_fft1(double* v, int64_t n, int inverse);
int orc_fft3(double* t, int64_t n1, int64_t n2, int64_t n3, int inverse);

/* ---- embedding / factor transform (operator.hpp:39-90) ----------------- */
int orc_circulant_embed(const double* t, const int64_t dims[3], const int sign[3], double* out);
int orc_transform_factor(const double* u, int64_t n, int64_t r, int sign, double* out);

/* ---- component tables (components.hpp:46-92, operator.hpp:205-219) ------
 * kind 0 = N, 1 = K ; basis 0 = PWC (reference), 1 = PWL (generalisation).
 * comps: ncomp x 4 ints (q, q', l, l'); parity: ncomp x 3 ints;
 * blocks: nblock x 4 ints (target, source, comp, dense_sign).  The FFT-path
 * coefficient of a block is dense_sign * prod(parity[comp]).               */
int orc_component_table(int kind, int basis, int* ncomp, int* comps, int* parity,
                        int* nblock, int* blocks);

/* ---- Tucker operator --------------------------------------------------
 * A component form is (ranks r1,r2,r3; core r1*r2*r3; U1 m1 x r1; U2 m2 x r2;
 * U3 m3 x r3) with factors already embedded + transformed (2n rows).
 * Forms are passed as arrays of pointers, one entry per component of the
 * canonical table of (kind, basis).                                        */
int orc_decompress_tucker(const int64_t edims[3], const int64_t ranks[3], const double* core,
                          const double* u1, const double* u2, const double* u3, double* dst);

/* decompress_cp (operator.hpp:248-261): slab_k = W1 diag(W3(k,:)) W2^T, merged
 * Fourier-domain Tucker+CP factors W_q (2n_q x rank, column-major).          */
int orc_decompress_cp(const int64_t edims[3], int64_t rank, const double* w1, const double* w2,
                      const double* w3, double* dst);

/* apply_operator (operator.hpp:273-382), strategy HosvdDecompress.         */
int orc_apply_operator_tucker(int kind, int basis, const int64_t grid[3], const int64_t* ranks,
                              const double* const* cores, const double* const* u1s,
                              const double* const* u2s, const double* const* u3s,
                              const double* x, double* y);
/* apply_operator strategy Dense: spectra = ncomp embedded-size spectra.    */
/* apply_operator_tucker as staged pieces of ONE matvec (the CPU baseline times them):
 * create (copies x; forms must stay alive), npieces = 2S + NC, piece(i) in order
 * (0..S-1 forward3 of current i, then components, then inverse3 of each target),
 * result(y), destroy.  Running all pieces == orc_apply_operator_tucker.             */
int orc_mv_create(int kind, int basis, const int64_t grid[3], const int64_t* ranks, const double* const* cores,
                  const double* const* u1s, const double* const* u2s, const double* const* u3s, const double* x,
                  void** handle);
int orc_mv_npieces(void* handle);
int orc_mv_piece(void* handle, int i);
int orc_mv_result(void* handle, double* y);
void orc_mv_destroy(void* handle);

int orc_apply_operator_dense(int kind, int basis, const int64_t grid[3],
                             const double* const* spectra, const double* x, double* y);
/* build the Dense spectrum of one spatial component (operator.hpp:158-162) */
int orc_dense_spectrum(const double* t, const int64_t dims[3], const int sign[3], double* out);

/* dense BTTB oracle (operator.hpp:388-434), generalised over the table.
 * tensors: ncomp spatial tensors n1*n2*n3; out: (T*Nv) x (S*Nv) column-major */
int orc_dense_bttb(int kind, int basis, const int64_t dims[3], const double* const* tensors,
                   double* out);

/* apply_system (solver.hpp:183-200): y = eps*g_l*x - (eps-1)*inv_v*(N x)   */
int orc_apply_system_tucker(int basis, const int64_t grid[3], const int64_t* ranks,
                            const double* const* cores, const double* const* u1s,
                            const double* const* u2s, const double* const* u3s,
                            const double* eps_r, double inv_v, const double* x, double* y);

/* ---- GMRES (solver.hpp:34-142) ----------------------------------------- */
typedef void (*orc_linmap)(const double* x, double* y, void* ctx);
int orc_gmres(orc_linmap apply, void* apply_ctx, orc_linmap precond, void* precond_ctx,
              int64_t n, const double* rhs, const double* x0, double tol, int inner, int outer,
              double* x, int* iterations, int* converged, double* final_rel_res,
              double* history, int history_cap, int* history_len);
/* GMRES on the Tucker system matvec (the solve_scene closure, solver.hpp:309-313) */
int orc_gmres_system_tucker(int basis, const int64_t grid[3], const int64_t* ranks,
                            const double* const* cores, const double* const* u1s,
                            const double* const* u2s, const double* const* u3s,
                            const double* eps_r, double inv_v, const double* rhs,
                            const double* x0, double tol, int inner, int outer, double* x,
                            int* iterations, int* converged, double* final_rel_res,
                            double* history, int history_cap, int* history_len);

/* ---- HOSVD (decomp.hpp:40-176) ----------------------------------------- */
int orc_truncated_svd_values(const double* m, int64_t rows, int64_t cols, double tol, int rule,
                             int64_t* rank, double* sigma /* min(rows,cols) */);
/* hosvd: query ranks first with out pointers NULL, then call again with
 * buffers sized core r1*r2*r3, U_q n_q*r_q.                                */
int orc_hosvd(const double* t, const int64_t dims[3], double tol, int rule, int64_t ranks[3],
              double* core, double* u1, double* u2, double* u3);
/* cp_als (decomp.hpp:237-298): f_q dims[q] x r (col-major, may be NULL), trace up to
 * trace_cap sweeps, flags = {converged, ill_posed_rank}. */
int orc_cp_als(const double* t, const int64_t dims[3], int64_t r, int max_iters, double stall_tol, uint64_t seed,
               double* f1, double* f2, double* f3, double* trace, int trace_cap, int* ntrace, int flags[2]);
/* tucker_cp (decomp.hpp:336-373): merged factors W_q (dims[q] x rank; NULL = rank only),
 * errs = {hosvd_relative_error, core_cp_relative_error, achieved_relative_error}. */
int orc_tucker_cp(const double* t, const int64_t dims[3], double tol, int cp_iters, int rule, int64_t cp_rank,
                  double stall_tol, int64_t* rank_out, double* w1, double* w2, double* w3, double errs[3],
                  double* trace, int trace_cap, int* ntrace);

/* solve_scene stages (solver.hpp:148-285), PWC fields (3 blocks of n_vox).
 * geo = {res0, res1, res2, org0, org1, org2}; pw = {pol0..2, dir0..2, amplitude}
 * (normalised here, grid.hpp:84-88).  kj may be NULL (no K operator, h untouched);
 * h may be NULL in postprocess (no b1).                                          */
int orc_build_rhs(const int64_t dims[3], const double geo[6], double frequency, const double pw[7],
                  const double* eps_r, int quad, double* rhs);
int orc_recover_fields(const int64_t dims[3], const double geo[6], double frequency, const double pw[7],
                       const double* eps_r, const double* j, const double* kj, double* e, double* h);
int orc_postprocess(const int64_t dims[3], const double geo[6], double frequency, const double* eps_r,
                    const double* e, const double* h, double* p_abs, double* b1, double* total);

/* ---- Green's-tensor assembly (assembly.hpp:159-233, kernels.hpp, quadrature.hpp) ----
 * op: 0 = N, 1 = K, 2 = scalar g (ScalarG), 3 = the N self remainder kernel (kernels.hpp:113);
 * quad5 = {far, near, near_radius, surface, volume} points (QuadratureSpec; NULL = defaults
 * 5, 10, 1, 12, 6).  out: n1 n2 n3 complex, SI units (entries scale as res^3 / ^4 / ^5).  */
int orc_assemble(const int64_t dims[3], const double res[3], double k0, int op, int q, int qp,
                 const int* quad5, double* out);
/* self_static_term (assembly.hpp:127-150): diagonal of the static nabla-nabla dyad      */
int orc_self_static_term(const double delta[3], const int* quad5, double dyad_diag[3], double* gram,
                         double* err, int* converged);
/* detail::correlation_entry (assembly.hpp:49-79) of kernel op at displacement d (voxel units) */
int orc_correlation_entry(int op, double k, int q, int qp, const double d[3], const double delta[3],
                          int points, int duffy, double* out);
int orc_kernel_eval(int op, double k, int q, int qp, const double r[3], double* out);
/* kernels::radial / radial_dynamic: (g, g', g'') interleaved complex                     */
int orc_radial(double R, double k, int dynamic, double* out6);
/* test_assembly.cpp:14-37 brute-force 6D pair integral                                   */
int orc_brute_pair_integral(int op, double k, int q, int qp, const double d[3], const double del[3],
                            int p, double* out);

#ifdef __cplusplus
}
#endif
#endif
