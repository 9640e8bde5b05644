// vie_b200.hpp -- C++ drop-in over the C ABI (vie_b200.h), mirroring the
// reference operator API (/root/reference/proj/include/vie, header-only C++):
//
//   reference                                  here (namespace vie::b200)
//   DftService            fft.hpp:13-96        DftService (CUDA device + stream + plans)
//   hosvd / TuckerForm     decomp.hpp:123-176   TuckerForm (spatial-domain forms)
//   component_parity       components.hpp:51    component_parity
//   build_operator_spectra operator.hpp:144     build_operator_spectra (Tucker only)
//   apply_operator         operator.hpp:273     apply_operator (HosvdDecompress semantics)
//   apply_system           solver.hpp:183       apply_system
//   gmres / GmresConfig    solver.hpp:12-142    gmres_system (device-resident GMRES)
//
// Same argument meaning and error behaviour: std::invalid_argument where the
// reference throws it (dim mismatch, missing representation, NoBuffer with a
// decompress strategy, bad GMRES config, non-finite rhs); std::runtime_error
// for CUDA failures.  Containers are plain std::vector<std::complex<double>>
// in the reference layouts (Tensor3: i + n1*(j + n2*k); factors column-major;
// fields component-major), so no Eigen is needed to use it.
#ifndef VIE_B200_HPP
#define VIE_B200_HPP

#include <cuda_runtime_api.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <functional>
#include <chrono>
#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#include "vie_b200.h"

namespace vie {
namespace b200 {

using cplx = std::complex<double>;
using Index = std::int64_t;

enum class OperatorKind { N = VIE_KIND_N, K = VIE_KIND_K };
enum class BasisOrder { PWC = VIE_BASIS_PWC, PWL = VIE_BASIS_PWL };
// operator.hpp:17 (Dense is the reference's uncompressed test path; not served here).
// *Decompress: all octant spectra in one HBM buffer; *Loop: the buffer-free fused kernel
// (vie_op_set_strategy).  CP forms are held as Tucker forms, so TuckerCp* select the same paths.
enum class MatvecStrategy { HosvdDecompress, HosvdLoop, TuckerCpDecompress, TuckerCpLoop };
enum class ScratchPolicy { WithBuffer, NoBuffer };

inline void check(int rc) {
  if (rc == VIE_OK) return;
  if (rc == VIE_EINVAL) throw std::invalid_argument(vie_last_error());
  throw std::runtime_error(std::string("vie_b200: ") + vie_last_error());
}
inline void cuda_check(cudaError_t e) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
}

// ------------------------------------------------------------------ containers
struct Tensor3 {  // tensor.hpp:17-71
  std::array<Index, 3> dims{0, 0, 0};
  std::vector<cplx> data;
  Tensor3() = default;
  Tensor3(Index n1, Index n2, Index n3) : dims{n1, n2, n3}, data(static_cast<size_t>(n1 * n2 * n3)) {
    if (n1 < 0 || n2 < 0 || n3 < 0) throw std::invalid_argument("Tensor3: negative dimension");
  }
  Index size() const { return static_cast<Index>(data.size()); }
  cplx& operator()(Index i, Index j, Index k) { return data[static_cast<size_t>(i + dims[0] * (j + dims[1] * k))]; }
  cplx operator()(Index i, Index j, Index k) const {
    return data[static_cast<size_t>(i + dims[0] * (j + dims[1] * k))];
  }
};

struct FactorMatrix {  // column-major rows x cols (Eigen::MatrixXcd layout)
  Index rows = 0, cols = 0;
  std::vector<cplx> data;
  FactorMatrix() = default;
  FactorMatrix(Index r, Index c) : rows(r), cols(c), data(static_cast<size_t>(r * c)) {}
  cplx& operator()(Index i, Index j) { return data[static_cast<size_t>(i + rows * j)]; }
  cplx operator()(Index i, Index j) const { return data[static_cast<size_t>(i + rows * j)]; }
};

enum class TruncationRule { SigmaMax = VIE_RULE_SIGMA_MAX, Energy = VIE_RULE_ENERGY };  // decomp.hpp:23

// Spatial-domain Tucker form as hosvd returns it (decomp.hpp:123-133).
struct TuckerForm {
  Tensor3 core;                          // r1 x r2 x r3
  std::array<FactorMatrix, 3> factors;   // n_q x r_q
  std::array<Index, 3> ranks{0, 0, 0};
  TruncationRule rule = TruncationRule::SigmaMax;
  double tol = 0.0;
};

// Spatial-domain Tucker+CP form, merged factors W_q = U_q V_q (decomp.hpp:143-148).
struct TuckerCPForm {
  std::array<FactorMatrix, 3> factors;  // n_q x rank
  Index rank = 0;
};

// ---- VIET container (container.hpp:15-159), byte-compatible with the reference's files
using ContainerValue = std::variant<Tensor3, TuckerForm, TuckerCPForm>;

inline void save_container(const std::string& path, const Tensor3& t) {
  const int64_t d[3] = {t.dims[0], t.dims[1], t.dims[2]}, r[3] = {0, 0, 0};
  check(vie_container_write(path.c_str(), 0, 0, 0.0, d, r, reinterpret_cast<const double*>(t.data.data())));
}
inline void save_container(const std::string& path, const TuckerForm& f, const std::array<Index, 3>& dims) {
  std::vector<cplx> p;
  for (const auto& u : f.factors) p.insert(p.end(), u.data.begin(), u.data.end());
  p.insert(p.end(), f.core.data.begin(), f.core.data.end());
  const int64_t d[3] = {dims[0], dims[1], dims[2]}, r[3] = {f.ranks[0], f.ranks[1], f.ranks[2]};
  check(vie_container_write(path.c_str(), 1, static_cast<int>(f.rule), f.tol, d, r,
                            reinterpret_cast<const double*>(p.data())));
}
inline void save_container(const std::string& path, const TuckerCPForm& f, const std::array<Index, 3>& dims) {
  std::vector<cplx> p;
  for (const auto& w : f.factors) p.insert(p.end(), w.data.begin(), w.data.end());
  const int64_t d[3] = {dims[0], dims[1], dims[2]}, r[3] = {f.rank, f.rank, f.rank};
  check(vie_container_write(path.c_str(), 2, 0, 0.0, d, r, reinterpret_cast<const double*>(p.data())));
}
inline ContainerValue load_container(const std::string& path) {
  int kind = 0, rule = 0;
  double tol = 0.0;
  int64_t d[3], r[3];
  check(vie_container_info(path.c_str(), &kind, &rule, &tol, d, r));
  int64_t n = kind == 0 ? d[0] * d[1] * d[2] : d[0] * r[0] + d[1] * r[1] + d[2] * r[2];
  if (kind == 1) n += r[0] * r[1] * r[2];
  std::vector<cplx> p(static_cast<size_t>(n));
  check(vie_container_read(path.c_str(), reinterpret_cast<double*>(p.data()), n));
  if (kind == 0) {
    Tensor3 t(d[0], d[1], d[2]);
    t.data = std::move(p);
    return t;
  }
  std::array<FactorMatrix, 3> fm;
  size_t off = 0;
  for (int q = 0; q < 3; ++q) {
    fm[q] = FactorMatrix(d[q], r[q]);
    std::copy(p.begin() + static_cast<std::ptrdiff_t>(off), p.begin() + static_cast<std::ptrdiff_t>(off + fm[q].data.size()),
              fm[q].data.begin());
    off += fm[q].data.size();
  }
  if (kind == 2) {
    TuckerCPForm f;
    f.factors = std::move(fm);
    f.rank = r[0];
    return f;
  }
  TuckerForm f;
  f.factors = std::move(fm);
  f.ranks = {r[0], r[1], r[2]};
  f.core = Tensor3(r[0], r[1], r[2]);
  std::copy(p.begin() + static_cast<std::ptrdiff_t>(off), p.end(), f.core.data.begin());
  f.rule = rule == 1 ? TruncationRule::Energy : TruncationRule::SigmaMax;
  f.tol = tol;
  return f;
}

struct KernelComponent {  // components.hpp:26-36 (+ PWL polynomial indices)
  OperatorKind op = OperatorKind::N;
  int row_axis = 0;
  int col_axis = 0;
  int row_poly = 0;  // l  (PWL: 0 constant, 1..3 linear in x, y, z)
  int col_poly = 0;  // l'
};

struct Parity {  // components.hpp:40-44
  std::array<int, 3> sign{1, 1, 1};
  int product() const { return sign[0] * sign[1] * sign[2]; }
};

// Reflection parity of a component (components.hpp:51-65; PWL: DESIGN.md).
inline Parity component_parity(const KernelComponent& c, BasisOrder order = BasisOrder::PWC) {
  int nc = 0, nb = 0;
  check(vie_component_table(static_cast<int>(c.op), static_cast<int>(order), &nc, nullptr, nullptr, &nb, nullptr));
  std::vector<int> comps(static_cast<size_t>(4 * nc)), par(static_cast<size_t>(3 * nc));
  check(vie_component_table(static_cast<int>(c.op), static_cast<int>(order), &nc, comps.data(), par.data(), &nb,
                            nullptr));
  for (int i = 0; i < nc; ++i) {
    const int* e = &comps[static_cast<size_t>(4 * i)];
    if (e[0] == c.row_axis && e[1] == c.col_axis && e[2] == c.row_poly && e[3] == c.col_poly)
      return Parity{{par[static_cast<size_t>(3 * i)], par[static_cast<size_t>(3 * i + 1)],
                     par[static_cast<size_t>(3 * i + 2)]}};
  }
  throw std::invalid_argument("component_parity: component not in the unique-component table");
}

// Unique components of (kind, order) in the canonical order (components.hpp:71-92).
inline std::vector<KernelComponent> unique_components(OperatorKind op, BasisOrder order = BasisOrder::PWC) {
  int nc = 0, nb = 0;
  check(vie_component_table(static_cast<int>(op), static_cast<int>(order), &nc, nullptr, nullptr, &nb, nullptr));
  std::vector<int> comps(static_cast<size_t>(4 * nc));
  check(vie_component_table(static_cast<int>(op), static_cast<int>(order), &nc, comps.data(), nullptr, &nb,
                            nullptr));
  std::vector<KernelComponent> out;
  for (int i = 0; i < nc; ++i)
    out.push_back({op, comps[static_cast<size_t>(4 * i)], comps[static_cast<size_t>(4 * i + 1)],
                   comps[static_cast<size_t>(4 * i + 2)], comps[static_cast<size_t>(4 * i + 3)]});
  return out;
}

struct CurrentField {  // grid.hpp:107-136 (PWC: 3 components, PWL: 12, s = 4q + l)
  BasisOrder order = BasisOrder::PWC;
  std::vector<Tensor3> comp;
  CurrentField() = default;
  explicit CurrentField(const std::array<Index, 3>& d, BasisOrder ord = BasisOrder::PWC) : order(ord) {
    comp.assign(ord == BasisOrder::PWC ? 3 : 12, Tensor3(d[0], d[1], d[2]));
  }
  std::array<Index, 3> dims() const { return comp.at(0).dims; }
  Index flat_size() const { return static_cast<Index>(comp.size()) * comp.at(0).size(); }
  std::vector<cplx> to_vector() const {
    std::vector<cplx> v;
    v.reserve(static_cast<size_t>(flat_size()));
    for (const auto& t : comp) v.insert(v.end(), t.data.begin(), t.data.end());
    return v;
  }
  static CurrentField from_vector(const std::vector<cplx>& v, const std::array<Index, 3>& d,
                                  BasisOrder ord = BasisOrder::PWC) {
    CurrentField f(d, ord);
    const size_t n = static_cast<size_t>(f.comp[0].size());
    if (v.size() != n * f.comp.size()) throw std::invalid_argument("CurrentField: vector size mismatch");
    for (size_t q = 0; q < f.comp.size(); ++q)
      std::copy(v.begin() + static_cast<long>(q * n), v.begin() + static_cast<long>((q + 1) * n),
                f.comp[q].data.begin());
    return f;
  }
};

// ------------------------------------------------------------------ device RAII
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t bytes) : bytes_(bytes) { cuda_check(cudaMalloc(&p_, bytes)); }
  ~DeviceBuffer() {
    if (p_) cudaFree(p_);
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), bytes_(o.bytes_) { o.p_ = nullptr; }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
      if (p_) cudaFree(p_);
      p_ = o.p_;
      bytes_ = o.bytes_;
      o.p_ = nullptr;
    }
    return *this;
  }
  double* get() const { return static_cast<double*>(p_); }
  // Copies ordered on `st` (the context stream the library's kernels run on) and complete
  // on return: a plain cudaMemcpy runs on the legacy stream, which does not order with the
  // context's non-blocking stream, and a pageable H2D copy may return before it lands.
  void upload(const void* h, size_t bytes, cudaStream_t st) {
    cuda_check(cudaMemcpyAsync(p_, h, bytes, cudaMemcpyHostToDevice, st));
    cuda_check(cudaStreamSynchronize(st));
  }
  void download(void* h, size_t bytes, cudaStream_t st) const {
    cuda_check(cudaMemcpyAsync(h, p_, bytes, cudaMemcpyDeviceToHost, st));
    cuda_check(cudaStreamSynchronize(st));
  }

 private:
  void* p_ = nullptr;
  size_t bytes_ = 0;
};

class DftService {  // fft.hpp DftService: here the CUDA context, stream and plan cache
 public:
  explicit DftService(int device = 0) { check(vie_ctx_create(&ctx_, device)); }
  // releases the caller's reference; operators built on it keep the context alive
  ~DftService() { vie_ctx_destroy(ctx_); }
  DftService(const DftService&) = delete;
  DftService& operator=(const DftService&) = delete;
  vie_ctx handle() const { return ctx_; }
  cudaStream_t stream() const {
    void* s = nullptr;
    check(vie_ctx_stream(ctx_, &s));
    return static_cast<cudaStream_t>(s);
  }

 private:
  vie_ctx ctx_ = nullptr;
};

// ---- CP-ALS and Tucker+CP (decomp.hpp:135-148, 184-373)
struct CPForm {  // decomp.hpp:135-140
  std::array<FactorMatrix, 3> factors;
  Index rank = 0;
};
struct CpAlsResult {  // decomp.hpp:184-190
  CPForm form;
  std::vector<double> rel_error_trace;  // one entry per completed sweep
  bool converged = false;
  bool ill_posed_rank = false;
};
// cp_als (decomp.hpp:237-298): the library's host CP-ALS (sized for Tucker cores)
inline CpAlsResult cp_als(const Tensor3& t, Index r, int max_iters = 100, double stall_tol = 1e-12,
                          std::uint64_t seed = 0x5eed) {
  CpAlsResult res;
  res.form.rank = r;
  const int64_t d[3] = {t.dims[0], t.dims[1], t.dims[2]};
  for (int q = 0; q < 3; ++q) res.form.factors[static_cast<size_t>(q)] = FactorMatrix(d[q], std::max<Index>(r, 0));
  std::vector<double> tr(static_cast<size_t>(std::max(max_iters, 1)) + 1);
  int nt = 0, flags[2] = {0, 0};
  check(vie_cp_als(d, reinterpret_cast<const double*>(t.data.data()), r, max_iters, stall_tol, seed,
                   reinterpret_cast<double*>(res.form.factors[0].data.data()),
                   reinterpret_cast<double*>(res.form.factors[1].data.data()),
                   reinterpret_cast<double*>(res.form.factors[2].data.data()), tr.data(), static_cast<int>(tr.size()),
                   &nt, flags));
  res.rel_error_trace.assign(tr.begin(), tr.begin() + std::min<size_t>(static_cast<size_t>(nt), tr.size()));
  res.converged = flags[0] != 0;
  res.ill_posed_rank = flags[1] != 0;
  return res;
}

struct CompressionStats {  // decomp.hpp:150-156
  std::int64_t original_elements = 0;
  std::int64_t compressed_elements = 0;
  double compression_factor = 0.0;
  double achieved_relative_error = 0.0;
  std::array<Index, 3> ranks{0, 0, 0};
};
struct TuckerCpResult {  // decomp.hpp:300-307
  TuckerCPForm form;
  CompressionStats stats;
  double hosvd_relative_error = 0.0;
  double core_cp_relative_error = 0.0;
  std::vector<double> cp_error_trace;
};
// tucker_cp (decomp.hpp:336-373): HOSVD on the device of `dft`, CP-ALS on the core, merged
// factors; every residual norm on the device.  `parity_sign` is only checked (odd axes must
// have a zero offset-0 plane) -- the spatial result does not depend on it.
inline TuckerCpResult tucker_cp(const Tensor3& t, double tol, int cp_iters, TruncationRule rule, Index cp_rank,
                                double stall_tol, DftService& dft, const std::array<int, 3>& parity_sign = {1, 1, 1}) {
  const int64_t d[3] = {t.dims[0], t.dims[1], t.dims[2]};
  const int64_t cap = cp_rank >= 0 ? cp_rank : std::min({d[0], d[1], d[2]});
  std::array<std::vector<cplx>, 3> w;
  for (int q = 0; q < 3; ++q) w[static_cast<size_t>(q)].assign(static_cast<size_t>(std::max<int64_t>(d[q] * cap, 1)), 0.0);
  std::vector<double> tr(static_cast<size_t>(std::max(cp_iters, 1)) + 1);
  int64_t rank = 0;
  double errs[3] = {0, 0, 0};
  int nt = 0;
  check(vie_tucker_cp(dft.handle(), d, reinterpret_cast<const double*>(t.data.data()), 0, parity_sign.data(), tol,
                      static_cast<int>(rule), cp_iters, cp_rank, stall_tol, nullptr, &rank,
                      reinterpret_cast<double*>(w[0].data()), reinterpret_cast<double*>(w[1].data()),
                      reinterpret_cast<double*>(w[2].data()), cap, errs, tr.data(), static_cast<int>(tr.size()), &nt,
                      nullptr));
  TuckerCpResult res;
  res.form.rank = rank;
  for (int q = 0; q < 3; ++q) {
    FactorMatrix f(d[q], rank);
    std::copy(w[static_cast<size_t>(q)].begin(), w[static_cast<size_t>(q)].begin() + d[q] * rank, f.data.begin());
    res.form.factors[static_cast<size_t>(q)] = std::move(f);
  }
  res.hosvd_relative_error = errs[0];
  res.core_cp_relative_error = errs[1];
  res.cp_error_trace.assign(tr.begin(), tr.begin() + std::min<size_t>(static_cast<size_t>(nt), tr.size()));
  res.stats.original_elements = d[0] * d[1] * d[2];  // compression_stats(TuckerCPForm) (decomp.hpp:324-334)
  res.stats.ranks = {rank, rank, rank};
  res.stats.compressed_elements = rank * (d[0] + d[1] + d[2]);
  res.stats.compression_factor = static_cast<double>(res.stats.original_elements) /
                                 static_cast<double>(std::max<std::int64_t>(res.stats.compressed_elements, 1));
  res.stats.achieved_relative_error = errs[2];
  return res;
}
// the reference signature: a temporary context on device 0
inline TuckerCpResult tucker_cp(const Tensor3& t, double tol, int cp_iters = 1000,
                                TruncationRule rule = TruncationRule::Energy, Index cp_rank = -1,
                                double stall_tol = 0.0) {
  DftService dft(0);
  return tucker_cp(t, tol, cp_iters, rule, cp_rank, stall_tol, dft);
}

struct ApplyWorkspace {};  // the device workspace lives in the operator (operator.hpp:181-187)

struct ApplyTimings {  // operator.hpp:189-192
  double fft_ms = 0.0;      // row / column FFT passes (pad, axes 1-2 and their inverses, crop)
  double product_ms = 0.0;  // decompression + fused axis-3 FFT x Hadamard x IFFT
};

class EmbeddedSpectrum {  // operator.hpp:120-129, Tucker representation only
 public:
  EmbeddedSpectrum() = default;
  EmbeddedSpectrum(vie_op op, OperatorKind k, BasisOrder b, std::array<Index, 3> g)
      : op_(op), kind(k), order(b), grid_dims(g), embedded_dims{2 * g[0], 2 * g[1], 2 * g[2]} {}
  ~EmbeddedSpectrum() {
    if (op_) vie_op_destroy(op_);
  }
  EmbeddedSpectrum(const EmbeddedSpectrum&) = delete;
  EmbeddedSpectrum& operator=(const EmbeddedSpectrum&) = delete;
  EmbeddedSpectrum(EmbeddedSpectrum&& o) noexcept
      : op_(o.op_), kind(o.kind), order(o.order), grid_dims(o.grid_dims), embedded_dims(o.embedded_dims) {
    o.op_ = nullptr;
  }
  vie_op handle() const { return op_; }
  cudaStream_t stream() const {  // the context stream its kernels run on
    void* s = nullptr;
    check(vie_op_stream(op_, &s));
    return static_cast<cudaStream_t>(s);
  }
  Index n_cur() const { return order == BasisOrder::PWC ? 3 : 12; }
  Index n_vox() const { return grid_dims[0] * grid_dims[1] * grid_dims[2]; }

 private:
  vie_op op_ = nullptr;

 public:
  OperatorKind kind = OperatorKind::N;
  BasisOrder order = BasisOrder::PWC;
  std::array<Index, 3> grid_dims{0, 0, 0};
  std::array<Index, 3> embedded_dims{0, 0, 0};
};

// build_operator_spectra (operator.hpp:144-177) from spatial Tucker forms: the
// forms are shipped to the device and transform_factors (embedding + 1D DFT
// of each factor column, operator.hpp:76-90) runs there.
inline EmbeddedSpectrum build_operator_spectra(OperatorKind kind, BasisOrder order,
                                               const std::vector<std::pair<KernelComponent, TuckerForm>>& forms,
                                               DftService& dft) {
  if (forms.empty()) throw std::invalid_argument("build_operator_spectra: no components");
  const std::array<Index, 3> grid{forms.front().second.factors[0].rows, forms.front().second.factors[1].rows,
                                  forms.front().second.factors[2].rows};
  std::vector<vie_tucker> hs;
  std::vector<int> comps;
  struct Guard {
    std::vector<vie_tucker>& h;
    ~Guard() {
      for (auto t : h) vie_tucker_destroy(t);
    }
  } guard{hs};
  for (const auto& [comp, f] : forms) {
    if (comp.op != kind) throw std::invalid_argument("build_operator_spectra: component of another operator");
    const Parity p = component_parity(comp, order);
    const Index r[3] = {f.factors[0].cols, f.factors[1].cols, f.factors[2].cols};
    const int64_t dims[3] = {f.factors[0].rows, f.factors[1].rows, f.factors[2].rows};
    if (dims[0] != grid[0] || dims[1] != grid[1] || dims[2] != grid[2])
      throw std::invalid_argument("build_operator_spectra: inconsistent component dims");
    if (static_cast<Index>(f.core.data.size()) != r[0] * r[1] * r[2])
      throw std::invalid_argument("build_operator_spectra: core size does not match the factor ranks");
    const int64_t ranks[3] = {r[0], r[1], r[2]};
    vie_tucker t = nullptr;
    check(vie_tucker_from_factors(dft.handle(), dims, ranks, reinterpret_cast<const double*>(f.core.data.data()),
                                  reinterpret_cast<const double*>(f.factors[0].data.data()),
                                  reinterpret_cast<const double*>(f.factors[1].data.data()),
                                  reinterpret_cast<const double*>(f.factors[2].data.data()), p.sign.data(), 0, &t));
    hs.push_back(t);
    comps.insert(comps.end(), {comp.row_axis, comp.col_axis, comp.row_poly, comp.col_poly});
  }
  const int64_t g[3] = {grid[0], grid[1], grid[2]};
  vie_op op = nullptr;
  check(vie_op_create(dft.handle(), static_cast<int>(kind), static_cast<int>(order), g, static_cast<int>(hs.size()),
                      comps.data(), hs.data(), &op));
  return EmbeddedSpectrum(op, kind, order, grid);
}

// build_operator_spectra from Tucker+CP forms (the reference's tucker_cp
// representation, operator.hpp:92-106 + 144-177): vie_tucker_from_cp per component.
inline EmbeddedSpectrum build_operator_spectra(OperatorKind kind, BasisOrder order,
                                               const std::vector<std::pair<KernelComponent, TuckerCPForm>>& forms,
                                               DftService& dft) {
  if (forms.empty()) throw std::invalid_argument("build_operator_spectra: no components");
  const std::array<Index, 3> grid{forms.front().second.factors[0].rows, forms.front().second.factors[1].rows,
                                  forms.front().second.factors[2].rows};
  std::vector<vie_tucker> hs;
  std::vector<int> comps;
  struct Guard {
    std::vector<vie_tucker>& h;
    ~Guard() {
      for (auto t : h) vie_tucker_destroy(t);
    }
  } guard{hs};
  for (const auto& [comp, f] : forms) {
    if (comp.op != kind) throw std::invalid_argument("build_operator_spectra: component of another operator");
    for (int q = 0; q < 3; ++q)
      if (f.factors[q].rows != grid[q] || f.factors[q].cols != f.rank)
        throw std::invalid_argument("build_operator_spectra: inconsistent Tucker+CP factor shapes");
    const Parity p = component_parity(comp, order);
    const int64_t dims[3] = {grid[0], grid[1], grid[2]};
    vie_tucker t = nullptr;
    check(vie_tucker_from_cp(dft.handle(), dims, f.rank, reinterpret_cast<const double*>(f.factors[0].data.data()),
                             reinterpret_cast<const double*>(f.factors[1].data.data()),
                             reinterpret_cast<const double*>(f.factors[2].data.data()), p.sign.data(), 0, &t));
    hs.push_back(t);
    comps.insert(comps.end(), {comp.row_axis, comp.col_axis, comp.row_poly, comp.col_poly});
  }
  const int64_t g[3] = {grid[0], grid[1], grid[2]};
  vie_op op = nullptr;
  check(vie_op_create(dft.handle(), static_cast<int>(kind), static_cast<int>(order), g, static_cast<int>(hs.size()),
                      comps.data(), hs.data(), &op));
  return EmbeddedSpectrum(op, kind, order, grid);
}


struct SpectrumBuildOptions {  // operator.hpp:131-139 (one compressed representation per component)
  double tol = 1e-8;
  TruncationRule rule = TruncationRule::Energy;
  BasisOrder order = BasisOrder::PWC;
  bool tucker_cp = false;  // compress with tucker_cp (TuckerCPForm) instead of hosvd (TuckerForm)
  int cp_iters = 1000;
  Index cp_rank = -1;      // default min(r1, r2, r3)
};

// build_operator_spectra (operator.hpp:144-177) from SPATIAL defining tensors,
// exactly the reference signature: each component is compressed by
// tucker_compress (hosvd + transform_factors) and kept only as a Tucker form.
inline EmbeddedSpectrum build_operator_spectra(OperatorKind kind,
                                               const std::vector<std::pair<KernelComponent, Tensor3>>& tensors,
                                               const SpectrumBuildOptions& opts, DftService& dft) {
  if (tensors.empty()) throw std::invalid_argument("build_operator_spectra: no components");
  const std::array<Index, 3> grid = tensors.front().second.dims;
  std::vector<vie_tucker> hs;
  std::vector<int> comps;
  struct Guard {
    std::vector<vie_tucker>& h;
    ~Guard() {
      for (auto t : h) vie_tucker_destroy(t);
    }
  } guard{hs};
  for (const auto& [comp, t] : tensors) {
    if (t.dims != grid) throw std::invalid_argument("build_operator_spectra: inconsistent component dims");
    const Parity p = component_parity(comp, opts.order);
    const int64_t dims[3] = {grid[0], grid[1], grid[2]};
    int64_t ranks[3] = {0, 0, 0};
    vie_tucker h = nullptr;
    if (opts.tucker_cp)  // operator.hpp:165-168: tucker_cp, then transform_factors(TuckerCPForm)
      check(vie_tucker_cp(dft.handle(), dims, reinterpret_cast<const double*>(t.data.data()), 0, p.sign.data(),
                          opts.tol, static_cast<int>(opts.rule), opts.cp_iters, opts.cp_rank, 0.0, &h, nullptr,
                          nullptr, nullptr, nullptr, 0, nullptr, nullptr, 0, nullptr, nullptr));
    else
      check(vie_tucker_compress(dft.handle(), dims, reinterpret_cast<const double*>(t.data.data()), p.sign.data(),
                                opts.tol, static_cast<int>(opts.rule), &h, ranks));
    hs.push_back(h);
    comps.insert(comps.end(), {comp.row_axis, comp.col_axis, comp.row_poly, comp.col_poly});
  }
  const int64_t g[3] = {grid[0], grid[1], grid[2]};
  vie_op op = nullptr;
  check(vie_op_create(dft.handle(), static_cast<int>(kind), static_cast<int>(opts.order), g,
                      static_cast<int>(hs.size()), comps.data(), hs.data(), &op));
  return EmbeddedSpectrum(op, kind, opts.order, grid);
}

inline bool is_loop(MatvecStrategy s) { return s == MatvecStrategy::HosvdLoop || s == MatvecStrategy::TuckerCpLoop; }
inline void set_strategy(const EmbeddedSpectrum& op, MatvecStrategy s) {
  check(vie_op_set_strategy(op.handle(), is_loop(s) ? VIE_STRATEGY_HOSVD_LOOP : VIE_STRATEGY_HOSVD_DECOMPRESS));
}

// apply_operator (operator.hpp:273-382).  Host containers in/out; the matvec
// runs on the device (vie_matvec_host: H2D, matvec, D2H).
// With `timings` (ApplyTimings, operator.hpp:189-192) the device stages run serialised
// between CUDA events (vie_matvec_timed) and the split is returned.
inline CurrentField apply_operator(const EmbeddedSpectrum& op, const CurrentField& x, MatvecStrategy strategy,
                                   ScratchPolicy policy, ApplyWorkspace* ws, DftService& dft,
                                   ApplyTimings* timings = nullptr) {
  (void)ws;
  (void)dft;
  if (x.dims() != op.grid_dims || static_cast<Index>(x.comp.size()) != op.n_cur())
    throw std::invalid_argument("apply_operator: dim mismatch");
  if (!is_loop(strategy) && policy == ScratchPolicy::NoBuffer)
    throw std::invalid_argument("apply_operator: decompress strategies need ScratchPolicy::WithBuffer");
  set_strategy(op, strategy);
  const std::vector<cplx> xv = x.to_vector();
  std::vector<cplx> yv(xv.size());
  if (!timings) {
    check(vie_matvec_host(op.handle(), reinterpret_cast<const double*>(xv.data()),
                          reinterpret_cast<double*>(yv.data())));
  } else {
    const cudaStream_t st = op.stream();
    const size_t bytes = xv.size() * sizeof(cplx);
    DeviceBuffer dx(bytes), dy(bytes);
    dx.upload(xv.data(), bytes, st);
    check(vie_matvec_timed(op.handle(), dx.get(), dy.get(), &timings->fft_ms, &timings->product_ms));
    dy.download(yv.data(), bytes, st);
  }
  return CurrentField::from_vector(yv, op.grid_dims, op.order);
}

struct MatvecBenchResult {  // operator.hpp:440-450
  MatvecStrategy strategy = MatvecStrategy::HosvdDecompress;
  std::array<Index, 3> embedded_dims{0, 0, 0};
  double median_ms = 0.0;
  double product_ms = 0.0;      // median over repetitions
  double product_min_ms = 0.0;  // minimum
  double fft_ms = 0.0;
  int repetitions = 0;
};

// matvec_bench (operator.hpp:451-502): warm-up, then `repetitions` timed device applies
// (x resident on the device, CUDA events; the stage split from vie_matvec_timed).
inline MatvecBenchResult matvec_bench(const EmbeddedSpectrum& op, const CurrentField& x, MatvecStrategy strategy,
                                      int repetitions, DftService& dft) {
  (void)dft;
  if (repetitions < 1) throw std::invalid_argument("matvec_bench: repetitions must be >= 1");
  if (x.dims() != op.grid_dims || static_cast<Index>(x.comp.size()) != op.n_cur())
    throw std::invalid_argument("apply_operator: dim mismatch");
  MatvecBenchResult r;
  r.strategy = strategy;
  r.embedded_dims = op.embedded_dims;
  r.repetitions = repetitions;
  const cudaStream_t st = op.stream();
  const std::vector<cplx> xv = x.to_vector();
  const size_t bytes = xv.size() * sizeof(cplx);
  DeviceBuffer dx(bytes), dy(bytes);
  dx.upload(xv.data(), bytes, st);
  check(vie_matvec(op.handle(), dx.get(), dy.get(), nullptr));  // warm-up
  cudaEvent_t e0, e1;
  cuda_check(cudaEventCreate(&e0));
  cuda_check(cudaEventCreate(&e1));
  std::vector<double> total, prod, fft;
  for (int rep = 0; rep < repetitions; ++rep) {
    cuda_check(cudaEventRecord(e0, st));
    check(vie_matvec(op.handle(), dx.get(), dy.get(), nullptr));
    cuda_check(cudaEventRecord(e1, st));
    cuda_check(cudaEventSynchronize(e1));
    float ms = 0.f;
    cuda_check(cudaEventElapsedTime(&ms, e0, e1));
    total.push_back(ms);
    double f = 0.0, p = 0.0;
    check(vie_matvec_timed(op.handle(), dx.get(), dy.get(), &f, &p));
    fft.push_back(f);
    prod.push_back(p);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  auto median = [](std::vector<double> v) {
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
  };
  r.median_ms = median(total);
  r.product_ms = median(prod);
  r.product_min_ms = *std::min_element(prod.begin(), prod.end());
  r.fft_ms = median(fft);
  return r;
}

// Many independent applications from host memory (vie_matvec_host_batch): the copies
// of neighbouring fields overlap each device matvec (full overlap needs pinned memory;
// with pageable std::vector storage the results are identical, the copies serialise).
inline std::vector<CurrentField> apply_operator_batch(const EmbeddedSpectrum& op, const std::vector<CurrentField>& xs) {
  std::vector<std::vector<cplx>> xv, yv;
  std::vector<const double*> xp;
  std::vector<double*> yp;
  for (const CurrentField& x : xs) {
    if (x.dims() != op.grid_dims || static_cast<Index>(x.comp.size()) != op.n_cur())
      throw std::invalid_argument("apply_operator: dim mismatch");
    xv.push_back(x.to_vector());
    yv.emplace_back(xv.back().size());
  }
  for (size_t i = 0; i < xs.size(); ++i) {
    xp.push_back(reinterpret_cast<const double*>(xv[i].data()));
    yp.push_back(reinterpret_cast<double*>(yv[i].data()));
  }
  check(vie_matvec_host_batch(op.handle(), static_cast<int64_t>(xs.size()), xp.data(), yp.data()));
  std::vector<CurrentField> ys;
  for (const auto& y : yv) ys.push_back(CurrentField::from_vector(y, op.grid_dims, op.order));
  return ys;
}

// apply_system (solver.hpp:183-200) with eps_r per voxel (n_vox values) and
// inv_v = 1 / voxel volume.
inline CurrentField apply_system(const std::vector<cplx>& eps_r, double inv_v, const EmbeddedSpectrum& op_n,
                                 const CurrentField& x) {
  if (x.dims() != op_n.grid_dims || static_cast<Index>(eps_r.size()) != op_n.n_vox())
    throw std::invalid_argument("apply_system: dim mismatch");
  const std::vector<cplx> xv = x.to_vector();
  const size_t bytes = xv.size() * sizeof(cplx);
  const cudaStream_t st = op_n.stream();
  DeviceBuffer dx(bytes), dy(bytes), de(eps_r.size() * sizeof(cplx));
  dx.upload(xv.data(), bytes, st);
  de.upload(eps_r.data(), eps_r.size() * sizeof(cplx), st);
  check(vie_system_matvec(op_n.handle(), de.get(), inv_v, dx.get(), dy.get(), 1, nullptr));
  std::vector<cplx> yv(xv.size());
  dy.download(yv.data(), bytes, st);
  return CurrentField::from_vector(yv, op_n.grid_dims, op_n.order);
}

struct GmresConfig {  // solver.hpp:12-16
  double tolerance = 1e-5;
  int inner = 50;
  int outer = 200;
};

struct GmresResult {  // solver.hpp:18-24
  std::vector<cplx> solution;
  std::vector<double> residual_history;
  double final_relative_residual = 0.0;
  int iterations = 0;
  bool converged = false;
};

// gmres (solver.hpp:34-142) on the apply_system closure of solve_scene
// (solver.hpp:309-313), device resident.  precond_diag: optional diagonal right
// preconditioner M = diag(precond_diag) (solver.hpp:74, :131).
inline GmresResult gmres_system(const std::vector<cplx>& eps_r, double inv_v, const EmbeddedSpectrum& op_n,
                                const std::vector<cplx>& rhs, const GmresConfig& cfg = {},
                                const std::vector<cplx>* x0 = nullptr,
                                const std::vector<cplx>* precond_diag = nullptr) {
  const size_t n = static_cast<size_t>(op_n.n_cur() * op_n.n_vox());
  if (rhs.size() != n || static_cast<Index>(eps_r.size()) != op_n.n_vox())
    throw std::invalid_argument("gmres: size mismatch");
  if (x0 && x0->size() != n) throw std::invalid_argument("gmres: initial guess size mismatch");
  if (precond_diag && precond_diag->size() != n) throw std::invalid_argument("gmres: preconditioner size mismatch");
  const size_t bytes = n * sizeof(cplx);
  const cudaStream_t st = op_n.stream();
  DeviceBuffer db(bytes), dx(bytes), de(eps_r.size() * sizeof(cplx));
  db.upload(rhs.data(), bytes, st);
  de.upload(eps_r.data(), eps_r.size() * sizeof(cplx), st);
  DeviceBuffer dx0, dpc;
  if (x0) {
    dx0 = DeviceBuffer(bytes);
    dx0.upload(x0->data(), bytes, st);
  }
  vie_precond pc{nullptr, nullptr, nullptr};
  if (precond_diag) {
    dpc = DeviceBuffer(bytes);
    dpc.upload(precond_diag->data(), bytes, st);
    pc.diag = dpc.get();
  }
  GmresResult res;
  std::vector<double> hist(static_cast<size_t>(cfg.inner) * static_cast<size_t>(cfg.outer) + 1);
  int it = 0, hl = 0, cv = 0;
  double fr = 0.0;
  check(vie_gmres_solve(op_n.handle(), de.get(), inv_v, db.get(), x0 ? dx0.get() : nullptr, cfg.tolerance, cfg.inner,
                        cfg.outer, precond_diag ? &pc : nullptr, dx.get(), &it, &fr, hist.data(),
                        static_cast<int>(hist.size()), &hl, &cv, nullptr));
  res.solution.resize(n);
  dx.download(res.solution.data(), bytes, st);
  res.residual_history.assign(hist.begin(), hist.begin() + std::min<long>(hl, static_cast<long>(hist.size())));
  res.final_relative_residual = fr;
  res.iterations = it;
  res.converged = cv != 0;
  return res;
}

// gmres(apply, rhs, cfg, x0, precond) with the reference's signature (solver.hpp:26,
// :34-36): host closures on std::vector, run by the device GMRES (vie_gmres); every
// application of a closure round-trips its vector through the host.
using LinearMap = std::function<std::vector<cplx>(const std::vector<cplx>&)>;

namespace detail {
struct HostMap {
  const LinearMap* f;
  size_t n;
  std::vector<cplx> in;
  static void call(void* user, const double* x, double* y, void* stream) {
    auto* h = static_cast<HostMap*>(user);
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    h->in.resize(h->n);
    cuda_check(cudaMemcpyAsync(h->in.data(), x, h->n * sizeof(cplx), cudaMemcpyDeviceToHost, st));
    cuda_check(cudaStreamSynchronize(st));
    const std::vector<cplx> out = (*h->f)(h->in);
    if (out.size() != h->n) throw std::invalid_argument("gmres: linear map changed the vector size");
    cuda_check(cudaMemcpyAsync(y, out.data(), h->n * sizeof(cplx), cudaMemcpyHostToDevice, st));
    cuda_check(cudaStreamSynchronize(st));
  }
};
}  // namespace detail

inline GmresResult gmres(const LinearMap& apply, const std::vector<cplx>& rhs, const GmresConfig& cfg = {},
                         const std::vector<cplx>* x0 = nullptr, const LinearMap& precond = nullptr,
                         DftService* dft = nullptr) {
  for (const cplx& v : rhs)
    if (!std::isfinite(v.real()) || !std::isfinite(v.imag()))
      throw std::invalid_argument("gmres: non-finite right-hand side");
  if (cfg.tolerance < 0 || cfg.inner < 1 || cfg.outer < 1) throw std::invalid_argument("gmres: invalid configuration");
  const size_t n = rhs.size();
  if (x0 && x0->size() != n) throw std::invalid_argument("gmres: initial guess size mismatch");
  DftService own(0);
  DftService& d = dft ? *dft : own;
  const cudaStream_t st = d.stream();
  const size_t bytes = n * sizeof(cplx);
  DeviceBuffer db(bytes), dx(bytes), dx0;
  db.upload(rhs.data(), bytes, st);
  if (x0) {
    dx0 = DeviceBuffer(bytes);
    dx0.upload(x0->data(), bytes, st);
  }
  detail::HostMap ha{&apply, n, {}}, hp{&precond, n, {}};
  vie_precond pc{nullptr, &detail::HostMap::call, &hp};
  GmresResult res;
  std::vector<double> hist(static_cast<size_t>(cfg.inner) * static_cast<size_t>(cfg.outer) + 1);
  int it = 0, hl = 0, cv = 0;
  double fr = 0.0;
  check(vie_gmres(d.handle(), static_cast<int64_t>(n), &detail::HostMap::call, &ha, db.get(), x0 ? dx0.get() : nullptr,
                  cfg.tolerance, cfg.inner, cfg.outer, precond ? &pc : nullptr, dx.get(), &it, &fr, hist.data(),
                  static_cast<int>(hist.size()), &hl, &cv, nullptr));
  res.solution.resize(n);
  dx.download(res.solution.data(), bytes, st);
  res.residual_history.assign(hist.begin(), hist.begin() + std::min<long>(hl, static_cast<long>(hist.size())));
  res.final_relative_residual = fr;
  res.iterations = it;
  res.converged = cv != 0;
  return res;
}

// ------------------------------------------------------------------ solve_scene stages
struct VoxelGrid {  // grid.hpp:24-46
  std::array<Index, 3> dims{1, 1, 1};
  std::array<double, 3> resolution{1.0, 1.0, 1.0};
  std::array<double, 3> origin{0.0, 0.0, 0.0};
  Index num_voxels() const { return dims[0] * dims[1] * dims[2]; }
  double voxel_volume() const { return resolution[0] * resolution[1] * resolution[2]; }
};

struct DielectricMap {  // grid.hpp:52-75: eps_r per voxel, flat = i + n1 (j + n2 k)
  VoxelGrid grid;
  std::vector<cplx> eps_r;
  double frequency = 0.0;
  DielectricMap() = default;
  DielectricMap(const VoxelGrid& g, double f)
      : grid(g), eps_r(static_cast<size_t>(g.num_voxels()), cplx(1.0)), frequency(f) {}
  cplx& eps(Index i, Index j, Index k) { return eps_r[static_cast<size_t>(i + grid.dims[0] * (j + grid.dims[1] * k))]; }
  void set_voxel(Index i, Index j, Index k, double eps_prime, double sigma) {  // grid.hpp:72-74
    eps(i, j, k) = cplx(eps_prime, -sigma / (8.8541878128e-12 * 2.0 * 3.141592653589793238462643383279502884 * frequency));
  }
};

struct PlaneWave {  // grid.hpp:78-100 (normalised and checked by the library)
  std::array<double, 3> polarization{1.0, 0.0, 0.0};
  std::array<double, 3> direction{0.0, 0.0, 1.0};
  double amplitude = 1.0;
};

inline vie_scene make_scene(const DielectricMap& m, const PlaneWave& inc) {
  vie_scene s{};
  for (int a = 0; a < 3; ++a) {
    s.dims[a] = m.grid.dims[a];
    s.resolution[a] = m.grid.resolution[a];
    s.origin[a] = m.grid.origin[a];
    s.polarization[a] = inc.polarization[a];
    s.direction[a] = inc.direction[a];
  }
  s.frequency = m.frequency;
  s.amplitude = inc.amplitude;
  return s;
}

// The scene-stage calls below pass ctx = NULL and stream = NULL, so the library runs them
// on the legacy default stream; the copies use the same stream.
inline CurrentField field_from_device(const DeviceBuffer& b, const std::array<Index, 3>& d) {
  std::vector<cplx> v(static_cast<size_t>(3 * d[0] * d[1] * d[2]));
  b.download(v.data(), v.size() * sizeof(cplx), cudaStreamLegacy);
  return CurrentField::from_vector(v, d);
}

// build_rhs (solver.hpp:148-179)
inline CurrentField build_rhs(const DielectricMap& m, const PlaneWave& inc, int quad_points_per_axis = 1) {
  const vie_scene sc = make_scene(m, inc);
  const size_t nv = m.eps_r.size();
  DeviceBuffer de(nv * sizeof(cplx)), dr(3 * nv * sizeof(cplx));
  de.upload(m.eps_r.data(), nv * sizeof(cplx), cudaStreamLegacy);
  check(vie_build_rhs(nullptr, &sc, de.get(), quad_points_per_axis, dr.get(), nullptr));
  return field_from_device(dr, m.grid.dims);
}

struct Fields {  // solver.hpp:202-206
  CurrentField e;
  CurrentField h;
  bool has_h = false;
};

// recover_fields (solver.hpp:211-249); op_k: the K operator or nullptr
inline Fields recover_fields(const CurrentField& j, const DielectricMap& m, const PlaneWave& inc,
                             const EmbeddedSpectrum* op_k) {
  if (j.dims() != m.grid.dims || j.comp.size() != 3) throw std::invalid_argument("recover_fields: dim mismatch");
  const vie_scene sc = make_scene(m, inc);
  const size_t nv = m.eps_r.size();
  const std::vector<cplx> jv = j.to_vector();
  DeviceBuffer de(nv * sizeof(cplx)), dj(3 * nv * sizeof(cplx)), dE(3 * nv * sizeof(cplx));
  DeviceBuffer dh(op_k ? 3 * nv * sizeof(cplx) : 0);
  de.upload(m.eps_r.data(), nv * sizeof(cplx), cudaStreamLegacy);
  dj.upload(jv.data(), jv.size() * sizeof(cplx), cudaStreamLegacy);
  // the K matvec runs on the legacy stream too (stream = cudaStreamLegacy, ctx = NULL)
  check(vie_recover_fields(nullptr, &sc, de.get(), dj.get(), op_k ? op_k->handle() : nullptr, dE.get(),
                           op_k ? dh.get() : nullptr, cudaStreamLegacy));
  Fields f;
  f.e = field_from_device(dE, m.grid.dims);
  if (op_k) {
    f.h = field_from_device(dh, m.grid.dims);
    f.has_h = true;
  }
  return f;
}

struct PostProcess {  // solver.hpp:251-256 (real per-voxel values)
  std::vector<double> p_abs;
  double total_absorbed_power = 0.0;
  std::vector<double> b1_plus;
  bool has_b1 = false;
};

// postprocess (solver.hpp:258-284)
inline PostProcess postprocess(const Fields& f, const DielectricMap& m) {
  const vie_scene sc = make_scene(m, PlaneWave{});
  const size_t nv = m.eps_r.size();
  const std::vector<cplx> ev = f.e.to_vector();
  DeviceBuffer de(nv * sizeof(cplx)), dE(3 * nv * sizeof(cplx)), dp(nv * sizeof(double));
  DeviceBuffer dh(f.has_h ? 3 * nv * sizeof(cplx) : 0), db(f.has_h ? nv * sizeof(double) : 0);
  de.upload(m.eps_r.data(), nv * sizeof(cplx), cudaStreamLegacy);
  dE.upload(ev.data(), ev.size() * sizeof(cplx), cudaStreamLegacy);
  if (f.has_h) {
    const std::vector<cplx> hv = f.h.to_vector();
    dh.upload(hv.data(), hv.size() * sizeof(cplx), cudaStreamLegacy);
  }
  PostProcess out;
  check(vie_postprocess(nullptr, &sc, de.get(), dE.get(), f.has_h ? dh.get() : nullptr, dp.get(),
                        f.has_h ? db.get() : nullptr, &out.total_absorbed_power, nullptr));
  out.p_abs.resize(nv);
  dp.download(out.p_abs.data(), nv * sizeof(double), cudaStreamLegacy);
  if (f.has_h) {
    out.b1_plus.resize(nv);
    db.download(out.b1_plus.data(), nv * sizeof(double), cudaStreamLegacy);
    out.has_b1 = true;
  }
  return out;
}

struct SolveReport {  // solver.hpp:286-295
  CurrentField j;
  std::vector<double> residual_history;
  double final_relative_residual = 0.0;
  int iterations = 0;
  bool converged = false;
  double wall_time_s = 0.0;
  Fields fields;
  PostProcess post;
};

// solve_scene (solver.hpp:300-326): build_rhs, restarted GMRES on the JVIE system
// (M_eps - M_chi N / V) device resident, recover_fields (K operator optional),
// postprocess.  PWC operators on the map's grid.
inline SolveReport solve_scene(const DielectricMap& m, const PlaneWave& inc, const EmbeddedSpectrum& op_n,
                               const EmbeddedSpectrum* op_k, const GmresConfig& cfg = {}) {
  const auto t0 = std::chrono::steady_clock::now();
  if (op_n.grid_dims != m.grid.dims || op_n.order != BasisOrder::PWC)
    throw std::invalid_argument("solve_scene: op_n must be the PWC operator of the map's grid");
  const CurrentField rhs = build_rhs(m, inc);
  GmresResult g = gmres_system(m.eps_r, 1.0 / m.grid.voxel_volume(), op_n, rhs.to_vector(), cfg);
  SolveReport rep;
  rep.j = CurrentField::from_vector(g.solution, m.grid.dims);
  rep.residual_history = std::move(g.residual_history);
  rep.final_relative_residual = g.final_relative_residual;
  rep.iterations = g.iterations;
  rep.converged = g.converged;
  rep.fields = recover_fields(rep.j, m, inc, op_k);
  rep.post = postprocess(rep.fields, m);
  rep.wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return rep;
}

}  // namespace b200
}  // namespace vie

#endif  // VIE_B200_HPP
