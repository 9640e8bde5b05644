// api.cu -- C ABI (include/vie_b200.h): context + FFT plan cache, device
// Tucker forms, the operator and its matvec pipeline, device-resident GMRES.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <map>
#include <tuple>
#include <memory>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/vie_b200.h"
#include "kernels.cuh"

using vie::CompDev;
using vie::FftPlan;
using vie::Geom;
using cd = std::complex<double>;

namespace {

thread_local std::string g_err;

struct Invalid : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct NcclError : std::runtime_error {  // -> VIE_ENCCL
  using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {  // -> VIE_EIO (the reference's std::runtime_error of container.hpp)
  using std::runtime_error::runtime_error;
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return VIE_OK;
  } catch (const Invalid& e) {
    g_err = e.what();
    return VIE_EINVAL;
  } catch (const vie::CudaError& e) {
    g_err = e.what();
    return e.code == cudaErrorMemoryAllocation ? VIE_ENOMEM : VIE_ECUDA;
  } catch (const NcclError& e) {
    g_err = e.what();
    return VIE_ENCCL;
  } catch (const IoError& e) {
    g_err = e.what();
    return VIE_EIO;
  } catch (const std::bad_alloc& e) {
    g_err = std::string("host allocation failed: ") + e.what();
    return VIE_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return VIE_EINVAL;
  }
}

template <class T>
T* dev_alloc(size_t count) {
  void* p = nullptr;
  if (count == 0) return nullptr;
  VIE_CUDA_CHECK(cudaMalloc(&p, count * sizeof(T)));
  return static_cast<T*>(p);
}
void dev_free(void* p) {
  if (p) cudaFree(p);
}
// Copy ordered on `st` and complete on return.  A plain cudaMemcpy runs on the legacy
// stream, which does not order with the non-blocking streams the kernels use, and a
// pageable host-to-device cudaMemcpy may return before the data has reached the device.
void copy_sync(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  VIE_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st));
  VIE_CUDA_CHECK(cudaStreamSynchronize(st));
}

struct PlanHolder {
  FftPlan plan{};
  double2* tw = nullptr;
  int* slot = nullptr;
  vie::StageDesc* st = nullptr;
  std::vector<int> radices;
  ~PlanHolder() {
    dev_free(tw);
    dev_free(slot);
    dev_free(st);
  }
};

}  // namespace

struct vie_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  double* post_partials = nullptr;  // vie_postprocess partial sums (kRedBlocks + 1), allocated once
  std::mutex post_mu;               // serialises vie_postprocess calls on this context
  // plan cache keyed by (length, pruned, wide)
  std::map<std::tuple<int, bool, bool, bool>, std::unique_ptr<PlanHolder>> plans;
  // references: the caller's (vie_ctx_create) plus one per live Tucker form and operator,
  // which hold device pointers into the plans and run on the stream
  std::atomic<int> refs{1};
};

// NCCL communicator over the ranks of a slab-partitioned operator (one process per GPU)
// Loopback transport (tests): R ranks of one process (one host thread each, any devices),
// exchanging through device-to-device copies between host barriers -- no kernel ever waits on
// another rank's kernel.  Same chunk semantics as the NCCL exchange.
struct vie_loopback_s {
  int nranks = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  std::vector<void*> ptr;             // per rank: the buffer published for the current step
  std::vector<std::vector<double>> h;  // per rank: host scalars of an all-reduce
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t gen = generation;
    if (++arrived == nranks) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

// NCCL communicator over the ranks of a slab-partitioned operator (one process per GPU), or
// the loopback transport above
struct vie_comm_s {
  ncclComm_t nccl = nullptr;
  vie_loopback_s* lb = nullptr;
  int nranks = 1, rank = 0;
  int device = 0;
  ~vie_comm_s() {
    if (nccl) ncclCommDestroy(nccl);
  }
};

namespace {
void ctx_retain(vie_ctx c) { c->refs.fetch_add(1); }
void ctx_release(vie_ctx c) {
  if (c->refs.fetch_sub(1) != 1) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  c->plans.clear();
  if (c->post_partials) cudaFree(c->post_partials);
  cudaStreamDestroy(c->stream);
  delete c;
}
}  // namespace

struct vie_tucker_s {
  vie_ctx ctx = nullptr;
  int64_t dims[3] = {0, 0, 0};
  int64_t ranks[3] = {0, 0, 0};
  int sign[3] = {1, 1, 1};
  double2* core = nullptr;   // r1*r2*r3
  double2* uo[3] = {nullptr, nullptr, nullptr};  // (n_q + 1) x r_q octant rows
  // the spatial form as given (domain 0), for the VIET container (container.hpp): factors
  // n_q x r_q column-major and the core; rule / tol of the compression (-1: none); CP rank (> 0:
  // a Tucker+CP form held with a superdiagonal core, saved as kind tucker_cp)
  std::vector<double2> hu[3], hcore;
  int rule = -1;
  double tol = 0.0;
  int64_t cp_rank = 0;
  ~vie_tucker_s() {
    dev_free(core);
    for (auto* u : uo) dev_free(u);
    if (ctx) ctx_release(ctx);
  }
};

struct vie_op_s {
  vie_ctx ctx = nullptr;
  int kind = 0, basis = 0;
  Geom g{};
  int rmax = 0;
  uint64_t active = 0;
  std::vector<CompDev> comps_host;
  CompDev* comps_dev = nullptr;
  double2* forms = nullptr;
  double2* Z = nullptr;
  double2* u3img = nullptr;  // U3 shared-memory images of the tile decomposition (decomp_tile.cuh)
  double2* Shat = nullptr;
  double2* A = nullptr;
  double2* B = nullptr;
  double2* Bo = nullptr;   // pencil output slab (even axis-3 frequencies)
  double2* Bo1 = nullptr;  // pencil output slab (odd axis-3 frequencies)
  int64_t ws_bytes = 0;
  FftPlan P1{}, P2{}, P3{}, PH{};
  vie::Pass2 Q1{}, Q2{};           // register-staged two-stage row / column passes
  bool q1 = false, q2 = false;  // (false: generic multi-stage passes P1 / P2)
  bool pencil2 = false;         // compile-time-shaped two-branch pencil kernel for this n3
  bool pencil3 = false;         // PWL: whole-mirror-group pencil kernel with the DMMA Hadamard (interior groups)
  bool pencil4 = false;         // PWL: half-mirror-group DMMA pencil kernel, 2 CTAs per SM (replaces pencil3)
  // fused decompression x pencil (kernels_fused.cu): no whole-spectrum buffer; the interior rows
  // go through an L2-resident tile ring, the edge rows through the compact edge buffer Sedge
  bool fused = false;     // current strategy is hosvd_loop (fused kernel)
  bool fused_ok = false;  // the fused kernel supports this operator
  vie::FusedPlan fp{};
  int64_t ws_fixed = 0;   // workspace bytes without the spectrum storage
  double2* ring = nullptr;
  double2* Sedge = nullptr;
  int4* fitems = nullptr;
  unsigned* fcounters = nullptr;
  int fork_after = 0;           // decompression fork point: 0 before the row pass, 1 after it, 2 after the column pass
  // slab decomposition (vie_op_set_partition): this rank's z-planes [k0, k0 + nk) and
  // axis-1 positions [p1off, p1off + W) (Geom)
  int nranks = 1, rank = 0;
  vie_comm comm = nullptr;  // vie_op_set_comm: the in-library exchange and the distributed GMRES
  double2* xs_send = nullptr;  // vie_slab_matvec exchange buffers (slab_elems each)
  double2* xs_recv = nullptr;
  double2* xs_out = nullptr;
  double2* xs_back = nullptr;
  cudaEvent_t ev_slab = nullptr;
  cudaStream_t s_comm = nullptr;     // vie_slab_matvec: the exchange stream
  std::vector<cudaEvent_t> ev_grp;   // vie_slab_matvec: per current group, 4 events
  // host-buffer staging (vie_matvec_host; the batch call double-buffers with hx2 / hy2)
  double2* hx = nullptr;
  double2* hy = nullptr;
  double2* hx2 = nullptr;
  double2* hy2 = nullptr;
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_h2d[2] = {}, ev_done[2] = {}, ev_d2h[2] = {};
  // GMRES state (GmresWork, cached for vie_gmres_solve)
  int g_inner = 0;
  double2* V = nullptr;
  double2* tmp = nullptr;
  double2* zp = nullptr;    // preconditioned vector M v
  double2* scal = nullptr;  // device scalars
  double2* red_partials = nullptr;
  unsigned int* red_counter = nullptr;
  cudaEvent_t ev_user = nullptr;  // orders the solve after the caller's stream
  // side stream: the x-independent decompression runs concurrently with the
  // forward FFT passes (and with the H2D copy of vie_matvec_host)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // stats
  int profiling = 0;
  int last_launches = 0;
  double stage_ms[8] = {0};
  cudaEvent_t ev[8] = {};
  ~vie_op_s() {
    for (void* p : {static_cast<void*>(comps_dev), static_cast<void*>(forms), static_cast<void*>(Z), static_cast<void*>(u3img),
                    static_cast<void*>(Shat), static_cast<void*>(A), static_cast<void*>(B), static_cast<void*>(Bo), static_cast<void*>(Bo1),
                    static_cast<void*>(hx), static_cast<void*>(hy), static_cast<void*>(hx2), static_cast<void*>(hy2),
                    static_cast<void*>(V), static_cast<void*>(ring), static_cast<void*>(Sedge), static_cast<void*>(fitems),
                    static_cast<void*>(fcounters), static_cast<void*>(xs_send), static_cast<void*>(xs_recv),
                    static_cast<void*>(xs_out), static_cast<void*>(xs_back),
                    static_cast<void*>(tmp), static_cast<void*>(zp), static_cast<void*>(scal), static_cast<void*>(red_partials),
                    static_cast<void*>(red_counter)})
      dev_free(p);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    for (int i = 0; i < 2; ++i)
      for (cudaEvent_t e : {ev_h2d[i], ev_done[i], ev_d2h[i]})
        if (e) cudaEventDestroy(e);
    if (side) cudaStreamDestroy(side);
    if (s_h2d) cudaStreamDestroy(s_h2d);
    if (s_d2h) cudaStreamDestroy(s_d2h);
    if (ev_user) cudaEventDestroy(ev_user);
    if (ev_slab) cudaEventDestroy(ev_slab);
    for (cudaEvent_t e : ev_grp) cudaEventDestroy(e);
    if (s_comm) cudaStreamDestroy(s_comm);
    if (ctx) ctx_release(ctx);
  }
};

namespace {

// ---------------------------------------------------------------- FFT plans
// Radix set of the register DFTs (fft.cuh VIE_FFT_RADICES).  Radices are capped
// at kMaxRadix: larger register DFTs raise register pressure and cut the warps
// per SM below what the shared-memory passes need to hide latency (ncu r1).
const int kRadices[] = {24, 20, 16, 15, 12, 10, 8, 7, 6, 5, 4, 3, 2};  // must match VIE_FFT_RADICES(_WIDE)
// lengths with a prime factor 11..31: the EXT two-stage passes (fft.cuh VIE_FFT_RADICES_EXT)
const int kExtRadices[] = {34, 31, 29, 26, 24, 23, 22, 20, 19, 17, 16, 15, 14, 13, 12, 11, 10, 8, 7, 6, 5, 4, 3, 2};
constexpr int kMaxRadix = 10;

bool has_ext_prime(int n) {  // a prime factor > 7 (the EXT radix set covers 11..31)
  for (int p : {2, 3, 5, 7})
    while (n % p == 0) n /= p;
  return n > 1;
}
#ifndef VIE_WIDE_PASSES
#define VIE_WIDE_PASSES 1
#endif
constexpr bool kWidePasses = VIE_WIDE_PASSES;  // two-stage plans for the row/column passes
#ifndef VIE_PASS2
#define VIE_PASS2 1
#endif
constexpr bool kPass2 = VIE_PASS2;
#ifndef VIE_PENCIL2
#define VIE_PENCIL2 1
#endif
constexpr bool kPencil2 = VIE_PENCIL2;

int env_int(const char* name, int dflt) {  // tuning overrides (benchmarks only)
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

// Fewest stages, then smallest largest radix; first radix even when the
// transform is pad/crop pruned (half_in / half_out).
bool factor_plan(int n, bool even_first, int depth, std::vector<int>& cur, std::vector<int>& best,
                 int maxr = kMaxRadix, bool ext = false) {
  if (n == 1) {
    if (best.empty() || cur.size() < best.size() ||
        (cur.size() == best.size() && *std::max_element(cur.begin(), cur.end()) <
                                          *std::max_element(best.begin(), best.end())))
      best = cur;
    return true;
  }
  if (depth == 0) return false;
  bool any = false;
  auto step = [&](int r) {
    if (r > maxr || n % r) return;
    if (even_first && cur.empty() && (r & 1)) return;
    cur.push_back(r);
    any |= factor_plan(n / r, even_first, depth - 1, cur, best, maxr, ext);
    cur.pop_back();
  };
  if (ext)
    for (int r : kExtRadices) step(r);
  else
    for (int r : kRadices) step(r);
  return any;
}

// wide = plan for the pencil kernel (radices up to 20, VIE_FFT_RADICES_WIDE)
// ext = lengths with a prime factor 11..31, for the EXT two-stage passes only (<= 2 stages)
const FftPlan& get_plan(vie_ctx ctx, int n, bool pruned = true, bool wide = false,
                        std::vector<int>* radices = nullptr, bool ext = false) {
  const auto key = std::make_tuple(n, pruned, wide, ext);
  std::lock_guard<std::mutex> lk(ctx->mu);
  auto it = ctx->plans.find(key);
  if (it != ctx->plans.end()) {
    if (radices) *radices = it->second->radices;
    return it->second->plan;
  }
  if (n < 1 || (pruned && (n & 1))) throw Invalid("FFT plan: embedded length must be even");
  std::vector<int> rad, cur;
  for (int depth = 1; depth <= (ext ? 2 : vie::kMaxStages) && rad.empty(); ++depth)
    factor_plan(n, pruned, depth, cur, rad, ext ? 34 : (wide ? 24 : kMaxRadix), ext);
  if (n > 1 && rad.empty())
    throw Invalid("FFT plan: length " + std::to_string(n) +
                  (ext ? " is not R0 x R1 with an even R0 <= 34 and R1 <= 34 of 2,3,5,7,11,..,31-smooth radices"
                       : " has a prime factor > 7"));
  auto h = std::make_unique<PlanHolder>();
  h->radices = rad;
  if (radices) *radices = rad;
  FftPlan& P = h->plan;
  P.n = n;
  P.nst = static_cast<int>(rad.size());
  std::vector<vie::StageDesc> sd(rad.size());
  int L = n;
  for (int s = 0; s < P.nst; ++s) {
    sd[s].radix = rad[s];
    sd[s].L = L;
    sd[s].M = L / rad[s];
    sd[s].tws = n / L;
    sd[s].div_nbf.init(static_cast<uint32_t>(n / rad[s]));
    sd[s].div_M.init(static_cast<uint32_t>(sd[s].M));
    L = sd[s].M;
  }
  std::vector<double2> tw(static_cast<size_t>(n));
  for (int e = 0; e < n; ++e) {
    const long double a = -2.0L * 3.14159265358979323846264338327950288L * e / n;
    tw[static_cast<size_t>(e)] = make_double2(static_cast<double>(cosl(a)), static_cast<double>(sinl(a)));
  }
  std::vector<int> slot(static_cast<size_t>(n));
  for (int f = 0; f < n; ++f) {
    int rem = f, sl = 0;
    for (int s = 0; s < P.nst; ++s) {
      sl += (rem % sd[s].radix) * sd[s].M;
      rem /= sd[s].radix;
    }
    slot[static_cast<size_t>(f)] = sl;
  }
  h->tw = dev_alloc<double2>(static_cast<size_t>(n));
  h->slot = dev_alloc<int>(static_cast<size_t>(n));
  h->st = dev_alloc<vie::StageDesc>(sd.size());
  copy_sync(h->tw, tw.data(), sizeof(double2) * n, ctx->stream);
  copy_sync(h->slot, slot.data(), sizeof(int) * n, ctx->stream);
  copy_sync(h->st, sd.data(), sizeof(vie::StageDesc) * sd.size(), ctx->stream);
  P.tw = h->tw;
  P.slot = h->slot;
  P.st = h->st;
  const FftPlan& ref = h->plan;
  ctx->plans[key] = std::move(h);
  return ref;
}

// ---------------------------------------------------------------- tables (host)
struct HComp {
  int q, qp, l, lp;
  int par[3];
};
struct HBlock {
  int t, s, c, dsign;
};

template <int KIND, int BASIS>
void copy_table(std::vector<HComp>& cs, std::vector<HBlock>& bs) {
  constexpr auto tb = vie::make_table<KIND, BASIS>();
  for (const auto& c : tb.comps) cs.push_back({c.q, c.qp, c.l, c.lp, {c.p0, c.p1, c.p2}});
  for (const auto& b : tb.blocks) {
    const auto& c = tb.comps[static_cast<size_t>(b.c)];
    bs.push_back({b.t, b.s, b.c, b.coef * c.p0 * c.p1 * c.p2});  // back to the dense sign
  }
}

void host_table(int kind, int basis, std::vector<HComp>& cs, std::vector<HBlock>& bs) {
  cs.clear();
  bs.clear();
  if (kind == 0 && basis == 0) copy_table<0, 0>(cs, bs);
  else if (kind == 1 && basis == 0) copy_table<1, 0>(cs, bs);
  else if (kind == 0 && basis == 1) copy_table<0, 1>(cs, bs);
  else if (kind == 1 && basis == 1) copy_table<1, 1>(cs, bs);
  else throw Invalid("component table: kind must be N/K and basis PWC/PWL");
}

// RAII pool of scratch device buffers
struct DevPool {
  std::vector<void*> p;
  ~DevPool() {
    for (void* x : p) dev_free(x);
  }
  template <class T>
  T* alloc(size_t n) {
    T* x = dev_alloc<T>(n);
    p.push_back(x);
    return x;
  }
};

// ---------------------------------------------------------------- hosvd (host parts)
// truncation_rank (decomp.hpp:72-103)
int64_t truncation_rank_host(const std::vector<double>& s, double tol, int rule) {
  const int64_t n = static_cast<int64_t>(s.size());
  if (n == 0) return 0;
  const double smax = s[0];
  if (smax <= 0.0) return 0;
  if (rule == VIE_RULE_SIGMA_MAX) {
    const double threshold = (tol / std::sqrt(3.0)) * smax;
    int64_t r = 0;
    for (int64_t j = 0; j < n; ++j)
      if (s[static_cast<size_t>(j)] > 0.0 && s[static_cast<size_t>(j)] >= threshold - 1e-14 * smax) r = j + 1;
    return r;
  }
  double total = 0.0;
  for (double x : s) total += x * x;
  const double budget = (tol / std::sqrt(3.0)) * std::sqrt(total);
  const double budget2 = budget * budget;
  double tail = 0.0;
  int64_t r = n;
  while (r > 0) {
    const double cand = tail + s[static_cast<size_t>(r - 1)] * s[static_cast<size_t>(r - 1)];
    if (cand <= budget2 || s[static_cast<size_t>(r - 1)] == 0.0) {
      tail = cand;
      --r;
    } else {
      break;
    }
  }
  return r;
}

// Cyclic Jacobi eigendecomposition of a Hermitian n x n matrix (col-major):
// eigenvalues descending in lam, eigenvectors in the columns of V.  Rotation
// J = [[c, s e^{i phi}], [-s e^{-i phi}, c]] zeroes a_pq = |a_pq| e^{i phi}.
void herm_eig_jacobi(std::vector<cd>& a, int n, std::vector<double>& lam, std::vector<cd>& V, bool relative = true) {
  auto A = [&](int i, int j) -> cd& { return a[static_cast<size_t>(i) + static_cast<size_t>(n) * j]; };
  std::vector<cd> v(static_cast<size_t>(n) * n, cd(0.0));
  for (int i = 0; i < n; ++i) v[static_cast<size_t>(i) * (n + 1)] = 1.0;
  double fro = 0.0;
  for (const cd& x : a) fro += std::norm(x);
  fro = std::sqrt(fro);
  // relative (Demmel-Veselic) threshold: rotate while |a_pq| > eps sqrt(a_pp a_qq), so the
  // small eigenvalues of a graded Gram (rows of B = U0^H M carry the singular values) keep
  // their relative accuracy instead of being flushed at eps * ||A||
  for (int sweep = 0; sweep < 80 && fro > 0.0; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const cd apq = A(p, q);
        const double mag = std::abs(apq);
        if (mag <= 1e-300 || mag <= (relative ? 1e-16 * std::sqrt(std::abs(A(p, p).real() * A(q, q).real()))
                                              : 1e-16 * fro))
          continue;
        rotated = true;
        const double tau = (A(q, q).real() - A(p, p).real()) / (2.0 * mag);
        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (std::abs(tau) + std::sqrt(1.0 + tau * tau));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = t * c;
        const cd ph = apq / mag;
        const cd jpq = s * ph, jqp = -s * std::conj(ph);
        for (int k = 0; k < n; ++k) {  // A <- A J (columns p, q)
          const cd akp = A(k, p), akq = A(k, q);
          A(k, p) = akp * c + akq * jqp;
          A(k, q) = akp * jpq + akq * c;
        }
        for (int k = 0; k < n; ++k) {  // A <- J^H A (rows p, q)
          const cd apk = A(p, k), aqk = A(q, k);
          A(p, k) = c * apk + std::conj(jqp) * aqk;
          A(q, k) = std::conj(jpq) * apk + c * aqk;
        }
        A(p, q) = 0.0;
        A(q, p) = 0.0;
        for (int k = 0; k < n; ++k) {  // V <- V J
          cd& vkp = v[static_cast<size_t>(k) + static_cast<size_t>(n) * p];
          cd& vkq = v[static_cast<size_t>(k) + static_cast<size_t>(n) * q];
          const cd x = vkp, y = vkq;
          vkp = x * c + y * jqp;
          vkq = x * jpq + y * c;
        }
      }
    if (!rotated) break;
  }
  std::vector<int> order(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) order[static_cast<size_t>(i)] = i;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return A(x, x).real() > A(y, y).real(); });
  lam.resize(static_cast<size_t>(n));
  V.assign(static_cast<size_t>(n) * n, cd(0.0));
  for (int k = 0; k < n; ++k) {
    const int o = order[static_cast<size_t>(k)];
    lam[static_cast<size_t>(k)] = A(o, o).real();
    for (int i = 0; i < n; ++i)
      V[static_cast<size_t>(i) + static_cast<size_t>(n) * k] = v[static_cast<size_t>(i) + static_cast<size_t>(n) * o];
  }
}

// ---------------------------------------------------------------- matvec
// Launch the decompression on the side stream after all work queued on `st`.
// Spectrum storage of the current strategy, allocated on first use (and reported by
// vie_op_info): hosvd_decompress -> Shat, all octant spectra; hosvd_loop -> the fused
// kernel's tile ring, work queue and the compact edge rows.
void ensure_spectra(vie_op op) {
  const Geom& g = op->g;
  const int64_t rs = static_cast<int64_t>(g.NC) * (g.n3 + 1);
  if (op->fused && !op->ring) {
    std::vector<int4> items;
    vie::fused_plan_items(op->fp, g, items);
    op->ring = dev_alloc<double2>(static_cast<size_t>(op->fp.RING) * op->fp.BM * rs);
    op->Sedge = dev_alloc<double2>(static_cast<size_t>(vie::shat_rows(g.n1, g.n2, 1) * rs));
    op->fitems = dev_alloc<int4>(items.size());
    copy_sync(op->fitems, items.data(), sizeof(int4) * items.size(), op->ctx->stream);
    op->fcounters = dev_alloc<unsigned>(1 + 3 * static_cast<size_t>(op->fp.ntiles));
    op->fp.forms = op->forms;
    op->fp.u3img = op->u3img;
    op->fp.comps = op->comps_dev;
    op->fp.Z = op->Z;
    op->fp.ring = op->ring;
    op->fp.items = op->fitems;
    op->fp.counters = op->fcounters;
    op->fp.rmax = op->rmax;
  }
  if (!op->fused && !op->Shat) op->Shat = dev_alloc<double2>(static_cast<size_t>(vie::shat_rows(g.n1, g.n2, 0) * rs));
  int64_t spec = 0;
  if (op->Shat) spec += vie::shat_rows(g.n1, g.n2, 0) * rs;
  if (op->ring)
    spec += static_cast<int64_t>(op->fp.RING) * op->fp.BM * rs + vie::shat_rows(g.n1, g.n2, 1) * rs;
  op->ws_bytes = op->ws_fixed + static_cast<int64_t>(sizeof(double2)) * spec;
}

// Geometry of the edge pencil launches of the fused path (compact edge spectrum rows)
Geom edge_geom(const vie_op_s* op) {
  Geom ge = op->g;
  ge.ecompact = op->fused ? 1 : 0;
  return ge;
}

// The x-independent decompression stage: the whole octant spectrum (materialised path) or, on
// the fused path, Z = core x2 U2 and the edge rows only (the interior rows are decompressed
// inside the fused kernel).
void decomp_stage(vie_op op, cudaStream_t st) {
  ensure_spectra(op);  // (vie_matvec_host forks this stage before run_matvec)
  if (op->fused) {
    vie::launch_decomp_z(op->forms, op->comps_dev, op->Z, op->g, op->rmax, st);
    vie::launch_decomp_edges(op->fp, op->Sedge, edge_geom(op), st);
  } else {
    vie::launch_decomp(op->forms, op->comps_dev, op->comps_host.data(), op->Z, op->Shat, op->g, op->rmax, st, 0, -1,
                       true, 0, -1, op->u3img);
  }
}

void fork_decomp(vie_op op, cudaStream_t st) {
  VIE_CUDA_CHECK(cudaEventRecord(op->ev_fork, st));
  VIE_CUDA_CHECK(cudaStreamWaitEvent(op->side, op->ev_fork, 0));
  decomp_stage(op, op->side);
  VIE_CUDA_CHECK(cudaEventRecord(op->ev_join, op->side));
}

void run_matvec(vie_op op, const double2* x, double2* y, cudaStream_t st, const double2* eps, double inv_v,
                int diag, bool decomp_forked = false) {
  if (op->nranks > 1) throw Invalid("apply_operator: operator is partitioned (use the vie_slab_* stages)");
  ensure_spectra(op);
  const Geom& g = op->g;
  const double ne = 8.0 * g.n1 * static_cast<double>(g.n2) * g.n3;
  if (op->profiling) {  // serial launches so every stage gets its own event interval
    for (auto& e : op->ev)
      if (!e) VIE_CUDA_CHECK(cudaEventCreate(&e));
    VIE_CUDA_CHECK(cudaEventRecord(op->ev[0], st));
  }
  int k = 1;
  // profiling 1: serial stages, one event interval each; 2: the normal overlapped
  // schedule with events after the column pass, after the decompression join and at the end
  auto mark = [&] {
    if (op->profiling == 1) VIE_CUDA_CHECK(cudaEventRecord(op->ev[k++], st));
  };
  auto mark2 = [&] {
    if (op->profiling == 2) VIE_CUDA_CHECK(cudaEventRecord(op->ev[k++], st));
  };
  const bool overlap = op->profiling != 1;
  if (overlap && !decomp_forked && op->fork_after == 0) fork_decomp(op, st);
  if (op->q1) vie::launch_row_fwd2(x, op->A, g, op->Q1, st);
  else vie::launch_row_fwd(x, op->A, g, op->P1, st);
  if (overlap && !decomp_forked && op->fork_after == 1) fork_decomp(op, st);
  mark();
  if (op->q2) vie::launch_col_fwd2(op->A, op->B, g, op->Q2, st);
  else vie::launch_col_fwd(op->A, op->B, g, op->P2, st);
  if (overlap && !decomp_forked && op->fork_after >= 2) fork_decomp(op, st);
  mark();
  mark2();
  if (overlap) {
    VIE_CUDA_CHECK(cudaStreamWaitEvent(st, op->ev_join, 0));
    mark2();
  } else {
    if (decomp_forked) VIE_CUDA_CHECK(cudaStreamWaitEvent(st, op->ev_join, 0));
    else decomp_stage(op, st);
  }
  mark();
  if (op->fused) {  // edge rows from the compact edge buffer, the interior in the fused kernel
    const Geom ge = edge_geom(op);
    vie::launch_pencil(op->kind, op->basis, op->B, op->Bo, op->Bo1, op->Sedge, ge, op->PH, op->P3.tw, op->active, st,
                       1);
    vie::launch_pencil2(op->kind, op->basis, op->B, op->Bo, op->Sedge, ge, op->P3.tw, st, 0, 2);
    vie::launch_fused(op->kind, op->fp, op->B, op->Bo, g, op->P3.tw, st);
  } else if (op->pencil3) {  // interior mirror groups on the DMMA kernel; axis-1 edge group, axis-2 edge rows
    vie::launch_pencil(op->kind, op->basis, op->B, op->Bo, op->Bo1, op->Shat, g, op->PH, op->P3.tw, op->active, st,
                       1);
    vie::launch_pencil2(op->kind, op->basis, op->B, op->Bo, op->Shat, g, op->P3.tw, st, 0, 2);
    if (op->pencil4) vie::launch_pencil4(op->kind, op->B, op->Bo, op->Shat, g, op->P3.tw, st);
    else vie::launch_pencil3(op->kind, op->B, op->Bo, op->Shat, g, op->P3.tw, st);
  } else if (op->pencil2) {  // compile-time-shaped kernel + the axis-1 edge group on the generic one
    vie::launch_pencil(op->kind, op->basis, op->B, op->Bo, op->Bo1, op->Shat, g, op->PH, op->P3.tw, op->active, st,
                       1);
    vie::launch_pencil2(op->kind, op->basis, op->B, op->Bo, op->Shat, g, op->P3.tw, st);
  } else {
    vie::launch_pencil(op->kind, op->basis, op->B, op->Bo, op->Bo1, op->Shat, g, op->PH, op->P3.tw, op->active, st);
  }
  mark();
  if (op->q2) vie::launch_col_inv2(op->Bo, op->A, g, op->Q2, st);
  else vie::launch_col_inv(op->Bo, nullptr, op->A, g, op->P2, st);
  mark();
  // reference inverse3 divides by N_e (fft.hpp:34-37)
  if (op->q1) vie::launch_row_inv2(op->A, y, g, op->Q1, 1.0 / ne, eps, x, inv_v, op->basis, diag, st);
  else vie::launch_row_inv(op->A, y, g, op->P1, 1.0 / ne, eps, x, inv_v, op->basis, diag, st);
  mark();
  mark2();
  // row, column, (decomp_z + decomp), pencil (+ edge), column, row
  op->last_launches = 7 + (op->pencil2 ? 1 : 0) + (op->pencil3 ? 1 : 0);
  if (op->profiling) {
    VIE_CUDA_CHECK(cudaEventSynchronize(op->ev[k - 1]));
    for (int i = 1; i < k; ++i) {
      float ms = 0.f;
      VIE_CUDA_CHECK(cudaEventElapsedTime(&ms, op->ev[i - 1], op->ev[i]));
      op->stage_ms[i - 1] = ms;
    }
  }
}

cudaStream_t pick_stream(vie_op op, void* stream) {
  return stream ? static_cast<cudaStream_t>(stream) : op->ctx->stream;
}

void check_cplx_finite_host(const double* p, size_t n, const char* what) {
  for (size_t i = 0; i < 2 * n; ++i)
    if (!std::isfinite(p[i])) throw Invalid(std::string(what) + ": non-finite value");
}

}  // namespace

// ===================================================================== C ABI
extern "C" {

const char* vie_last_error(void) { return g_err.c_str(); }
const char* vie_version(void) { return "vie-b200 0.1.0 (sm_100a)"; }

int vie_ctx_create(vie_ctx* out, int device) {
  return guard([&] {
    if (!out) throw Invalid("vie_ctx_create: null output");
    int ndev = 0;
    VIE_CUDA_CHECK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw Invalid("vie_ctx_create: no such CUDA device");
    VIE_CUDA_CHECK(cudaSetDevice(device));
    auto* c = new vie_ctx_s;
    c->device = device;
    VIE_CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    *out = c;
  });
}

int vie_ctx_destroy(vie_ctx ctx) {
  return guard([&] {
    if (!ctx) return;
    ctx_release(ctx);  // freed once the last form / operator of the context is destroyed
  });
}

int vie_ctx_stream(vie_ctx ctx, void** stream) {
  return guard([&] {
    if (!ctx || !stream) throw Invalid("vie_ctx_stream: null argument");
    *stream = ctx->stream;
  });
}

int vie_op_stream(vie_op op, void** stream) {
  return guard([&] {
    if (!op || !stream) throw Invalid("vie_op_stream: null argument");
    *stream = op->ctx->stream;
  });
}

int vie_ctx_sync(vie_ctx ctx) {
  return guard([&] {
    if (!ctx) throw Invalid("vie_ctx_sync: null context");
    VIE_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  });
}

int vie_component_table(int kind, int basis, int* ncomp, int* comps, int* parity, int* nblock, int* blocks) {
  return guard([&] {
    std::vector<HComp> cs;
    std::vector<HBlock> bs;
    host_table(kind, basis, cs, bs);
    if (ncomp) *ncomp = static_cast<int>(cs.size());
    if (nblock) *nblock = static_cast<int>(bs.size());
    for (size_t i = 0; i < cs.size(); ++i) {
      if (comps) {
        comps[4 * i] = cs[i].q;
        comps[4 * i + 1] = cs[i].qp;
        comps[4 * i + 2] = cs[i].l;
        comps[4 * i + 3] = cs[i].lp;
      }
      if (parity)
        for (int a = 0; a < 3; ++a) parity[3 * i + static_cast<size_t>(a)] = cs[i].par[a];
    }
    if (blocks)
      for (size_t i = 0; i < bs.size(); ++i) {
        blocks[4 * i] = bs[i].t;
        blocks[4 * i + 1] = bs[i].s;
        blocks[4 * i + 2] = bs[i].c;
        blocks[4 * i + 3] = bs[i].dsign;
      }
  });
}

int vie_tucker_from_factors(vie_ctx ctx, const int64_t dims[3], const int64_t ranks[3], const double* core_host,
                            const double* u1_host, const double* u2_host, const double* u3_host, const int sign[3],
                            int domain, vie_tucker* out) {
  return guard([&] {
    if (!ctx || !dims || !ranks || !core_host || !u1_host || !u2_host || !u3_host || !sign || !out)
      throw Invalid("vie_tucker_from_factors: null argument");
    if (domain != 0 && domain != 1) throw Invalid("vie_tucker_from_factors: domain must be 0 or 1");
    VIE_CUDA_CHECK(cudaSetDevice(ctx->device));
    for (int q = 0; q < 3; ++q) {
      if (dims[q] < 1) throw Invalid("vie_tucker_from_factors: dims must be >= 1");
      if (ranks[q] < 1) throw Invalid("vie_tucker_from_factors: ranks must be >= 1");
      if (sign[q] != 1 && sign[q] != -1) throw Invalid("vie_tucker_from_factors: sign must be +-1");
    }
    std::unique_ptr<vie_tucker_s> t(new vie_tucker_s);
    ctx_retain(ctx);
    t->ctx = ctx;
    for (int q = 0; q < 3; ++q) {
      t->dims[q] = dims[q];
      t->ranks[q] = ranks[q];
      t->sign[q] = sign[q];
    }
    const size_t ncore = static_cast<size_t>(ranks[0] * ranks[1] * ranks[2]);
    check_cplx_finite_host(core_host, ncore, "vie_tucker_from_factors: core");
    if (domain == 0) {
      t->hcore.assign(reinterpret_cast<const double2*>(core_host), reinterpret_cast<const double2*>(core_host) + ncore);
      const double* uq[3] = {u1_host, u2_host, u3_host};
      for (int q = 0; q < 3; ++q)
        t->hu[q].assign(reinterpret_cast<const double2*>(uq[q]),
                        reinterpret_cast<const double2*>(uq[q]) + dims[q] * ranks[q]);
    }
    t->core = dev_alloc<double2>(ncore);
    copy_sync(t->core, core_host, ncore * sizeof(double2), ctx->stream);
    const double* uh[3] = {u1_host, u2_host, u3_host};
    for (int q = 0; q < 3; ++q) {
      const int64_t n = dims[q], r = ranks[q];
      t->uo[q] = dev_alloc<double2>(static_cast<size_t>((n + 1) * r));
      const cd* u = reinterpret_cast<const cd*>(uh[q]);
      if (domain == 0) {
        check_cplx_finite_host(uh[q], static_cast<size_t>(n * r), "vie_tucker_from_factors: factor");
        if (sign[q] < 0) {  // odd axis: the tensor (hence the factor) vanishes at offset 0
          double nrm = 0.0, row0 = 0.0;
          for (int64_t c = 0; c < r; ++c) {
            for (int64_t i = 0; i < n; ++i) nrm += std::norm(u[i + n * c]);
            row0 += std::norm(u[n * c]);
          }
          if (row0 > 1e-24 * nrm)
            throw Invalid("vie_tucker_from_factors: odd-parity factor has a nonzero row 0");
        }
        // direct DFT of the embedded columns (any length: only the w_2n twiddles are needed)
        DevPool tmp;
        double2* du = tmp.alloc<double2>(static_cast<size_t>(n * r));
        double2* tw = tmp.alloc<double2>(static_cast<size_t>(2 * n));
        std::vector<double2> twh(static_cast<size_t>(2 * n));
        for (int64_t e = 0; e < 2 * n; ++e) {
          const long double a = -3.14159265358979323846264338327950288L * e / n;
          twh[static_cast<size_t>(e)] = make_double2(static_cast<double>(cosl(a)), static_cast<double>(sinl(a)));
        }
        copy_sync(du, uh[q], sizeof(double2) * n * r, ctx->stream);
        copy_sync(tw, twh.data(), sizeof(double2) * twh.size(), ctx->stream);
        vie::launch_factor_transform(du, static_cast<int>(n), static_cast<int>(r), sign[q], tw, t->uo[q],
                                     ctx->stream);
        VIE_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
      } else {
        const int64_t m = 2 * n;
        check_cplx_finite_host(uh[q], static_cast<size_t>(m * r), "vie_tucker_from_factors: factor");
        double amax = 0.0, dev = 0.0;
        for (int64_t c = 0; c < r; ++c)
          for (int64_t p = 0; p < m; ++p) {
            amax = std::max(amax, std::abs(u[p + m * c]));
            const cd mir = u[(m - p) % m + m * c];
            dev = std::max(dev, std::abs(u[p + m * c] - static_cast<double>(sign[q]) * mir));
            if (p == 0 && sign[q] < 0) dev = std::max(dev, std::abs(u[p + m * c]));
          }
        if (dev > 1e-10 * std::max(amax, 1e-300))
          throw Invalid("vie_tucker_from_factors: Fourier factor lacks the parity symmetry U(m-p) = sign U(p)");
        std::vector<cd> oct(static_cast<size_t>((n + 1) * r));
        for (int64_t c = 0; c < r; ++c)
          for (int64_t p = 0; p <= n; ++p) oct[static_cast<size_t>(p + (n + 1) * c)] = u[p + m * c];
        copy_sync(t->uo[q], oct.data(), sizeof(double2) * oct.size(), ctx->stream);
      }
    }
    *out = t.release();
  });
}

int vie_tucker_from_cp(vie_ctx ctx, const int64_t dims[3], int64_t rank, const double* w1_host,
                       const double* w2_host, const double* w3_host, const int sign[3], int domain,
                       vie_tucker* out) {
  int rc = guard([&] {
    if (rank < 1) throw Invalid("TuckerCPForm: rank must be >= 1");
    if (rank > 64) throw Invalid("TuckerCPForm: rank above the device decompressor's limit (64)");
  });
  if (rc != VIE_OK) return rc;
  std::vector<cd> core(static_cast<size_t>(rank * rank * rank), cd(0.0));
  for (int64_t l = 0; l < rank; ++l) core[static_cast<size_t>(l + rank * (l + rank * l))] = 1.0;  // superdiagonal
  const int64_t ranks[3] = {rank, rank, rank};
  const int rc2 = vie_tucker_from_factors(ctx, dims, ranks, reinterpret_cast<const double*>(core.data()), w1_host,
                                          w2_host, w3_host, sign, domain, out);
  if (rc2 == VIE_OK) (*out)->cp_rank = rank;
  return rc2;
}

int vie_tucker_ranks(vie_tucker t, int64_t ranks_out[3]) {
  return guard([&] {
    if (!t || !ranks_out) throw Invalid("vie_tucker_ranks: null argument");
    for (int q = 0; q < 3; ++q) ranks_out[q] = t->ranks[q];
  });
}

int vie_tucker_destroy(vie_tucker t) {
  return guard([&] {
    if (t) {
      cudaSetDevice(t->ctx->device);
      delete t;  // releases its context reference
    }
  });
}

int vie_op_create(vie_ctx ctx, int kind, int basis, const int64_t grid[3], int ncomp, const int* comp,
                  const vie_tucker* forms, vie_op* out) {
  return guard([&] {
    if (!ctx || !grid || !out) throw Invalid("vie_op_create: null argument");
    if (ncomp < 1 || !comp || !forms) throw Invalid("build_operator_spectra: no components");
    VIE_CUDA_CHECK(cudaSetDevice(ctx->device));
    std::vector<HComp> cs;
    std::vector<HBlock> bs;
    host_table(kind, basis, cs, bs);
    for (int q = 0; q < 3; ++q)
      if (grid[q] < 1) throw Invalid("vie_op_create: grid dims must be >= 1");
    if (grid[0] * grid[1] * grid[2] > (int64_t(1) << 31) / 8)
      throw Invalid("vie_op_create: grid too large for 32-bit spectral indexing");
    std::unique_ptr<vie_op_s> op(new vie_op_s);
    ctx_retain(ctx);
    op->ctx = ctx;
    op->kind = kind;
    op->basis = basis;
    Geom& g = op->g;
    g.n1 = static_cast<int>(grid[0]);
    g.n2 = static_cast<int>(grid[1]);
    g.n3 = static_cast<int>(grid[2]);
    g.m1 = 2 * g.n1;
    g.m2 = 2 * g.n2;
    g.m3 = 2 * g.n3;
    g.S = basis == 0 ? 3 : 12;
    g.NC = static_cast<int>(cs.size());
    g.nk = g.n3;  // one slab block (vie_op_set_partition re-blocks for the slab-decomposed matvec)
    g.W = g.m1;
    g.p1off = 0;
    g.bps = static_cast<int64_t>(g.m1) * g.m2;
    op->comps_host.assign(cs.size(), CompDev{1, 1, 1, 0, 0, 0, 0, 0, 0});
    std::vector<const vie_tucker_s*> byc(cs.size(), nullptr);
    for (int i = 0; i < ncomp; ++i) {
      const int* e = comp + 4 * i;
      int found = -1;
      for (size_t c = 0; c < cs.size(); ++c)
        if (cs[c].q == e[0] && cs[c].qp == e[1] && cs[c].l == e[2] && cs[c].lp == e[3]) found = static_cast<int>(c);
      if (found < 0) throw Invalid("vie_op_create: component is not in the canonical table of (kind, basis)");
      if (byc[static_cast<size_t>(found)]) throw Invalid("vie_op_create: duplicate component");
      const vie_tucker_s* t = forms[i];
      if (!t) throw Invalid("vie_op_create: null form");
      if (t->ctx != ctx) throw Invalid("vie_op_create: form belongs to another context");
      for (int q = 0; q < 3; ++q) {
        if (t->dims[q] != grid[q]) throw Invalid("build_operator_spectra: inconsistent component dims");
        if (t->sign[q] != cs[static_cast<size_t>(found)].par[q])
          throw Invalid("vie_op_create: form parity differs from the component parity");
      }
      byc[static_cast<size_t>(found)] = t;
    }
    // pack forms: core, U1o, U2o, U3o per active component; Z offsets
    int64_t off = 0, zoff = 0, u3ioff = 0;
    for (size_t c = 0; c < cs.size(); ++c) {
      const vie_tucker_s* t = byc[c];
      CompDev& d = op->comps_host[c];
      if (!t) continue;
      d.r1 = static_cast<int>(t->ranks[0]);
      d.r2 = static_cast<int>(t->ranks[1]);
      d.r3 = static_cast<int>(t->ranks[2]);
      d.active = 1;
      op->active |= (1ull << c);
      op->rmax = std::max({op->rmax, d.r1, d.r2, d.r3});
      d.off_core = off;
      off += static_cast<int64_t>(d.r1) * d.r2 * d.r3;
      d.off_u1 = off;
      off += static_cast<int64_t>(g.n1 + 1) * d.r1;
      d.off_u2 = off;
      off += static_cast<int64_t>(g.n2 + 1) * d.r2;
      d.off_u3 = off;
      off += static_cast<int64_t>(g.n3 + 1) * d.r3;
      d.off_z = zoff;
      zoff += static_cast<int64_t>(g.n2 + 1) * d.r1 * d.r3;
      d.off_u3i = u3ioff;
      u3ioff += vie::u3_image_elems(g.n3, d.r3);
    }
    if (static_cast<size_t>(op->rmax) * 32 * sizeof(double2) > vie::kMaxSmem)
      throw Invalid("vie_op_create: Tucker rank above the device limit (443)");
    if (vie::pencil_smem(g.n3, g.S, g.NC) > vie::kMaxSmem) throw Invalid("vie_op_create: grid edge n3 too large");
    op->forms = dev_alloc<double2>(static_cast<size_t>(off));
    for (size_t c = 0; c < cs.size(); ++c) {
      const vie_tucker_s* t = byc[c];
      if (!t) continue;
      const CompDev& d = op->comps_host[c];
      copy_sync(op->forms + d.off_core, t->core, sizeof(double2) * d.r1 * d.r2 * d.r3, ctx->stream);
      copy_sync(op->forms + d.off_u1, t->uo[0], sizeof(double2) * (g.n1 + 1) * d.r1, ctx->stream);
      copy_sync(op->forms + d.off_u2, t->uo[1], sizeof(double2) * (g.n2 + 1) * d.r2, ctx->stream);
      copy_sync(op->forms + d.off_u3, t->uo[2], sizeof(double2) * (g.n3 + 1) * d.r3, ctx->stream);
    }
    op->u3img = dev_alloc<double2>(static_cast<size_t>(std::max<int64_t>(u3ioff, 1)));
    vie::launch_u3_image(op->forms, op->comps_host.data(), g.NC, g.n3, op->u3img, ctx->stream);
    op->comps_dev = dev_alloc<CompDev>(cs.size());
    copy_sync(op->comps_dev, op->comps_host.data(), sizeof(CompDev) * cs.size(), ctx->stream);
    const int64_t nv = static_cast<int64_t>(g.n1) * g.n2 * g.n3;
    op->Z = dev_alloc<double2>(static_cast<size_t>(std::max<int64_t>(zoff, 1)));
    op->pencil2 = kPencil2 && vie::pencil2_supported(op->kind, op->basis, g.n3, op->active, g.NC);
    op->pencil3 = op->pencil2 && vie::pencil3_supported(op->kind, op->basis, g.n3, op->active, g.NC);
    op->pencil4 = op->pencil3 && vie::pencil4_supported(op->kind, op->basis, g.n3, op->active, g.NC);
    op->fused_ok = op->pencil4 && vie::fused_supported(op->kind, op->basis, g, op->active, op->rmax);
    // spectrum storage follows the strategy (vie_op_set_strategy) and is allocated on first use:
    // hosvd_decompress -> the whole octant spectrum Shat; hosvd_loop -> tile ring + edge rows
    {
      const char* s = std::getenv("VIE_STRATEGY");
      op->fused = op->fused_ok && s && std::string(s) == "loop";
    }
    op->A = dev_alloc<double2>(static_cast<size_t>(g.S * 2 * nv));
    op->B = dev_alloc<double2>(static_cast<size_t>(g.S * g.n3 * g.bps));
    op->Bo = dev_alloc<double2>(static_cast<size_t>(g.S * g.n3 * g.bps));
    op->ws_fixed = static_cast<int64_t>(sizeof(double2)) * (zoff + g.S * 2 * nv + 2 * g.S * g.n3 * g.bps);
    op->ws_bytes = op->ws_fixed;  // + the strategy's spectrum storage, allocated on first use
    if (const int poison = env_int("VIE_DEBUG_POISON", 0)) {  // debug: NaN-fill workspaces (reads of unwritten data)
      const int64_t nb = g.S * g.n3 * g.bps;
      const int64_t noct = static_cast<int64_t>(g.n1 + 1) * (g.n2 + 1) * (g.n3 + 1);
      if ((poison & 1) && op->Shat) VIE_CUDA_CHECK(cudaMemsetAsync(op->Shat, 0xFF, sizeof(double2) * noct * g.NC));
      if ((poison & 1) && op->ring)
        VIE_CUDA_CHECK(cudaMemsetAsync(op->ring, 0xFF,
                                       sizeof(double2) * op->fp.RING * op->fp.BM * g.NC * (g.n3 + 1)));
      if (poison & 2) VIE_CUDA_CHECK(cudaMemsetAsync(op->Z, 0xFF, sizeof(double2) * std::max<int64_t>(zoff, 1)));
      if (poison & 4) VIE_CUDA_CHECK(cudaMemsetAsync(op->A, 0xFF, sizeof(double2) * g.S * 2 * nv));
      if (poison & 8) VIE_CUDA_CHECK(cudaMemsetAsync(op->B, 0xFF, sizeof(double2) * nb));
      if (poison & 16) VIE_CUDA_CHECK(cudaMemsetAsync(op->Bo, 0xFF, sizeof(double2) * nb));
      VIE_CUDA_CHECK(cudaDeviceSynchronize());
    }
    op->P3 = get_plan(ctx, g.m3);
    // axes 1 and 2: register-staged two-stage passes when the axis has a <= 2-stage wide plan
    // (lengths with a prime factor 11..31 -- the Duke head's 186 and 238 -- only this way)
    if (kPass2 || has_ext_prime(g.m1) || has_ext_prime(g.m2)) {
      std::vector<int> r1, r2;
      const FftPlan& W1 = get_plan(ctx, g.m1, true, true, &r1, has_ext_prime(g.m1));
      const FftPlan& W2 = get_plan(ctx, g.m2, true, true, &r2, has_ext_prime(g.m2));
      op->q1 = vie::pass2_init(op->Q1, g.m1, r1.data(), static_cast<int>(r1.size()), W1.tw, env_int("VIE_ROW_LINES", 0));
      op->q2 = vie::pass2_init(op->Q2, g.m2, r2.data(), static_cast<int>(r2.size()), W2.tw, 0);
    }
    // generic multi-stage passes otherwise (7-smooth lengths only)
    if (!op->q1) op->P1 = get_plan(ctx, g.m1, true, kWidePasses);  // rows: two-stage plans measured faster
    if (!op->q2) op->P2 = get_plan(ctx, g.m2, true, false);        // columns: radix <= 10 at 3 CTAs/SM measured faster
    op->PH = get_plan(ctx, g.n3, false, true);
    int prio_lo = 0, prio_hi = 0;  // high priority: decompression CTAs are dispatched before FFT-pass CTAs
    VIE_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    VIE_CUDA_CHECK(cudaStreamCreateWithPriority(&op->side, cudaStreamNonBlocking,
                                                env_int("VIE_SIDE_PRIO", 1) ? prio_hi : prio_lo));
    op->fork_after = env_int("VIE_FORK_AFTER", 0);
    VIE_CUDA_CHECK(cudaEventCreateWithFlags(&op->ev_fork, cudaEventDisableTiming));
    VIE_CUDA_CHECK(cudaEventCreateWithFlags(&op->ev_join, cudaEventDisableTiming));
    *out = op.release();
  });
}

int vie_op_destroy(vie_op op) {
  return guard([&] {
    if (!op) return;
    cudaSetDevice(op->ctx->device);
    cudaStreamSynchronize(op->ctx->stream);
    delete op;
  });
}

int vie_op_set_strategy(vie_op op, int strategy) {
  return guard([&] {
    if (!op) throw Invalid("set_strategy: null operator");
    if (strategy != VIE_STRATEGY_HOSVD_DECOMPRESS && strategy != VIE_STRATEGY_HOSVD_LOOP)
      throw Invalid("set_strategy: unknown strategy");
    const bool loop = strategy == VIE_STRATEGY_HOSVD_LOOP;
    if (loop && (!op->fused_ok || op->nranks > 1))
      throw Invalid("apply_operator: hosvd_loop (fused decompress x pencil kernel) needs a PWL operator with "
                    "ranks <= 28, a compiled axis-3 shape and no slab partition");
    if (loop == op->fused) return;
    VIE_CUDA_CHECK(cudaSetDevice(op->ctx->device));
    VIE_CUDA_CHECK(cudaStreamSynchronize(op->ctx->stream));
    op->fused = loop;
    ensure_spectra(op);
  });
}

int vie_op_get_strategy(vie_op op, int* strategy) {
  return guard([&] {
    if (!op || !strategy) throw Invalid("get_strategy: null argument");
    *strategy = op->fused ? VIE_STRATEGY_HOSVD_LOOP : VIE_STRATEGY_HOSVD_DECOMPRESS;
  });
}

// Debug hook (not part of the drop-in ABI): device pointer and element count of an operator
// buffer -- 0 Shat (octant spectra), 1 A, 2 B, 3 Bo, 4 Z -- for the determinism probes.
int vie_debug_op_buffer(vie_op op, int which, void** ptr, int64_t* elems) {
  return guard([&] {
    if (!op || !ptr || !elems) throw Invalid("vie_debug_op_buffer: null argument");
    const Geom& g = op->g;
    const int64_t nv = static_cast<int64_t>(g.n1) * g.n2 * g.n3;
    switch (which) {
      case 0: *ptr = op->Shat; *elems = op->Shat ? static_cast<int64_t>(g.n1 + 1) * (g.n2 + 1) * g.NC * (g.n3 + 1) : 0; break;
      case 1: *ptr = op->A; *elems = g.S * 2 * nv; break;
      case 2: *ptr = op->B; *elems = static_cast<int64_t>(g.S) * g.n3 * g.bps; break;
      case 3: *ptr = op->Bo; *elems = static_cast<int64_t>(g.S) * g.n3 * g.bps; break;
      default: throw Invalid("vie_debug_op_buffer: unknown buffer");
    }
  });
}

int vie_op_info(vie_op op, int64_t* n_cur, int64_t* n_vox, int64_t* workspace_bytes) {
  return guard([&] {
    if (!op) throw Invalid("vie_op_info: null operator");
    if (n_cur) *n_cur = op->g.S;
    if (n_vox) *n_vox = static_cast<int64_t>(op->g.n1) * op->g.n2 * op->g.n3;
    if (workspace_bytes) *workspace_bytes = op->ws_bytes;
  });
}

int vie_matvec(vie_op op, const double* x, double* y, void* stream) {
  return guard([&] {
    if (!op || !x || !y) throw Invalid("apply_operator: null argument");
    if (x == y) throw Invalid("apply_operator: x and y must not alias");
    VIE_CUDA_CHECK(cudaSetDevice(op->ctx->device));
    run_matvec(op, reinterpret_cast<const double2*>(x), reinterpret_cast<double2*>(y), pick_stream(op, stream),
               nullptr, 0.0, 0);
  });
}

// ---------------------------------------------------------------- slab decomposition

int vie_op_set_partition(vie_op op, int nranks, int rank) {
  return guard([&] {
    if (!op) throw Invalid("set_partition: null operator");
    if (nranks < 1 || rank < 0 || rank >= nranks) throw Invalid("set_partition: bad rank / size");
    Geom& g = op->g;
    const int group = 2 * (g.S >= 12 ? 1 : (g.S >= 6 ? 2 : 4));  // axis-1 positions per pencil group (kernels_pencil.cu pencil_p1pairs)
    if (g.n3 % nranks) throw Invalid("set_partition: n3 must be divisible by the number of ranks");
    if (g.m1 % nranks || (g.m1 / nranks) % group)
      throw Invalid("set_partition: 2*n1 must split into whole pencil groups per rank");
    if (nranks > 1 && !(op->q1 && op->q2))
      throw Invalid("set_partition: axis lengths need two-stage plans for the slab passes");
    VIE_CUDA_CHECK(cudaSetDevice(op->ctx->device));
    VIE_CUDA_CHECK(cudaStreamSynchronize(op->ctx->stream));
    if (nranks > 1 && op->fused) op->fused = false;  // the slab stages use the materialised rows
    op->nranks = nranks;
    op->rank = rank;
    g.nk = g.n3 / nranks;
    g.W = g.m1 / nranks;
    g.p1off = rank * g.W;
    g.bps = static_cast<int64_t>(g.m2) * g.W;
  });
}

int vie_slab_info(vie_op op, int64_t* x_elems, int64_t* slab_elems, int64_t* k0, int64_t* nk) {
  return guard([&] {
    if (!op) throw Invalid("slab_info: null operator");
    const Geom& g = op->g;
    if (x_elems) *x_elems = static_cast<int64_t>(g.S) * g.n1 * g.n2 * g.nk;
    if (slab_elems) *slab_elems = static_cast<int64_t>(g.S) * g.nk * g.n2 * g.m1;
    if (k0) *k0 = static_cast<int64_t>(op->rank) * g.nk;
    if (nk) *nk = g.nk;
  });
}

namespace {
Geom slab_geom_rows(const vie_op op) {  // the rank's z-slab for the axis-1 passes
  Geom gl = op->g;
  gl.n3 = op->g.nk;
  gl.m3 = 2 * op->g.nk;
  return gl;
}
Geom slab_geom_cols(const vie_op op) {  // all k-planes (blocked by source rank) of the rank's W columns
  Geom gc = op->g;
  gc.nk = op->g.n3;
  return gc;
}
}  // namespace

int vie_slab_forward(vie_op op, const double* x_local, double* send, void* stream) {
  return guard([&] {
    if (!op || !x_local || !send) throw Invalid("slab_forward: null argument");
    VIE_CUDA_CHECK(cudaSetDevice(op->ctx->device));
    cudaStream_t st = pick_stream(op, stream);
    const Geom gl = slab_geom_rows(op);
    const double2* x = reinterpret_cast<const double2*>(x_local);
    double2* A = reinterpret_cast<double2*>(send);  // [q][s][k][j][W] (blocked by pencil rank)
    if (op->q1) vie::launch_row_fwd2(x, A, gl, op->Q1, st);
    else vie::launch_row_fwd(x, A, gl, op->P1, st);
  });
}

namespace {
// octant spectra rows of this rank's axis-1 positions: pairs (2j, 2j+1) -> row j,
// positions 0, 1 -> rows 0 and n1 (x-independent)
void slab_decomp(vie_op op, cudaStream_t st) {
  const Geom& g = op->g;
  const int lo = g.p1off / 2, hi = (g.p1off + g.W) / 2;
  vie::launch_decomp(op->forms, op->comps_dev, op->comps_host.data(), op->Z, op->Shat, g, op->rmax, st, 0, -1,
                     true, lo, hi, op->u3img);
  if (g.p1off == 0)
    vie::launch_decomp(op->forms, op->comps_dev, op->comps_host.data(), op->Z, op->Shat, g, op->rmax, st, 0, -1,
                       false, g.n1, g.n1 + 1, op->u3img);
}

// The rank's pencil kernels on its axis-1 groups (B -> Bo)
void slab_pencils(vie_op op, cudaStream_t st) {
  const Geom& g = op->g;
  if (op->pencil3) {
    if (g.p1off == 0)
      vie::launch_pencil(op->kind, op->basis, op->B, op->Bo, nullptr, op->Shat, g, op->PH, op->P3.tw, op->active,
                         st, 1);
    vie::launch_pencil2(op->kind, op->basis, op->B, op->Bo, op->Shat, g, op->P3.tw, st, 0, 2);
    if (op->pencil4) vie::launch_pencil4(op->kind, op->B, op->Bo, op->Shat, g, op->P3.tw, st);
    else vie::launch_pencil3(op->kind, op->B, op->Bo, op->Shat, g, op->P3.tw, st);
  } else if (op->pencil2) {
    if (g.p1off == 0)
      vie::launch_pencil(op->kind, op->basis, op->B, op->Bo, nullptr, op->Shat, g, op->PH, op->P3.tw, op->active,
                         st, 1);
    vie::launch_pencil2(op->kind, op->basis, op->B, op->Bo, op->Shat, g, op->P3.tw, st);
  } else {
    vie::launch_pencil(op->kind, op->basis, op->B, op->Bo, nullptr, op->Shat, g, op->PH, op->P3.tw, op->active, st);
  }
}

// axis-2 FFTs of the rank's W columns over all k-planes (recv -> B) / inverse (Bo -> out); gc:
// the column geometry of the currents moved, pm: their planes in B (current groups)
void slab_col_fwd(vie_op op, const double2* recv, const Geom& gc, vie::PlaneMap pm, cudaStream_t st) {
  if (op->q2) vie::launch_col_fwd2(recv, op->B, gc, op->Q2, st, pm);
  else vie::launch_col_fwd(recv, op->B, gc, op->P2, st);
}
void slab_col_inv(vie_op op, double2* out, const Geom& gc, vie::PlaneMap pm, cudaStream_t st) {
  if (op->q2) vie::launch_col_inv2(op->Bo, out, gc, op->Q2, st, pm);
  else vie::launch_col_inv(op->Bo, nullptr, out, gc, op->P2, st);
}

// axis-2 FFTs of the rank's columns, the pencil stage on its octant rows, inverse axis-2 FFTs
void slab_pencil_stage(vie_op op, const double2* recv, double2* out, cudaStream_t st, bool with_decomp) {
  const Geom gc = slab_geom_cols(op);
  slab_col_fwd(op, recv, gc, {}, st);
  if (with_decomp) slab_decomp(op, st);
  slab_pencils(op, st);
  slab_col_inv(op, out, gc, {}, st);
}

// equal-split all-to-all of the rank-blocked slab (chunk q <-> rank q) as grouped NCCL
// point-to-point calls on `st` (the exchange step of SURVEY 8(e))
void slab_exchange(vie_op op, const double2* send, double2* recv, size_t chunk, cudaStream_t st) {
  vie_comm c = op->comm;  // chunk: double2 per peer
  if (c->lb) {  // loopback: send chunk q -> rank q's recv chunk [rank], between host barriers
    vie_loopback_s* lb = c->lb;
    VIE_CUDA_CHECK(cudaStreamSynchronize(st));  // send is complete, recv is free
    lb->ptr[static_cast<size_t>(c->rank)] = recv;
    lb->barrier();
    for (int q = 0; q < c->nranks; ++q)
      VIE_CUDA_CHECK(cudaMemcpyAsync(static_cast<double2*>(lb->ptr[static_cast<size_t>(q)]) + c->rank * chunk,
                                     send + q * chunk, sizeof(double2) * chunk, cudaMemcpyDefault, st));
    VIE_CUDA_CHECK(cudaStreamSynchronize(st));
    lb->barrier();  // every rank's chunks have landed
    return;
  }
  if (ncclGroupStart() != ncclSuccess) throw NcclError("ncclGroupStart failed");
  for (int q = 0; q < c->nranks; ++q) {
    const ncclResult_t r1 = ncclSend(send + q * chunk, 2 * chunk, ncclDouble, q, c->nccl, st);
    const ncclResult_t r2 = ncclRecv(recv + q * chunk, 2 * chunk, ncclDouble, q, c->nccl, st);
    if (r1 != ncclSuccess || r2 != ncclSuccess) throw NcclError(std::string("NCCL send/recv: ") + ncclGetErrorString(r1 != ncclSuccess ? r1 : r2));
  }
  const ncclResult_t r = ncclGroupEnd();
  if (r != ncclSuccess) throw NcclError(std::string("ncclGroupEnd: ") + ncclGetErrorString(r));
}

// The whole slab matvec of this rank with the in-library exchange.  The x-independent
// decomposition runs on the side stream from the start; the S currents move in G groups (SURVEY
// 8(e): the all-to-all of one group overlaps the FFTs of the others): on the compute stream the
// axis-1 FFTs of every group, then per group [wait for its exchange] its axis-2 FFTs; the
// exchanges run on the comm stream as each group's FFTs finish.  The same on the way back.
// Exchange buffers are group-major: [g][rank][s in group][k][j][w < W].
void slab_matvec_run(vie_op op, const double2* x, double2* y, const double2* eps, double inv_v, int diag,
                     cudaStream_t st) {
  if (!op->comm) throw Invalid("slab_matvec: no communicator (vie_op_set_comm)");
  ensure_spectra(op);
  const Geom& g = op->g;
  const int64_t se = static_cast<int64_t>(g.S) * g.nk * g.n2 * g.m1;
  for (double2** p : {&op->xs_send, &op->xs_recv, &op->xs_out, &op->xs_back})
    if (!*p) *p = dev_alloc<double2>(static_cast<size_t>(se));
  // current groups: PWL 3 x 4 (the apply_system weights repeat every 4 currents), PWC 3 x 1
  static const int g_env = env_int("VIE_SLAB_GROUPS", 3);
  const int G = (op->q1 && op->q2 && g_env > 1 && g.S % g_env == 0 && (g.S / g_env) % (g.S == 12 ? 4 : 1) == 0)
                    ? g_env : 1;
  const int Sg = g.S / G, R = op->nranks;
  if (!op->s_comm) VIE_CUDA_CHECK(cudaStreamCreateWithFlags(&op->s_comm, cudaStreamNonBlocking));
  if (static_cast<int>(op->ev_grp.size()) < 4 * G) {
    for (cudaEvent_t e : op->ev_grp) cudaEventDestroy(e);
    op->ev_grp.assign(static_cast<size_t>(4 * G), nullptr);
    for (cudaEvent_t& e : op->ev_grp) VIE_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  cudaEvent_t* ev_row = op->ev_grp.data();
  cudaEvent_t* ev_in = ev_row + G;
  cudaEvent_t* ev_ci = ev_in + G;
  cudaEvent_t* ev_back = ev_ci + G;
  cudaStream_t cs = op->s_comm;
  VIE_CUDA_CHECK(cudaEventRecord(op->ev_fork, st));
  VIE_CUDA_CHECK(cudaStreamWaitEvent(op->side, op->ev_fork, 0));
  slab_decomp(op, op->side);
  VIE_CUDA_CHECK(cudaEventRecord(op->ev_join, op->side));
  Geom gl = slab_geom_rows(op);  // one group's rows: S = Sg
  gl.S = Sg;
  Geom gc = slab_geom_cols(op);  // one group's column planes
  gc.S = Sg;
  const size_t chunk = static_cast<size_t>(Sg) * g.nk * g.n2 * g.W;  // double2 per peer per group
  const int64_t xg = static_cast<int64_t>(Sg) * g.nk * g.n2 * g.n1;   // x / y elements per group
  const int64_t blk = static_cast<int64_t>(R) * chunk;                // exchange elements per group
  auto pmap = [&](int gi) {
    vie::PlaneMap pm;
    pm.in_per_r = Sg * g.nk;
    pm.out_per_r = g.S * g.nk;
    pm.off = gi * Sg * g.nk;
    return pm;
  };
  for (int gi = 0; gi < G; ++gi) {
    if (op->q1) vie::launch_row_fwd2(x + gi * xg, op->xs_send + gi * blk, gl, op->Q1, st);
    else vie::launch_row_fwd(x + gi * xg, op->xs_send + gi * blk, gl, op->P1, st);
    VIE_CUDA_CHECK(cudaEventRecord(ev_row[gi], st));
  }
  for (int gi = 0; gi < G; ++gi) {
    VIE_CUDA_CHECK(cudaStreamWaitEvent(cs, ev_row[gi], 0));
    slab_exchange(op, op->xs_send + gi * blk, op->xs_recv + gi * blk, chunk, cs);
    VIE_CUDA_CHECK(cudaEventRecord(ev_in[gi], cs));
  }
  for (int gi = 0; gi < G; ++gi) {
    VIE_CUDA_CHECK(cudaStreamWaitEvent(st, ev_in[gi], 0));
    slab_col_fwd(op, op->xs_recv + gi * blk, gc, pmap(gi), st);
  }
  VIE_CUDA_CHECK(cudaStreamWaitEvent(st, op->ev_join, 0));
  slab_pencils(op, st);
  for (int gi = 0; gi < G; ++gi) {
    slab_col_inv(op, op->xs_out + gi * blk, gc, pmap(gi), st);
    VIE_CUDA_CHECK(cudaEventRecord(ev_ci[gi], st));
  }
  for (int gi = 0; gi < G; ++gi) {
    VIE_CUDA_CHECK(cudaStreamWaitEvent(cs, ev_ci[gi], 0));
    slab_exchange(op, op->xs_out + gi * blk, op->xs_back + gi * blk, chunk, cs);
    VIE_CUDA_CHECK(cudaEventRecord(ev_back[gi], cs));
  }
  const double ne = 8.0 * g.n1 * static_cast<double>(g.n2) * g.n3;  // global N_e
  for (int gi = 0; gi < G; ++gi) {
    VIE_CUDA_CHECK(cudaStreamWaitEvent(st, ev_back[gi], 0));
    const double2* xgi = x + gi * xg;
    if (op->q1)
      vie::launch_row_inv2(op->xs_back + gi * blk, y + gi * xg, gl, op->Q1, 1.0 / ne, eps, xgi, inv_v, op->basis, diag,
                           st);
    else
      vie::launch_row_inv(op->xs_back + gi * blk, y + gi * xg, gl, op->P1, 1.0 / ne, eps, xgi, inv_v, op->basis, diag,
                          st);
  }
}
}  // namespace

int vie_slab_pencil(vie_op op, const double* recv, double* out, void* stream) {
  return guard([&] {
    if (!op || !recv || !out) throw Invalid("slab_pencil: null argument");
    if (recv == out) throw Invalid("slab_pencil: recv and out must not alias");
    VIE_CUDA_CHECK(cudaSetDevice(op->ctx->device));
    ensure_spectra(op);
    slab_pencil_stage(op, reinterpret_cast<const double2*>(recv), reinterpret_cast<double2*>(out),
                      pick_stream(op, stream), true);
  });
}

int vie_slab_inverse(vie_op op, const double* back, double* y_local, const double* eps_local, double inv_v,
                     const double* x_local, int diag_term, void* stream) {
  return guard([&] {
    if (!op || !back || !y_local) throw Invalid("slab_inverse: null argument");
    if (eps_local && op->kind != VIE_KIND_N) throw Invalid("apply_system: needs the N operator");
    if (eps_local && diag_term && !x_local) throw Invalid("apply_system: null argument");
    VIE_CUDA_CHECK(cudaSetDevice(op->ctx->device));
    cudaStream_t st = pick_stream(op, stream);
    const Geom gl = slab_geom_rows(op);
    const double ne = 8.0 * op->g.n1 * static_cast<double>(op->g.n2) * op->g.n3;  // global N_e
    const double2* A = reinterpret_cast<const double2*>(back);
    double2* y = reinterpret_cast<double2*>(y_local);
    const double2* eps = reinterpret_cast<const double2*>(eps_local);
    const double2* xin = reinterpret_cast<const double2*>(x_local);
    if (op->q1)
      vie::launch_row_inv2(A, y, gl, op->Q1, 1.0 / ne, eps, xin, inv_v, op->basis, diag_term ? 1 : 0, st);
    else
      vie::launch_row_inv(A, y, gl, op->P1, 1.0 / ne, eps, xin, inv_v, op->basis, diag_term ? 1 : 0, st);
  });
}

int vie_comm_unique_id(unsigned char id[VIE_COMM_ID_BYTES]) {
  return guard([&] {
    if (!id) throw Invalid("comm_unique_id: null argument");
    static_assert(sizeof(ncclUniqueId) <= VIE_COMM_ID_BYTES, "NCCL unique id size");
    ncclUniqueId u;
    const ncclResult_t r = ncclGetUniqueId(&u);
    if (r != ncclSuccess) throw NcclError(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    std::memset(id, 0, VIE_COMM_ID_BYTES);
    std::memcpy(id, &u, sizeof(u));
  });
}

int vie_comm_create(vie_ctx ctx, int nranks, int rank, const unsigned char id[VIE_COMM_ID_BYTES], vie_comm* out) {
  return guard([&] {
    if (!ctx || !id || !out) throw Invalid("comm_create: null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) throw Invalid("comm_create: bad rank / size");
    VIE_CUDA_CHECK(cudaSetDevice(ctx->device));
    std::unique_ptr<vie_comm_s> c(new vie_comm_s);
    c->nranks = nranks;
    c->rank = rank;
    c->device = ctx->device;
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    const ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, u, rank);
    if (r != ncclSuccess) throw NcclError(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    *out = c.release();
  });
}

int vie_comm_destroy(vie_comm comm) {
  return guard([&] { delete comm; });
}

int vie_loopback_create(int nranks, vie_loopback* out) {
  return guard([&] {
    if (nranks < 1 || !out) throw Invalid("loopback_create: bad size / null argument");
    std::unique_ptr<vie_loopback_s> lb(new vie_loopback_s);
    lb->nranks = nranks;
    lb->ptr.assign(static_cast<size_t>(nranks), nullptr);
    lb->h.assign(static_cast<size_t>(nranks), {});
    *out = lb.release();
  });
}

int vie_loopback_destroy(vie_loopback lb) {
  return guard([&] { delete lb; });
}

int vie_comm_create_loopback(vie_ctx ctx, vie_loopback lb, int rank, vie_comm* out) {
  return guard([&] {
    if (!ctx || !lb || !out) throw Invalid("comm_create_loopback: null argument");
    if (rank < 0 || rank >= lb->nranks) throw Invalid("comm_create_loopback: bad rank");
    std::unique_ptr<vie_comm_s> c(new vie_comm_s);
    c->lb = lb;
    c->nranks = lb->nranks;
    c->rank = rank;
    c->device = ctx->device;
    *out = c.release();
  });
}

int vie_op_set_comm(vie_op op, vie_comm comm) {
  return guard([&] {
    if (!op) throw Invalid("set_comm: null operator");
    if (comm && (comm->nranks != op->nranks || comm->rank != op->rank))
      throw Invalid("set_comm: communicator rank / size differ from the operator's partition");
    if (comm && comm->device != op->ctx->device) throw Invalid("set_comm: communicator on another device");
    op->comm = comm;
  });
}

int vie_slab_matvec(vie_op op, const double* x_local, double* y_local, const double* eps_local, double inv_v,
                    int diag_term, void* stream) {
  return guard([&] {
    if (!op || !x_local || !y_local) throw Invalid("slab_matvec: null argument");
    if (x_local == y_local) throw Invalid("slab_matvec: x and y must not alias");
    if (eps_local && op->kind != VIE_KIND_N) throw Invalid("apply_system: needs the N operator");
    VIE_CUDA_CHECK(cudaSetDevice(op->ctx->device));
    slab_matvec_run(op, reinterpret_cast<const double2*>(x_local), reinterpret_cast<double2*>(y_local),
                    reinterpret_cast<const double2*>(eps_local), inv_v, eps_local ? (diag_term ? 1 : 0) : 0,
                    pick_stream(op, stream));
  });
}

int vie_matvec_host(vie_op op, const double* x_host, double* y_host) {
  return guard([&] {
    if (!op || !x_host || !y_host) throw Invalid("apply_operator: null argument");
    VIE_CUDA_CHECK(cudaSetDevice(op->ctx->device));
    const int64_t n = static_cast<int64_t>(op->g.S) * op->g.n1 * op->g.n2 * op->g.n3;
    if (!op->hx) op->hx = dev_alloc<double2>(static_cast<size_t>(n));
    if (!op->hy) op->hy = dev_alloc<double2>(static_cast<size_t>(n));
    cudaStream_t st = op->ctx->stream;
    fork_decomp(op, st);  // decompression overlaps the H2D copy
    VIE_CUDA_CHECK(cudaMemcpyAsync(op->hx, x_host, sizeof(double2) * n, cudaMemcpyHostToDevice, st));
    run_matvec(op, op->hx, op->hy, st, nullptr, 0.0, 0, true);
    VIE_CUDA_CHECK(cudaMemcpyAsync(y_host, op->hy, sizeof(double2) * n, cudaMemcpyDeviceToHost, st));
    VIE_CUDA_CHECK(cudaStreamSynchronize(st));
  });
}

int vie_matvec_host_batch(vie_op op, int64_t count, const double* const* x_host, double* const* y_host) {
  return guard([&] {
    if (!op || count < 0 || (count > 0 && (!x_host || !y_host))) throw Invalid("apply_operator: null argument");
    for (int64_t i = 0; i < count; ++i)
      if (!x_host[i] || !y_host[i]) throw Invalid("apply_operator: null argument");
    VIE_CUDA_CHECK(cudaSetDevice(op->ctx->device));
    const int64_t n = static_cast<int64_t>(op->g.S) * op->g.n1 * op->g.n2 * op->g.n3;
    const size_t bytes = sizeof(double2) * static_cast<size_t>(n);
    for (double2** p : {&op->hx, &op->hy, &op->hx2, &op->hy2})
      if (!*p) *p = dev_alloc<double2>(static_cast<size_t>(n));
    if (!op->s_h2d) VIE_CUDA_CHECK(cudaStreamCreateWithFlags(&op->s_h2d, cudaStreamNonBlocking));
    if (!op->s_d2h) VIE_CUDA_CHECK(cudaStreamCreateWithFlags(&op->s_d2h, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i)
      for (cudaEvent_t* e : {&op->ev_h2d[i], &op->ev_done[i], &op->ev_d2h[i]})
        if (!*e) VIE_CUDA_CHECK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    double2* dx[2] = {op->hx, op->hx2};
    double2* dy[2] = {op->hy, op->hy2};
    cudaStream_t st = op->ctx->stream;
    // three-stage pipeline: H2D(i+1) and D2H(i-1) on their own copy streams overlap
    // matvec(i); two device slots per direction, each reused once its consumer is done
    for (int64_t i = 0; i < count; ++i) {
      const int sl = static_cast<int>(i & 1);
      if (i >= 2) VIE_CUDA_CHECK(cudaStreamWaitEvent(op->s_h2d, op->ev_done[sl], 0));  // matvec(i-2) read dx[sl]
      VIE_CUDA_CHECK(cudaMemcpyAsync(dx[sl], x_host[i], bytes, cudaMemcpyHostToDevice, op->s_h2d));
      VIE_CUDA_CHECK(cudaEventRecord(op->ev_h2d[sl], op->s_h2d));
      VIE_CUDA_CHECK(cudaStreamWaitEvent(st, op->ev_h2d[sl], 0));
      if (i >= 2) VIE_CUDA_CHECK(cudaStreamWaitEvent(st, op->ev_d2h[sl], 0));  // D2H(i-2) drained dy[sl]
      run_matvec(op, dx[sl], dy[sl], st, nullptr, 0.0, 0);
      VIE_CUDA_CHECK(cudaEventRecord(op->ev_done[sl], st));
      VIE_CUDA_CHECK(cudaStreamWaitEvent(op->s_d2h, op->ev_done[sl], 0));
      VIE_CUDA_CHECK(cudaMemcpyAsync(y_host[i], dy[sl], bytes, cudaMemcpyDeviceToHost, op->s_d2h));
      VIE_CUDA_CHECK(cudaEventRecord(op->ev_d2h[sl], op->s_d2h));
    }
    VIE_CUDA_CHECK(cudaStreamSynchronize(op->s_d2h));
    VIE_CUDA_CHECK(cudaStreamSynchronize(st));
  });
}

int vie_system_matvec(vie_op op, const double* eps_r, double inv_v, const double* x, double* y, int diag_term,
                      void* stream) {
  return guard([&] {
    if (!op || !eps_r || !x || !y) throw Invalid("apply_system: null argument");
    if (x == y) throw Invalid("apply_system: x and y must not alias");
    if (op->kind != VIE_KIND_N) throw Invalid("apply_system: needs the N operator");
    VIE_CUDA_CHECK(cudaSetDevice(op->ctx->device));
    run_matvec(op, reinterpret_cast<const double2*>(x), reinterpret_cast<double2*>(y), pick_stream(op, stream),
               reinterpret_cast<const double2*>(eps_r), inv_v, diag_term ? 1 : 0);
  });
}

}  // extern "C"

namespace {

// ---------------------------------------------------------------- GMRES core
// Device-resident restarted GMRES(inner) with modified Gram-Schmidt and complex Givens
// rotations, exactly the reference's order of operations (solver.hpp:34-142), on any
// device linear map `apply`, with an optional right preconditioner M (solver.hpp:74,
// :131: w = A M v_j, x += M V y; residual estimates stay those of the original system).
// `allreduce`, when set, sums device scalars over the ranks of a distributed solve (the
// MGS dots and norms) right after each reduction kernel.
struct GmresWork {
  double2* V = nullptr;    // (inner + 1) * n basis
  double2* tmp = nullptr;  // n
  double2* zp = nullptr;   // n (preconditioned vector), only with a preconditioner
  double2* scal = nullptr; // 256 device scalars
  vie::RedBuf rb{};
};
struct GmresOut {
  int iters = 0;
  bool conv = false;
  double final_rel = 0.0;
  std::vector<double> history;
};
using DevMap = std::function<void(const double2*, double2*)>;
using DevReduce = std::function<void(double2*, int)>;

GmresOut gmres_core(cudaStream_t st, int64_t n, const DevMap& apply, const DevMap& precond, const DevReduce& allreduce,
                    const double2* rhs, const double2* x0, double tol, int inner, int outer, double2* x,
                    const GmresWork& w) {
  if (tol < 0 || inner < 1 || outer < 1) throw Invalid("gmres: invalid configuration");
  if (inner + 2 > 256) throw Invalid("gmres: inner > 254 not supported");
  double2* V = w.V;
  double2* tmp = w.tmp;
  double2* hd = w.scal;  // hd[0..j+1]
  auto reduce = [&](double2* p, int count) {
    if (allreduce) allreduce(p, count);
  };
  auto fetch = [&](int count, std::vector<double2>& h) {
    h.resize(static_cast<size_t>(count));
    VIE_CUDA_CHECK(cudaMemcpyAsync(h.data(), hd, sizeof(double2) * count, cudaMemcpyDeviceToHost, st));
    VIE_CUDA_CHECK(cudaStreamSynchronize(st));
  };
  std::vector<double2> hbuf;
  GmresOut out;
  // ||b|| (solver.hpp:43) and the non-finite check (:37)
  vie::launch_nrm2sq(rhs, n, hd, w.rb, st);
  reduce(hd, 1);
  fetch(1, hbuf);
  if (!std::isfinite(hbuf[0].x)) throw Invalid("gmres: non-finite right-hand side");
  const double bnorm = std::sqrt(hbuf[0].x);
  if (x0) {
    if (x0 != x) VIE_CUDA_CHECK(cudaMemcpyAsync(x, x0, sizeof(double2) * n, cudaMemcpyDeviceToDevice, st));
  } else {
    VIE_CUDA_CHECK(cudaMemsetAsync(x, 0, sizeof(double2) * n, st));
  }
  if (bnorm == 0.0) {  // solver.hpp:46-51
    VIE_CUDA_CHECK(cudaMemsetAsync(x, 0, sizeof(double2) * n, st));
    out.conv = true;
    out.history.push_back(0.0);
    VIE_CUDA_CHECK(cudaStreamSynchronize(st));
    return out;
  }
  const int m = inner;
  std::vector<cd> hess(static_cast<size_t>((m + 1) * m), cd(0.0));
  auto H = [&](int i, int j) -> cd& { return hess[static_cast<size_t>(i + (m + 1) * j)]; };
  std::vector<cd> gv(static_cast<size_t>(m + 1)), cs(static_cast<size_t>(m)), sn(static_cast<size_t>(m));
  for (int restart = 0; restart < outer && !out.conv; ++restart) {
    apply(x, tmp);
    vie::launch_residual(rhs, tmp, V, n, hd, w.rb, st);  // V_0 = r
    reduce(hd, 1);
    fetch(1, hbuf);
    const double beta = std::sqrt(hbuf[0].x);
    if (beta / bnorm <= tol) {
      out.conv = true;
      break;
    }
    vie::launch_scale_inv(V, V, nullptr, beta, n, st);  // basis.col(0) = r / beta
    std::fill(gv.begin(), gv.end(), cd(0.0));
    gv[0] = beta;
    int j = 0;
    bool breakdown = false;
    for (; j < m; ++j) {
      double2* vj = V + static_cast<int64_t>(j) * n;
      double2* wv = V + static_cast<int64_t>(j + 1) * n;
      if (precond) {  // w = A (M v_j)
        precond(vj, w.zp);
        apply(w.zp, wv);
      } else {
        apply(vj, wv);
      }
      vie::launch_dot(V, wv, n, hd, w.rb, st);  // h_0j
      reduce(hd, 1);
      for (int i = 0; i <= j; ++i) {
        const double2* vi = V + static_cast<int64_t>(i) * n;
        const double2* vn = i < j ? V + static_cast<int64_t>(i + 1) * n : nullptr;
        vie::launch_mgs_step(wv, vi, hd + i, vn, n, hd + i + 1, w.rb, st);
        reduce(hd + i + 1, 1);
      }
      fetch(j + 2, hbuf);
      for (int i = 0; i <= j; ++i) H(i, j) = cd(hbuf[static_cast<size_t>(i)].x, hbuf[static_cast<size_t>(i)].y);
      const double wnorm = std::sqrt(hbuf[static_cast<size_t>(j + 1)].x);
      H(j + 1, j) = wnorm;
      for (int i = 0; i < j; ++i) {
        const cd t = cs[static_cast<size_t>(i)] * H(i, j) + sn[static_cast<size_t>(i)] * H(i + 1, j);
        H(i + 1, j) = -std::conj(sn[static_cast<size_t>(i)]) * H(i, j) + std::conj(cs[static_cast<size_t>(i)]) * H(i + 1, j);
        H(i, j) = t;
      }
      {
        const cd a = H(j, j), bb = H(j + 1, j);
        const double denom = std::sqrt(std::norm(a) + std::norm(bb));
        if (denom == 0.0) {
          cs[static_cast<size_t>(j)] = 1.0;
          sn[static_cast<size_t>(j)] = 0.0;
        } else {
          cs[static_cast<size_t>(j)] = std::conj(a) / denom;
          sn[static_cast<size_t>(j)] = std::conj(bb) / denom;
        }
        H(j, j) = cs[static_cast<size_t>(j)] * a + sn[static_cast<size_t>(j)] * bb;
        H(j + 1, j) = 0.0;
        const cd t = cs[static_cast<size_t>(j)] * gv[static_cast<size_t>(j)];
        gv[static_cast<size_t>(j + 1)] = -std::conj(sn[static_cast<size_t>(j)]) * gv[static_cast<size_t>(j)];
        gv[static_cast<size_t>(j)] = t;
      }
      ++out.iters;
      const double rel = std::abs(gv[static_cast<size_t>(j + 1)]) / bnorm;
      out.history.push_back(rel);
      if (rel <= tol) {
        ++j;
        out.conv = true;
        break;
      }
      if (wnorm < 1e-14 * beta) {
        ++j;
        breakdown = true;
        break;
      }
      vie::launch_scale_inv(wv, wv, nullptr, wnorm, n, st);  // basis.col(j+1) = w / wnorm
    }
    std::vector<cd> yv(static_cast<size_t>(j), cd(0.0));
    for (int i = j - 1; i >= 0; --i) {
      cd sacc = gv[static_cast<size_t>(i)];
      for (int l = i + 1; l < j; ++l) sacc -= H(i, l) * yv[static_cast<size_t>(l)];
      yv[static_cast<size_t>(i)] = sacc / H(i, i);
    }
    if (j > 0) {
      std::vector<double2> yd(static_cast<size_t>(j));
      for (int l = 0; l < j; ++l) yd[static_cast<size_t>(l)] = make_double2(yv[static_cast<size_t>(l)].real(), yv[static_cast<size_t>(l)].imag());
      VIE_CUDA_CHECK(cudaMemcpyAsync(hd, yd.data(), sizeof(double2) * j, cudaMemcpyHostToDevice, st));
      if (precond) {  // x += M (V y)  (solver.hpp:130-131)
        VIE_CUDA_CHECK(cudaMemsetAsync(tmp, 0, sizeof(double2) * n, st));
        vie::launch_basis_update(tmp, V, n, hd, j, n, st);
        precond(tmp, w.zp);
        vie::launch_axpy1(x, w.zp, n, st);
      } else {
        vie::launch_basis_update(x, V, n, hd, j, n, st);  // x += V y
      }
      VIE_CUDA_CHECK(cudaStreamSynchronize(st));  // the host y staging is reused next cycle
    }
    if (breakdown && !out.conv) {
      apply(x, tmp);
      vie::launch_residual(rhs, tmp, nullptr, n, hd, w.rb, st);
      reduce(hd, 1);
      fetch(1, hbuf);
      const double rel = std::sqrt(hbuf[0].x) / bnorm;
      out.conv = rel <= tol;
      if (out.conv) break;
    }
  }
  apply(x, tmp);
  vie::launch_residual(rhs, tmp, nullptr, n, hd, w.rb, st);
  reduce(hd, 1);
  fetch(1, hbuf);
  out.final_rel = std::sqrt(hbuf[0].x) / bnorm;
  VIE_CUDA_CHECK(cudaStreamSynchronize(st));
  return out;
}

DevMap make_precond(const vie_precond* pc, int64_t n, cudaStream_t st) {
  if (!pc || (!pc->diag && !pc->apply)) return nullptr;
  if (pc->diag && pc->apply) throw Invalid("gmres: preconditioner has both a diagonal and a callback");
  if (pc->diag) {
    const double2* d = reinterpret_cast<const double2*>(pc->diag);
    return [d, n, st](const double2* in, double2* out) { vie::launch_cmul_elem(d, in, out, n, st); };
  }
  return [pc, st](const double2* in, double2* out) {
    pc->apply(pc->user, reinterpret_cast<const double*>(in), reinterpret_cast<double*>(out), st);
  };
}

void report(const GmresOut& g, int* iterations, double* final_rel_res, double* history_host, int history_cap,
            int* history_len, int* converged) {
  if (iterations) *iterations = g.iters;
  if (final_rel_res) *final_rel_res = g.final_rel;
  if (converged) *converged = g.conv ? 1 : 0;
  if (history_len) *history_len = static_cast<int>(g.history.size());
  if (history_host)
    for (int i = 0; i < history_cap && i < static_cast<int>(g.history.size()); ++i)
      history_host[i] = g.history[static_cast<size_t>(i)];
}

// the solve runs on the context stream ordered after `user` (event), and `user` waits for it
struct StreamJoin {
  cudaStream_t st, user;
  cudaEvent_t ev;
  StreamJoin(cudaStream_t s, cudaStream_t u, cudaEvent_t e) : st(s), user(u), ev(e) {
    if (user && user != st) {
      VIE_CUDA_CHECK(cudaEventRecord(ev, user));
      VIE_CUDA_CHECK(cudaStreamWaitEvent(st, ev, 0));
    }
  }
  void done() {
    if (user && user != st) {
      VIE_CUDA_CHECK(cudaEventRecord(ev, st));
      VIE_CUDA_CHECK(cudaStreamWaitEvent(user, ev, 0));
    }
  }
};

}  // namespace

extern "C" {

int vie_gmres_solve(vie_op op, const double* eps_r, double inv_v, const double* rhs_d, const double* x0_d,
                    double tol, int inner, int outer, const vie_precond* precond, double* x_d, int* iterations,
                    double* final_rel_res, double* history_host, int history_cap, int* history_len, int* converged,
                    void* stream) {
  return guard([&] {
    if (!op || !eps_r || !rhs_d || !x_d) throw Invalid("gmres: null argument");
    if (tol < 0 || inner < 1 || outer < 1) throw Invalid("gmres: invalid configuration");
    if (op->kind != VIE_KIND_N) throw Invalid("gmres: needs the N operator");
    if (op->nranks > 1 && !op->comm) throw Invalid("gmres: partitioned operator needs a communicator (vie_op_set_comm)");
    VIE_CUDA_CHECK(cudaSetDevice(op->ctx->device));
    cudaStream_t st = op->ctx->stream;
    const Geom& g = op->g;
    // distributed (slab-partitioned, with a communicator): the vectors are this rank's z-slabs
    const bool dist = op->comm != nullptr;
    const int64_t n = static_cast<int64_t>(g.S) * g.n1 * g.n2 * (dist ? g.nk : g.n3);
    if (op->g_inner < inner) {
      dev_free(op->V);
      op->V = nullptr;
      op->V = dev_alloc<double2>(static_cast<size_t>(n) * (inner + 1));
      op->g_inner = inner;
    }
    if (!op->tmp) op->tmp = dev_alloc<double2>(static_cast<size_t>(n));
    if (precond && !op->zp) op->zp = dev_alloc<double2>(static_cast<size_t>(n));
    if (!op->scal) op->scal = dev_alloc<double2>(256);
    if (!op->red_partials) {
      op->red_partials = dev_alloc<double2>(vie::kRedBlocks);
      op->red_counter = dev_alloc<unsigned int>(1);
      VIE_CUDA_CHECK(cudaMemsetAsync(op->red_counter, 0, sizeof(unsigned int), st));
    }
    if (!op->ev_user) VIE_CUDA_CHECK(cudaEventCreateWithFlags(&op->ev_user, cudaEventDisableTiming));
    StreamJoin sj(st, static_cast<cudaStream_t>(stream), op->ev_user);
    GmresWork w{op->V, op->tmp, op->zp, op->scal, vie::RedBuf{op->red_partials, op->red_counter}};
    const double2* eps = reinterpret_cast<const double2*>(eps_r);
    auto sysmv = [&](const double2* in, double2* outv) {
      if (dist) slab_matvec_run(op, in, outv, eps, inv_v, 1, st);
      else run_matvec(op, in, outv, st, eps, inv_v, 1);
    };
    // every dot / norm of the distributed solve is summed over the ranks (solver.hpp:75-79 on
    // distributed vectors): one ncclAllReduce of the device scalars, in place, on the solve stream
    DevReduce allreduce;
    if (dist)
      allreduce = [&](double2* p, int count) {
        vie_comm c = op->comm;
        if (c->lb) {  // loopback: host sum in rank order, the same on every rank
          vie_loopback_s* lb = c->lb;
          auto& mine = lb->h[static_cast<size_t>(c->rank)];
          mine.resize(2 * static_cast<size_t>(count));
          VIE_CUDA_CHECK(cudaMemcpyAsync(mine.data(), p, sizeof(double2) * count, cudaMemcpyDeviceToHost, st));
          VIE_CUDA_CHECK(cudaStreamSynchronize(st));
          lb->barrier();
          std::vector<double> sum(2 * static_cast<size_t>(count), 0.0);
          for (int q = 0; q < c->nranks; ++q)
            for (size_t i = 0; i < sum.size(); ++i) sum[i] += lb->h[static_cast<size_t>(q)][i];
          lb->barrier();  // every rank has read every contribution
          VIE_CUDA_CHECK(cudaMemcpyAsync(p, sum.data(), sizeof(double2) * count, cudaMemcpyHostToDevice, st));
          VIE_CUDA_CHECK(cudaStreamSynchronize(st));
          return;
        }
        const ncclResult_t rr = ncclAllReduce(p, p, 2 * static_cast<size_t>(count), ncclDouble, ncclSum, c->nccl, st);
        if (rr != ncclSuccess) throw NcclError(std::string("ncclAllReduce: ") + ncclGetErrorString(rr));
      };
    const GmresOut r = gmres_core(st, n, sysmv, make_precond(precond, n, st), allreduce,
                                  reinterpret_cast<const double2*>(rhs_d), reinterpret_cast<const double2*>(x0_d), tol,
                                  inner, outer, reinterpret_cast<double2*>(x_d), w);
    sj.done();
    report(r, iterations, final_rel_res, history_host, history_cap, history_len, converged);
  });
}

int vie_gmres(vie_ctx ctx, int64_t n, vie_linear_map_fn apply, void* apply_user, const double* rhs_d,
              const double* x0_d, double tol, int inner, int outer, const vie_precond* precond, double* x_d,
              int* iterations, double* final_rel_res, double* history_host, int history_cap, int* history_len,
              int* converged, void* stream) {
  return guard([&] {
    if (!ctx || !apply || !rhs_d || !x_d || n < 1) throw Invalid("gmres: null argument");
    VIE_CUDA_CHECK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    DevPool pool;
    GmresWork w;
    if (inner >= 1 && inner + 2 <= 256) w.V = pool.alloc<double2>(static_cast<size_t>(n) * (inner + 1));
    w.tmp = pool.alloc<double2>(static_cast<size_t>(n));
    if (precond) w.zp = pool.alloc<double2>(static_cast<size_t>(n));
    w.scal = pool.alloc<double2>(256);
    w.rb.partials = pool.alloc<double2>(vie::kRedBlocks);
    w.rb.counter = pool.alloc<unsigned int>(1);
    VIE_CUDA_CHECK(cudaMemsetAsync(w.rb.counter, 0, sizeof(unsigned int), st));
    cudaEvent_t ev = nullptr;
    VIE_CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    struct EvGuard {
      cudaEvent_t e;
      ~EvGuard() { cudaEventDestroy(e); }
    } evg{ev};
    StreamJoin sj(st, static_cast<cudaStream_t>(stream), ev);
    auto amap = [&](const double2* in, double2* outv) {
      apply(apply_user, reinterpret_cast<const double*>(in), reinterpret_cast<double*>(outv), st);
    };
    const GmresOut r = gmres_core(st, n, amap, make_precond(precond, n, st), nullptr,
                                  reinterpret_cast<const double2*>(rhs_d), reinterpret_cast<const double2*>(x0_d), tol,
                                  inner, outer, reinterpret_cast<double2*>(x_d), w);
    sj.done();
    VIE_CUDA_CHECK(cudaStreamSynchronize(st));
    report(r, iterations, final_rel_res, history_host, history_cap, history_len, converged);
  });
}

int vie_matvec_timed(vie_op op, const double* x, double* y, double* fft_ms, double* product_ms) {
  return guard([&] {
    if (!op || !x || !y) throw Invalid("apply_operator: null argument");
    if (x == y) throw Invalid("apply_operator: x and y must not alias");
    VIE_CUDA_CHECK(cudaSetDevice(op->ctx->device));
    const int saved = op->profiling;
    op->profiling = 1;  // serial stages, one event interval each
    try {
      run_matvec(op, reinterpret_cast<const double2*>(x), reinterpret_cast<double2*>(y), op->ctx->stream, nullptr,
                 0.0, 0);
    } catch (...) {
      op->profiling = saved;
      throw;
    }
    op->profiling = saved;
    const double* t = op->stage_ms;  // row, column, decompression, pencil, column^-1, row^-1
    if (fft_ms) *fft_ms = t[0] + t[1] + t[4] + t[5];
    if (product_ms) *product_ms = t[2] + t[3];
  });
}

int vie_op_set_profiling(vie_op op, int enable) {
  return guard([&] {
    if (!op) throw Invalid("vie_op_set_profiling: null operator");
    op->profiling = enable == 2 ? 2 : (enable ? 1 : 0);
  });
}

int vie_op_last_stats(vie_op op, int* launches, double* stage_ms) {
  return guard([&] {
    if (!op) throw Invalid("vie_op_last_stats: null operator");
    if (launches) *launches = op->last_launches;
    if (stage_ms)
      for (int i = 0; i < 8; ++i) stage_ms[i] = op->stage_ms[i];
  });
}

#ifdef VIE_PENCIL_PROFILE
}  // extern "C"
namespace vie {
void pencil_phase_read(unsigned long long* out8, bool reset);
void pencil2_phase_read(unsigned long long* out8, bool reset);
void pencil3_phase_read(unsigned long long* out8, bool reset);
void pencil4_phase_read(unsigned long long* out8, bool reset);
}
extern "C" {
int vie_debug_pencil_phases(unsigned long long* out8, int reset) {
  return guard([&] { vie::pencil_phase_read(out8, reset != 0); });
}
int vie_debug_pencil2_phases(unsigned long long* out8, int reset) {
  return guard([&] { vie::pencil2_phase_read(out8, reset != 0); });
}
int vie_debug_pencil3_phases(unsigned long long* out8, int reset) {
  return guard([&] { vie::pencil3_phase_read(out8, reset != 0); });
}
int vie_debug_pencil4_phases(unsigned long long* out8, int reset) {
  return guard([&] { vie::pencil4_phase_read(out8, reset != 0); });
}
#endif

}  // extern "C"

namespace {
// hosvd + transform_factors of a DEVICE spatial tensor dt (decomp.hpp:160-176,
// operator.hpp:76-90): per mode, the Gram of the unfolding on the device and its
// Hermitian Jacobi eigendecomposition on the host give a first basis U0; the unfolding
// is then projected, B = U0^H M (device mode product), and the eigendecomposition of
// B B^H (rows of B carry the singular values, so its entries are accurate relative to
// sigma_i sigma_j, not sigma_max^2) refines U = U0 V and sigma_k = sqrt(lambda_k): the
// squared-condition loss of the one-pass Gram method is removed and small singular
// values resolve down to ~eps sigma_max, as the reference's QR + JacobiSVD
// (decomp.hpp:40-70).  Ranks by truncation_rank (decomp.hpp:72-103).
struct HosvdResult {
  std::vector<cd> U[3];  // n_q x r_q spatial factors (host)
  int64_t rk[3];
  std::vector<cd> core;       // r1 r2 r3 (host)
  const double2* core_dev;    // the same on the device (owned by the caller's pool)
};

void hosvd_dev(vie_ctx ctx, const int64_t dims[3], const double2* dt, const int sign[3], double tol, int rule,
               int passes, DevPool& dev, HosvdResult& h) {
  std::vector<cd>* U = h.U;
  int64_t* rk = h.rk;
  for (int q = 0; q < 3; ++q) {
    if (dims[q] < 1) throw Invalid("hosvd: degenerate tensor dimensions");
    if (sign[q] != 1 && sign[q] != -1) throw Invalid("tucker_compress: sign must be +-1");
  }
  if (!(tol >= 0.0)) throw Invalid("truncated_svd: tol must be >= 0");
  if (rule != VIE_RULE_SIGMA_MAX && rule != VIE_RULE_ENERGY) throw Invalid("tucker_compress: bad rule");
  if (dims[0] > 4096 || dims[1] > 4096 || dims[2] > 4096) throw Invalid("tucker_compress: dims too large");
  cudaStream_t st = ctx->stream;
  for (int q = 0; q < 3; ++q) {
    const int n = static_cast<int>(dims[q]);
    double2* dG = dev.alloc<double2>(static_cast<size_t>(n) * n);
    auto gram_eig = [&](const double2* t, std::vector<double>& lam, std::vector<cd>& V, bool relative) {
      vie::launch_gram(t, dims, q + 1, dG, st);
      std::vector<cd> G(static_cast<size_t>(n) * n);
      VIE_CUDA_CHECK(cudaMemcpyAsync(G.data(), dG, sizeof(double2) * G.size(), cudaMemcpyDeviceToHost, st));
      VIE_CUDA_CHECK(cudaStreamSynchronize(st));
      herm_eig_jacobi(G, n, lam, V, relative);
    };
    std::vector<double> lam;
    std::vector<cd> V0;
    gram_eig(dt, lam, V0, passes <= 1);  // first pass: absolute threshold (a basis to refine)
    std::vector<cd> Ufull = V0;  // n x n
    for (int pass = 1; pass < passes; ++pass) {
      // B = Ufull^H x_q t, then the eigendecomposition of B B^H (rotation V), Ufull <- Ufull V
      double2* dU = dev.alloc<double2>(static_cast<size_t>(n) * n);
      VIE_CUDA_CHECK(cudaMemcpyAsync(dU, Ufull.data(), sizeof(double2) * Ufull.size(), cudaMemcpyHostToDevice, st));
      double2* dB = dev.alloc<double2>(static_cast<size_t>(dims[0] * dims[1] * dims[2]));
      vie::launch_mode_product_h(dt, dims, q + 1, dU, n, dB, st);
      std::vector<cd> Vr;
      gram_eig(dB, lam, Vr, true);
      std::vector<cd> Un(static_cast<size_t>(n) * n, cd(0.0));
      for (int c = 0; c < n; ++c)
        for (int k = 0; k < n; ++k) {
          const cd v = Vr[static_cast<size_t>(k) + static_cast<size_t>(n) * c];
          if (v == cd(0.0)) continue;
          for (int i = 0; i < n; ++i)
            Un[static_cast<size_t>(i) + static_cast<size_t>(n) * c] += Ufull[static_cast<size_t>(i) + static_cast<size_t>(n) * k] * v;
        }
      Ufull.swap(Un);
    }
    std::vector<double> sig(static_cast<size_t>(n));
    for (int k = 0; k < n; ++k) sig[static_cast<size_t>(k)] = std::sqrt(std::max(lam[static_cast<size_t>(k)], 0.0));
    int64_t r = truncation_rank_host(sig, tol, rule);
    const bool zero = r == 0;
    if (zero) r = 1;  // rank-0 form == zero spectrum; keep one (zeroed) column
    rk[q] = r;
    U[q].assign(static_cast<size_t>(n * r), cd(0.0));
    for (int64_t c = 0; c < r; ++c)
      for (int i = 0; i < n; ++i)
        U[q][static_cast<size_t>(i + n * c)] = zero ? cd(0.0) : Ufull[static_cast<size_t>(i + n * c)];
    if (sign[q] < 0) {  // odd axis: the offset-0 row is zero (components.hpp:46-50)
      double nrm = 0.0, row0 = 0.0;
      for (int64_t c = 0; c < r; ++c) {
        row0 += std::norm(U[q][static_cast<size_t>(n * c)]);
        for (int i = 0; i < n; ++i) nrm += std::norm(U[q][static_cast<size_t>(i + n * c)]);
      }
      if (row0 > 1e-20 * std::max(nrm, 1e-300))
        throw Invalid("tucker_compress: odd-parity component has a nonzero offset-0 plane");
      for (int64_t c = 0; c < r; ++c) U[q][static_cast<size_t>(n * c)] = 0.0;
    }
  }
  // core = t x1 U1^H x2 U2^H x3 U3^H (decomp.hpp:171-174), on the device
  int64_t d[3] = {dims[0], dims[1], dims[2]};
  const double2* cur = dt;
  for (int q = 0; q < 3; ++q) {
    double2* dU = dev.alloc<double2>(U[q].size());
    VIE_CUDA_CHECK(cudaMemcpyAsync(dU, U[q].data(), sizeof(double2) * U[q].size(), cudaMemcpyHostToDevice, st));
    int64_t od[3] = {d[0], d[1], d[2]};
    od[q] = rk[q];
    double2* nxt = dev.alloc<double2>(static_cast<size_t>(od[0] * od[1] * od[2]));
    vie::launch_mode_product_h(cur, d, q + 1, dU, static_cast<int>(rk[q]), nxt, st);
    cur = nxt;
    d[0] = od[0];
    d[1] = od[1];
    d[2] = od[2];
  }
  h.core.assign(static_cast<size_t>(rk[0] * rk[1] * rk[2]), cd(0.0));
  VIE_CUDA_CHECK(cudaMemcpyAsync(h.core.data(), cur, sizeof(double2) * h.core.size(), cudaMemcpyDeviceToHost, st));
  VIE_CUDA_CHECK(cudaStreamSynchronize(st));
  h.core_dev = cur;
}

void tucker_compress_dev(vie_ctx ctx, const int64_t dims[3], const double2* dt, const int sign[3], double tol,
                         int rule, vie_tucker* out, int64_t ranks_out[3], int passes) {
  DevPool dev;
  HosvdResult h;
  hosvd_dev(ctx, dims, dt, sign, tol, rule, passes, dev, h);
  const int64_t* rk = h.rk;
  const std::vector<cd>* U = h.U;
  const std::vector<cd>& core = h.core;
  const int rc = vie_tucker_from_factors(ctx, dims, rk, reinterpret_cast<const double*>(core.data()),
                                         reinterpret_cast<const double*>(U[0].data()),
                                         reinterpret_cast<const double*>(U[1].data()),
                                         reinterpret_cast<const double*>(U[2].data()), sign, 0, out);
  if (rc != VIE_OK) throw Invalid(g_err);
  (*out)->rule = rule;
  (*out)->tol = tol;
  if (ranks_out)
    for (int q = 0; q < 3; ++q) ranks_out[q] = rk[q];
}

int hosvd_passes() { return env_int("VIE_HOSVD_PASSES", 2); }

// tucker_cp (decomp.hpp:336-373) of a DEVICE tensor: the device HOSVD above, cp_als on its core
// (cp_als.cu), merged factors W_q = U_q V_q; the three relative errors of TuckerCpResult
// (hosvd, core CP, achieved) from device residual norms.  out (optional): the device form of
// transform_factors(TuckerCPForm) (vie_tucker_from_cp); w (optional): the spatial W_q on the host.
void tucker_cp_dev(vie_ctx ctx, const int64_t dims[3], const double2* dt, const int sign[3], double tol, int rule,
                   int cp_iters, int64_t cp_rank, double stall_tol, vie_tucker* out, int64_t* rank_out,
                   double* const w[3], int64_t w_cap, double errs[3], double* trace, int trace_cap, int* ntrace) {
  if (cp_iters < 1) throw Invalid("cp_als: max_iters must be >= 1");
  DevPool dev;
  HosvdResult h;
  hosvd_dev(ctx, dims, dt, sign, tol, rule, hosvd_passes(), dev, h);
  const int64_t r = cp_rank >= 0 ? cp_rank : std::min({h.rk[0], h.rk[1], h.rk[2]});
  if (rank_out) *rank_out = r;
  if (w && r > w_cap) throw Invalid("tucker_cp: factor buffers hold fewer columns than the CP rank");
  const vie::CpAlsHost cp =
      vie::cp_als_host(reinterpret_cast<const double2*>(h.core.data()), h.rk, r, cp_iters, stall_tol, 0x5eedull);
  std::vector<cd> W[3];
  for (int q = 0; q < 3; ++q) {
    const int64_t n = dims[q], rq = h.rk[q];
    W[q].assign(static_cast<size_t>(n * r), cd(0.0));
    for (int64_t l = 0; l < r; ++l)
      for (int64_t k = 0; k < rq; ++k) {
        const double2 v = cp.f[q][static_cast<size_t>(k + rq * l)];
        const cd vk(v.x, v.y);
        if (vk == cd(0.0)) continue;
        for (int64_t i = 0; i < n; ++i)
          W[q][static_cast<size_t>(i + n * l)] += h.U[q][static_cast<size_t>(i + n * k)] * vk;
      }
  }
  cudaStream_t st = ctx->stream;
  const int64_t nv = dims[0] * dims[1] * dims[2];
  double* acc = dev.alloc<double>(3);
  VIE_CUDA_CHECK(cudaMemsetAsync(acc, 0, 3 * sizeof(double), st));
  vie::launch_diff_norm2(dt, nullptr, nv, acc, st);
  {  // Tucker reconstruction core x1 U1 x2 U2 x3 U3 (mode products with U_q^H as the "U^H" operand)
    int64_t d[3] = {h.rk[0], h.rk[1], h.rk[2]};
    const double2* cur = h.core_dev;
    for (int q = 0; q < 3; ++q) {
      const int64_t n = dims[q], rq = h.rk[q];
      std::vector<cd> uh(static_cast<size_t>(rq * n));
      for (int64_t i = 0; i < n; ++i)
        for (int64_t k = 0; k < rq; ++k)
          uh[static_cast<size_t>(k + rq * i)] = std::conj(h.U[q][static_cast<size_t>(i + n * k)]);
      double2* du = dev.alloc<double2>(uh.size());
      VIE_CUDA_CHECK(cudaMemcpyAsync(du, uh.data(), sizeof(double2) * uh.size(), cudaMemcpyHostToDevice, st));
      int64_t od[3] = {d[0], d[1], d[2]};
      od[q] = n;
      double2* nxt = dev.alloc<double2>(static_cast<size_t>(od[0] * od[1] * od[2]));
      vie::launch_mode_product_h(cur, d, q + 1, du, static_cast<int>(n), nxt, st);
      VIE_CUDA_CHECK(cudaStreamSynchronize(st));  // uh leaves scope
      cur = nxt;
      d[0] = od[0];
      d[1] = od[1];
      d[2] = od[2];
    }
    vie::launch_diff_norm2(dt, cur, nv, acc + 1, st);
  }
  double2* dw[3];
  for (int q = 0; q < 3; ++q) {
    dw[q] = dev.alloc<double2>(std::max<size_t>(W[q].size(), 1));
    if (!W[q].empty())
      VIE_CUDA_CHECK(cudaMemcpyAsync(dw[q], W[q].data(), sizeof(double2) * W[q].size(), cudaMemcpyHostToDevice, st));
  }
  vie::launch_cp_residual2(dt, dims, dw[0], dw[1], dw[2], static_cast<int>(r), acc + 2, st);
  double hacc[3];
  VIE_CUDA_CHECK(cudaMemcpyAsync(hacc, acc, sizeof(hacc), cudaMemcpyDeviceToHost, st));
  VIE_CUDA_CHECK(cudaStreamSynchronize(st));
  const double tn = std::sqrt(hacc[0]);
  if (errs) {
    errs[0] = tn > 0 ? std::sqrt(hacc[1]) / tn : 0.0;
    errs[1] = cp.trace.empty() ? 0.0 : cp.trace.back();
    errs[2] = tn > 0 ? std::sqrt(hacc[2]) / tn : 0.0;
  }
  if (ntrace) *ntrace = static_cast<int>(cp.trace.size());
  if (trace)
    for (int i = 0; i < std::min(trace_cap, static_cast<int>(cp.trace.size())); ++i)
      trace[i] = cp.trace[static_cast<size_t>(i)];
  if (w)
    for (int q = 0; q < 3; ++q)
      if (w[q]) std::copy(W[q].begin(), W[q].end(), reinterpret_cast<cd*>(w[q]));
  if (out) {
    const int rc = vie_tucker_from_cp(ctx, dims, r, reinterpret_cast<const double*>(W[0].data()),
                                      reinterpret_cast<const double*>(W[1].data()),
                                      reinterpret_cast<const double*>(W[2].data()), sign, 0, out);
    if (rc != VIE_OK) throw Invalid(g_err);
    (*out)->rule = rule;
    (*out)->tol = tol;
  }
}
}  // namespace

extern "C" {

int vie_tucker_compress(vie_ctx ctx, const int64_t dims[3], const double* t_host, const int sign[3], double tol,
                        int rule, vie_tucker* out, int64_t ranks_out[3]) {
  return guard([&] {
    if (!ctx || !dims || !t_host || !sign || !out) throw Invalid("tucker_compress: null argument");
    for (int q = 0; q < 3; ++q)
      if (dims[q] < 1) throw Invalid("hosvd: degenerate tensor dimensions");
    VIE_CUDA_CHECK(cudaSetDevice(ctx->device));
    const int64_t nv = dims[0] * dims[1] * dims[2];
    check_cplx_finite_host(t_host, static_cast<size_t>(nv), "tucker_compress: tensor");
    DevPool dev;
    double2* dt = dev.alloc<double2>(static_cast<size_t>(nv));
    copy_sync(dt, t_host, sizeof(double2) * nv, ctx->stream);
    tucker_compress_dev(ctx, dims, dt, sign, tol, rule, out, ranks_out, hosvd_passes());
  });
}

int vie_tucker_compress_device(vie_ctx ctx, const int64_t dims[3], const double* t_dev, const int sign[3],
                               double tol, int rule, vie_tucker* out, int64_t ranks_out[3], void* stream) {
  return guard([&] {
    if (!ctx || !dims || !t_dev || !sign || !out) throw Invalid("tucker_compress: null argument");
    VIE_CUDA_CHECK(cudaSetDevice(ctx->device));
    cudaEvent_t ev = nullptr;
    VIE_CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    StreamJoin sj(ctx->stream, static_cast<cudaStream_t>(stream), ev);
    try {
      tucker_compress_dev(ctx, dims, reinterpret_cast<const double2*>(t_dev), sign, tol, rule, out, ranks_out,
                          hosvd_passes());
    } catch (...) {
      cudaEventDestroy(ev);
      throw;
    }
    sj.done();
    VIE_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    cudaEventDestroy(ev);
  });
}

int vie_tucker_cp(vie_ctx ctx, const int64_t dims[3], const double* t, int t_on_device, const int sign[3],
                  double tol, int rule, int cp_iters, int64_t cp_rank, double stall_tol, vie_tucker* out,
                  int64_t* rank_out, double* w1, double* w2, double* w3, int64_t w_cap, double errs[3], double* trace,
                  int trace_cap, int* ntrace, void* stream) {
  return guard([&] {
    if (!ctx || !dims || !t || !sign) throw Invalid("tucker_cp: null argument");
    for (int q = 0; q < 3; ++q)
      if (dims[q] < 1) throw Invalid("hosvd: degenerate tensor dimensions");
    VIE_CUDA_CHECK(cudaSetDevice(ctx->device));
    double* const w[3] = {w1, w2, w3};
    const bool want_w = w1 || w2 || w3;
    if (!t_on_device) {
      const int64_t nv = dims[0] * dims[1] * dims[2];
      check_cplx_finite_host(t, static_cast<size_t>(nv), "tucker_cp: tensor");
      DevPool dev;
      double2* dt = dev.alloc<double2>(static_cast<size_t>(nv));
      copy_sync(dt, t, sizeof(double2) * nv, ctx->stream);
      tucker_cp_dev(ctx, dims, dt, sign, tol, rule, cp_iters, cp_rank, stall_tol, out, rank_out,
                    want_w ? w : nullptr, w_cap, errs, trace, trace_cap, ntrace);
      return;
    }
    cudaEvent_t ev = nullptr;
    VIE_CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    StreamJoin sj(ctx->stream, static_cast<cudaStream_t>(stream), ev);
    try {
      tucker_cp_dev(ctx, dims, reinterpret_cast<const double2*>(t), sign, tol, rule, cp_iters, cp_rank, stall_tol,
                    out, rank_out, want_w ? w : nullptr, w_cap, errs, trace, trace_cap, ntrace);
    } catch (...) {
      cudaEventDestroy(ev);
      throw;
    }
    sj.done();
    VIE_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    cudaEventDestroy(ev);
  });
}

int vie_cp_als(const int64_t dims[3], const double* t_host, int64_t r, int max_iters, double stall_tol,
               uint64_t seed, double* f1, double* f2, double* f3, double* trace, int trace_cap, int* ntrace,
               int flags[2]) {
  return guard([&] {
    if (!dims || !t_host) throw Invalid("cp_als: null argument");
    for (int q = 0; q < 3; ++q)
      if (dims[q] < 0) throw Invalid("cp_als: negative dims");
    const vie::CpAlsHost o =
        vie::cp_als_host(reinterpret_cast<const double2*>(t_host), dims, r, max_iters, stall_tol, seed);
    double* fs[3] = {f1, f2, f3};
    for (int q = 0; q < 3; ++q)
      if (fs[q]) std::copy(o.f[q].begin(), o.f[q].end(), reinterpret_cast<double2*>(fs[q]));
    if (ntrace) *ntrace = static_cast<int>(o.trace.size());
    if (trace)
      for (int i = 0; i < std::min(trace_cap, static_cast<int>(o.trace.size())); ++i)
        trace[i] = o.trace[static_cast<size_t>(i)];
    if (flags) {
      flags[0] = o.converged;
      flags[1] = o.ill_posed;
    }
  });
}

// ---- Green's-tensor assembly (assembly.hpp:159-246) ----
namespace {
vie::AssemblyDesc asm_desc(const int64_t dims[3], const double res[3], double k0, int kind, int q, int qp,
                           const vie_quadrature* quad) {
  vie::AssemblyDesc ad{};
  for (int a = 0; a < 3; ++a) {
    if (dims[a] < 1) throw Invalid("VoxelGrid: dims must be >= 1");
    if (!(res[a] > 0.0)) throw Invalid("VoxelGrid: resolution must be > 0");
    ad.dims[a] = dims[a];
    ad.res[a] = res[a];
  }
  if (kind < 0 || kind > 2) throw Invalid("assemble_defining_tensor: kind must be N, K or scalar g");
  if (q < 0 || q > 2 || qp < 0 || qp > 2) throw Invalid("assemble_defining_tensor: axes must be 0..2");
  if (!std::isfinite(k0) || k0 < 0.0) throw Invalid("assemble_defining_tensor: k0 must be finite and >= 0");
  ad.k0 = k0;
  ad.op = kind;
  ad.q = q;
  ad.qp = qp;
  const vie_quadrature dflt = {5, 10, 1, 12, 6};  // QuadratureSpec defaults (assembly.hpp:24-29)
  const vie_quadrature& qs = quad ? *quad : dflt;
  if (qs.far_points_per_axis < 1 || qs.near_points_per_axis < 1 || qs.surface_points_per_axis < 1 ||
      qs.volume_points_per_axis < 1)
    throw Invalid("QuadratureSpec: quadrature budget of zero");
  if (qs.near_radius < 1) throw Invalid("QuadratureSpec: near_radius must be >= 1");
  ad.far = qs.far_points_per_axis;
  ad.near = qs.near_points_per_axis;
  ad.near_radius = qs.near_radius;
  ad.surface = qs.surface_points_per_axis;
  ad.volume = qs.volume_points_per_axis;
  return ad;
}
}  // namespace

int vie_assemble(vie_ctx ctx, const int64_t dims[3], const double resolution[3], double k0, int kind, int row_axis,
                 int col_axis, int basis, const vie_quadrature* quad, double* t, void* stream) {
  return guard([&] {
    if (!ctx || !dims || !resolution || !t) throw Invalid("assemble_defining_tensor: null argument");
    if (basis != VIE_BASIS_PWC)
      throw Invalid(
          "assemble_defining_tensor: PWL Galerkin assembly (60 N / 30 K unique entries) is not supported; use PWC");
    const vie::AssemblyDesc ad = asm_desc(dims, resolution, k0, kind, row_axis, col_axis, quad);
    VIE_CUDA_CHECK(cudaSetDevice(ctx->device));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    DevPool dev;
    double2* self = dev.alloc<double2>(1);
    double* rules = dev.alloc<double>(2 * vie::kAsmRuleElems + 4);
    vie::launch_assemble(ad, reinterpret_cast<double2*>(t), self, rules, st, nullptr, nullptr);
    VIE_CUDA_CHECK(cudaStreamSynchronize(st));  // scratch is freed on return
  });
}

int vie_correlation_entry(vie_ctx ctx, int op, double k, int q, int qp, const double d[3], const double delta[3],
                          int points, int duffy, double* out_host) {
  return guard([&] {
    if (!ctx || !d || !delta || !out_host) throw Invalid("correlation_entry: null argument");
    if (op < 0 || op > 3 || points < 1 || points > 31) throw Invalid("correlation_entry: bad kernel or budget");
    VIE_CUDA_CHECK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    DevPool dev;
    double* rules = dev.alloc<double>(2 * vie::kAsmRuleElems + 4);
    double2* o = dev.alloc<double2>(1);
    vie::launch_correlation_entry(op, k, q, qp, d, delta, points, duffy, rules, o, st);
    VIE_CUDA_CHECK(cudaMemcpyAsync(out_host, o, sizeof(double2), cudaMemcpyDeviceToHost, st));
    VIE_CUDA_CHECK(cudaStreamSynchronize(st));
  });
}

int vie_self_static_term(vie_ctx ctx, const double delta[3], const vie_quadrature* quad, double dyad_diag[3],
                         double* gram, double* error_indicator, int* converged) {
  return guard([&] {
    if (!ctx || !delta) throw Invalid("self_static_term: null argument");
    const int64_t one[3] = {1, 1, 1};
    vie::AssemblyDesc ad = asm_desc(one, delta, 0.0, 0, 0, 0, quad);
    for (int a = 0; a < 3; ++a) ad.res[a] = delta[a];
    VIE_CUDA_CHECK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    DevPool dev;
    double* rules = dev.alloc<double>(2 * vie::kAsmRuleElems + 4);
    double* out = dev.alloc<double>(4);
    // the kernel works in x-edge units: rescale the dyad back (it scales as the volume)
    vie::launch_assemble(ad, nullptr, nullptr, rules, st, out, out + 3);
    double h[4];
    VIE_CUDA_CHECK(cudaMemcpyAsync(h, out, sizeof(h), cudaMemcpyDeviceToHost, st));
    VIE_CUDA_CHECK(cudaStreamSynchronize(st));
    const double s3 = delta[0] * delta[0] * delta[0];
    if (dyad_diag)
      for (int a = 0; a < 3; ++a) dyad_diag[a] = h[a] * s3;
    const double g = delta[0] * delta[1] * delta[2];
    if (gram) *gram = g;
    if (error_indicator) *error_indicator = h[3];
    if (converged) *converged = h[3] < 1e-7 ? 1 : 0;
  });
}

}  // extern "C"

// ---- scene stages (solve_scene, solver.hpp:148-285) ----
namespace {

// VoxelGrid / DielectricMap / PlaneWave (grid.hpp:24-100) -> device descriptor;
// throws Invalid where the reference constructors throw.
vie::SceneDev make_scene(const vie_scene* sc, int quad) {
  if (!sc) throw Invalid("scene: null argument");
  vie::SceneDev d{};
  for (int a = 0; a < 3; ++a) {
    if (sc->dims[a] < 1) throw Invalid("VoxelGrid: dims must be >= 1");
    if (!(sc->resolution[a] > 0.0)) throw Invalid("VoxelGrid: resolution must be > 0");
    d.n[a] = sc->dims[a];
    d.res[a] = sc->resolution[a];
    d.org[a] = sc->origin[a];
  }
  const double pn = std::sqrt(sc->polarization[0] * sc->polarization[0] + sc->polarization[1] * sc->polarization[1] +
                              sc->polarization[2] * sc->polarization[2]);
  const double dn = std::sqrt(sc->direction[0] * sc->direction[0] + sc->direction[1] * sc->direction[1] +
                              sc->direction[2] * sc->direction[2]);
  if (!(pn > 0.0) || !(dn > 0.0)) throw Invalid("PlaneWave: zero polarization or direction");
  for (int a = 0; a < 3; ++a) {
    d.pol[a] = sc->polarization[a] / pn;
    d.dir[a] = sc->direction[a] / dn;
  }
  if (std::abs(d.pol[0] * d.dir[0] + d.pol[1] * d.dir[1] + d.pol[2] * d.dir[2]) > 1e-12)
    throw Invalid("PlaneWave: polarization must be orthogonal to direction");
  const double pi = 3.141592653589793238462643383279502884;
  const double c0 = 299792458.0;
  d.omega = 2.0 * pi * sc->frequency;                        // grid.hpp:62
  d.k0 = d.omega / c0;                                       // grid.hpp:63
  d.ce = make_double2(0.0, d.omega * vie::kEpsilon0);        // grid.hpp:64
  d.amp = sc->amplitude;
  d.hdir[0] = d.dir[1] * d.pol[2] - d.dir[2] * d.pol[1];     // direction.cross(polarization)
  d.hdir[1] = d.dir[2] * d.pol[0] - d.dir[0] * d.pol[2];
  d.hdir[2] = d.dir[0] * d.pol[1] - d.dir[1] * d.pol[0];
  d.hamp = sc->amplitude / std::sqrt(vie::kMu0 / vie::kEpsilon0);  // amplitude / eta0
  if (quad < 1) throw Invalid("build_rhs: bad quadrature order");
  if (quad > vie::kMaxQuad) throw Invalid("build_rhs: at most 8 quadrature points per axis");
  d.quad = quad;
  // Gauss-Legendre on [0, 1]: Newton on the Legendre roots (quadrature.hpp:23-52)
  const int m = (quad + 1) / 2;
  for (int i = 0; i < m; ++i) {
    double x = std::cos(pi * (i + 0.75) / (quad + 0.5));
    double deriv = 0.0;
    for (int iter = 0; iter < 100; ++iter) {
      double p1 = 1.0, p2 = 0.0;
      for (int k = 0; k < quad; ++k) {
        const double p3 = p2;
        p2 = p1;
        p1 = ((2.0 * k + 1.0) * x * p2 - k * p3) / (k + 1.0);
      }
      deriv = quad * (x * p1 - p2) / (x * x - 1.0);
      const double dx = p1 / deriv;
      x -= dx;
      if (std::abs(dx) < 1e-15) break;
    }
    const double w = 1.0 / ((1.0 - x * x) * deriv * deriv);
    d.qn[i] = 0.5 * (1.0 - x);
    d.qw[i] = w;
    d.qn[quad - 1 - i] = 0.5 * (1.0 + x);
    d.qw[quad - 1 - i] = w;
  }
  return d;
}

// ctx may be NULL for the scene stages: the caller's current device, and the
// given stream (NULL = the legacy default stream).
cudaStream_t ctx_stream(vie_ctx ctx, void* stream) {
  if (ctx) VIE_CUDA_CHECK(cudaSetDevice(ctx->device));
  return stream ? static_cast<cudaStream_t>(stream) : (ctx ? ctx->stream : cudaStreamLegacy);
}

}  // namespace

extern "C" {

int vie_build_rhs(vie_ctx ctx, const vie_scene* scene, const double* eps_r, int quad_points_per_axis, double* rhs,
                  void* stream) {
  return guard([&] {
    if (!eps_r || !rhs) throw Invalid("build_rhs: null argument");
    const vie::SceneDev sc = make_scene(scene, quad_points_per_axis);
    vie::launch_build_rhs(sc, reinterpret_cast<const double2*>(eps_r), reinterpret_cast<double2*>(rhs),
                          ctx_stream(ctx, stream));
  });
}

int vie_recover_fields(vie_ctx ctx, const vie_scene* scene, const double* eps_r, const double* j, vie_op op_k,
                       double* e, double* h, void* stream) {
  return guard([&] {
    if (!eps_r || !j || !e) throw Invalid("recover_fields: null argument");
    const vie::SceneDev sc = make_scene(scene, 1);
    if (op_k) {
      if (!h) throw Invalid("recover_fields: h buffer needed with the K operator");
      if (op_k->kind != VIE_KIND_K) throw Invalid("recover_fields: op_k must be a K operator");
      if (op_k->g.S != 3) throw Invalid("recover_fields: PWC fields only (grid.hpp:114-115)");
      if (op_k->g.n1 != sc.n[0] || op_k->g.n2 != sc.n[1] || op_k->g.n3 != sc.n[2])
        throw Invalid("apply_operator: dim mismatch");
      if (h == j || h == e) throw Invalid("recover_fields: h must not alias j or e");
    }
    cudaStream_t st = ctx_stream(ctx ? ctx : (op_k ? op_k->ctx : nullptr), stream);
    const double2* eps = reinterpret_cast<const double2*>(eps_r);
    const double2* jd = reinterpret_cast<const double2*>(j);
    vie::launch_recover_e(sc, eps, jd, reinterpret_cast<double2*>(e), st);
    if (op_k) {
      double2* hd = reinterpret_cast<double2*>(h);
      run_matvec(op_k, jd, hd, st, nullptr, 0.0, 0);  // K j (solver.hpp:234)
      vie::launch_add_hinc(sc, 1.0 / (sc.res[0] * sc.res[1] * sc.res[2]), hd, st);
    }
  });
}

int vie_postprocess(vie_ctx ctx, const vie_scene* scene, const double* eps_r, const double* e, const double* h,
                    double* p_abs, double* b1_plus, double* total_absorbed_power_host, void* stream) {
  return guard([&] {
    if (!eps_r || !e || !p_abs) throw Invalid("postprocess: null argument");
    if (h && !b1_plus) throw Invalid("postprocess: b1_plus buffer needed with h");
    const vie::SceneDev sc = make_scene(scene, 1);
    cudaStream_t st = ctx_stream(ctx, stream);
    // partials buffer: owned by the context and allocated once (a pool allocation per call
    // costs milliseconds when the pool trims at the synchronisation below); calls on one
    // context serialise on its lock until their result is read.  Without a context: a
    // per-call allocation, freed on return.
    std::unique_lock<std::mutex> lock;
    DevPool own;
    double* buf = nullptr;
    if (ctx) {
      lock = std::unique_lock<std::mutex>(ctx->post_mu);
      if (!ctx->post_partials) ctx->post_partials = dev_alloc<double>(vie::kRedBlocks + 1);
      buf = ctx->post_partials;
    } else {
      buf = own.alloc<double>(vie::kRedBlocks + 1);
    }
    vie::launch_postprocess(sc, reinterpret_cast<const double2*>(eps_r), reinterpret_cast<const double2*>(e),
                            reinterpret_cast<const double2*>(h), p_abs, h ? b1_plus : nullptr, buf + 1, buf,
                            sc.res[0] * sc.res[1] * sc.res[2], st);
    double total = 0.0;
    VIE_CUDA_CHECK(cudaMemcpyAsync(&total, buf, sizeof(double), cudaMemcpyDeviceToHost, st));
    VIE_CUDA_CHECK(cudaStreamSynchronize(st));
    if (total_absorbed_power_host) *total_absorbed_power_host = total;
  });
}

}  // extern "C"

// ---------------------------------------------------------------- VIET container
// container.hpp:15-159: "VIET", u32 version 1, u8 kind (0 dense, 1 tucker, 2 tucker_cp),
// u8 rule (0 sigma_max, 1 energy), u16 0, f64 tol, u64 dims[3], u64 ranks[3], then complex
// payload as (re, im) f64 pairs -- dense: n1 n2 n3 axis-1 fastest; tucker: U1, U2, U3
// (column-major) then the core; tucker_cp: W1, W2, W3.  Little-endian host (x86-64).
namespace {
constexpr char kVietMagic[4] = {'V', 'I', 'E', 'T'};
constexpr uint32_t kVietVersion = 1;

struct VietHeader {
  int kind = 0, rule = 0;
  double tol = 0.0;
  int64_t dims[3] = {0, 0, 0}, ranks[3] = {0, 0, 0};
};

int64_t viet_payload(const VietHeader& h) {  // complex values
  if (h.kind == 0) return h.dims[0] * h.dims[1] * h.dims[2];
  int64_t n = 0;
  for (int q = 0; q < 3; ++q) n += h.dims[q] * h.ranks[q];
  return h.kind == 1 ? n + h.ranks[0] * h.ranks[1] * h.ranks[2] : n;
}

template <class T>
void put(std::ofstream& os, T v) {
  os.write(reinterpret_cast<const char*>(&v), sizeof(T));
}
template <class T>
T get(std::ifstream& is) {
  T v;
  is.read(reinterpret_cast<char*>(&v), sizeof(T));
  if (!is) throw IoError("container: truncated file");
  return v;
}

void viet_write(const char* path, const VietHeader& h, const std::vector<std::pair<const double2*, int64_t>>& blocks) {
  std::ofstream os(path, std::ios::binary);
  if (!os) throw IoError(std::string("container: cannot open ") + path + " for writing");
  os.write(kVietMagic, 4);
  put<uint32_t>(os, kVietVersion);
  put<uint8_t>(os, static_cast<uint8_t>(h.kind));
  put<uint8_t>(os, static_cast<uint8_t>(h.rule));
  put<uint16_t>(os, 0);
  put<double>(os, h.tol);
  for (int q = 0; q < 3; ++q) put<uint64_t>(os, static_cast<uint64_t>(h.dims[q]));
  for (int q = 0; q < 3; ++q) put<uint64_t>(os, static_cast<uint64_t>(h.ranks[q]));
  for (const auto& b : blocks) os.write(reinterpret_cast<const char*>(b.first), static_cast<std::streamsize>(16 * b.second));
  if (!os) throw IoError(std::string("container: write failed: ") + path);
}

VietHeader viet_header(std::ifstream& is, const char* path) {
  if (!is) throw IoError(std::string("container: cannot open ") + path);
  char magic[4];
  is.read(magic, 4);
  if (!is) throw IoError("container: truncated file");
  if (std::memcmp(magic, kVietMagic, 4) != 0) throw IoError(std::string("container: bad magic in ") + path);
  if (get<uint32_t>(is) != kVietVersion) throw IoError("container: unsupported version");
  VietHeader h;
  h.kind = get<uint8_t>(is);
  h.rule = get<uint8_t>(is);
  get<uint16_t>(is);
  h.tol = get<double>(is);
  for (int q = 0; q < 3; ++q) h.dims[q] = static_cast<int64_t>(get<uint64_t>(is));
  for (int q = 0; q < 3; ++q) h.ranks[q] = static_cast<int64_t>(get<uint64_t>(is));
  if (h.kind < 0 || h.kind > 2) throw IoError("container: unknown form kind");
  return h;
}

std::vector<double2> viet_payload_read(std::ifstream& is, const VietHeader& h) {
  std::vector<double2> p(static_cast<size_t>(viet_payload(h)));
  is.read(reinterpret_cast<char*>(p.data()), static_cast<std::streamsize>(16 * p.size()));
  if (!is) throw IoError("container: truncated file");
  return p;
}
}  // namespace

extern "C" {

int vie_container_info(const char* path, int* kind, int* rule, double* tol, int64_t dims[3], int64_t ranks[3]) {
  return guard([&] {
    if (!path) throw Invalid("container: null path");
    std::ifstream is(path, std::ios::binary);
    const VietHeader h = viet_header(is, path);
    if (kind) *kind = h.kind;
    if (rule) *rule = h.rule;
    if (tol) *tol = h.tol;
    for (int q = 0; q < 3; ++q) {
      if (dims) dims[q] = h.dims[q];
      if (ranks) ranks[q] = h.ranks[q];
    }
  });
}

int vie_container_read(const char* path, double* payload, int64_t capacity) {
  return guard([&] {
    if (!path || !payload) throw Invalid("container: null argument");
    std::ifstream is(path, std::ios::binary);
    const VietHeader h = viet_header(is, path);
    if (viet_payload(h) > capacity) throw Invalid("container: payload larger than the buffer");
    const std::vector<double2> p = viet_payload_read(is, h);
    std::memcpy(payload, p.data(), 16 * p.size());
  });
}

int vie_container_write(const char* path, int kind, int rule, double tol, const int64_t dims[3],
                        const int64_t ranks[3], const double* payload) {
  return guard([&] {
    if (!path || !dims || !payload || (kind != 0 && !ranks)) throw Invalid("container: null argument");
    if (kind < 0 || kind > 2 || rule < 0 || rule > 1) throw Invalid("container: bad kind / rule");
    VietHeader h;
    h.kind = kind;
    h.rule = kind == 1 ? rule : 0;
    h.tol = kind == 1 ? tol : 0.0;
    for (int q = 0; q < 3; ++q) {
      h.dims[q] = dims[q];
      h.ranks[q] = kind == 0 ? 0 : ranks[q];
    }
    viet_write(path, h, {{reinterpret_cast<const double2*>(payload), viet_payload(h)}});
  });
}

int vie_tucker_save(vie_tucker t, const char* path) {
  return guard([&] {
    if (!t || !path) throw Invalid("save_container: null argument");
    if (t->hcore.empty()) throw Invalid("save_container: the form was given in the Fourier domain (no spatial factors)");
    VietHeader h;
    for (int q = 0; q < 3; ++q) h.dims[q] = t->dims[q];
    std::vector<std::pair<const double2*, int64_t>> blocks;
    for (int q = 0; q < 3; ++q) blocks.push_back({t->hu[q].data(), static_cast<int64_t>(t->hu[q].size())});
    if (t->cp_rank > 0) {
      h.kind = 2;
      for (int q = 0; q < 3; ++q) h.ranks[q] = t->cp_rank;
    } else {
      h.kind = 1;
      h.rule = t->rule == VIE_RULE_ENERGY ? 1 : 0;
      h.tol = t->rule < 0 ? 0.0 : t->tol;
      for (int q = 0; q < 3; ++q) h.ranks[q] = t->ranks[q];
      blocks.push_back({t->hcore.data(), static_cast<int64_t>(t->hcore.size())});
    }
    viet_write(path, h, blocks);
  });
}

int vie_tucker_load(vie_ctx ctx, const char* path, const int sign[3], vie_tucker* out) {
  return guard([&] {
    if (!ctx || !path || !sign || !out) throw Invalid("load_container: null argument");
    std::ifstream is(path, std::ios::binary);
    const VietHeader h = viet_header(is, path);
    if (h.kind == 0) throw Invalid("load_container: dense tensor, not a compressed form (vie_container_read)");
    const std::vector<double2> p = viet_payload_read(is, h);
    const double* base = reinterpret_cast<const double*>(p.data());
    const double* u[3];
    int64_t off = 0;
    for (int q = 0; q < 3; ++q) {
      u[q] = base + 2 * off;
      off += h.dims[q] * h.ranks[q];
    }
    int rc;
    if (h.kind == 2) {
      rc = vie_tucker_from_cp(ctx, h.dims, h.ranks[0], u[0], u[1], u[2], sign, 0, out);
    } else {
      rc = vie_tucker_from_factors(ctx, h.dims, h.ranks, base + 2 * off, u[0], u[1], u[2], sign, 0, out);
      if (rc == VIE_OK) {
        (*out)->rule = h.rule == 1 ? VIE_RULE_ENERGY : VIE_RULE_SIGMA_MAX;
        (*out)->tol = h.tol;
      }
    }
    if (rc != VIE_OK) throw Invalid(g_err);
  });
}

}  // extern "C"
