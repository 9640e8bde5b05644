// vie_oracle.cpp -- CPU restatement of the reference hot path.
//
// TEST INFRASTRUCTURE ONLY (see vie_oracle.h).  Never linked by the product.
//
// Reference: /root/reference/proj/include/vie/{tensor,grid,components,fft,
// operator,decomp,solver}.hpp.  Eigen3/FFTW3 are absent here, so the GEMMs,
// the DFT (own Stockham mixed-radix FFT) and the SVD (Householder QR + one-sided
// Jacobi) are restated from their published algorithms.  Parity with the
// reference is pinned at the definition level by the reference's own tests
// (see tests/test_oracle_*.py): dense BTTB expansion vs FFT path, factor
// transform vs dense embedding, adjointness, linearity, GMRES known answers.
#include "vie_oracle.h"

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <functional>
#include <limits>
#include <map>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

using cd = std::complex<double>;
using I64 = int64_t;

thread_local std::string g_err;
int g_threads = 1;

struct invalid : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

template <class F>
void parallel_for(I64 n, F&& fn) {
  const int nt = static_cast<int>(std::min<I64>(std::max(1, g_threads), std::max<I64>(n, 1)));
  if (nt <= 1) {
    for (I64 i = 0; i < n; ++i) fn(i, 0);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      const I64 lo = n * t / nt, hi = n * (t + 1) / nt;
      for (I64 i = lo; i < hi; ++i) fn(i, t);
    });
  for (auto& x : th) x.join();
}

// ---------------------------------------------------------------------------
// DFT service restatement (fft.hpp:22-96): forward e^{-i}, unnormalised;
// inverse e^{+i} divided by N.  Own Stockham autosort mixed-radix FFT.
// ---------------------------------------------------------------------------
struct FftPlan {
  I64 n = 0;
  std::vector<int> radices;
  std::vector<cd> w;  // w[t] = exp(-2 pi i t / n)
};

std::mutex g_plan_mu;
std::map<I64, FftPlan*> g_plans;

const FftPlan& get_plan(I64 n) {
  std::lock_guard<std::mutex> lk(g_plan_mu);
  auto it = g_plans.find(n);
  if (it != g_plans.end()) return *it->second;
  auto* p = new FftPlan;
  p->n = n;
  I64 m = n;
  while (m % 4 == 0) { p->radices.push_back(4); m /= 4; }
  while (m % 2 == 0) { p->radices.push_back(2); m /= 2; }
  for (I64 f = 3; f * f <= m; f += 2)
    while (m % f == 0) { p->radices.push_back(static_cast<int>(f)); m /= f; }
  if (m > 1) p->radices.push_back(static_cast<int>(m));
  p->w.resize(static_cast<size_t>(n));
  const double two_pi = 6.283185307179586476925286766559;
  for (I64 t = 0; t < n; ++t) {
    const double a = -two_pi * static_cast<double>(t) / static_cast<double>(n);
    p->w[static_cast<size_t>(t)] = cd(std::cos(a), std::sin(a));
  }
  g_plans[n] = p;
  return *p;
}

// In-place 1D transform of a contiguous line; `work` holds n + radix scratch.
void fft_line(cd* data, I64 n, bool inverse, std::vector<cd>& work) {
  if (n <= 1) return;
  const FftPlan& P = get_plan(n);
  if (static_cast<I64>(work.size()) < 2 * n + 64) work.resize(static_cast<size_t>(2 * n + 64));
  cd* x = data;
  cd* y = work.data();
  cd* v = work.data() + n;  // radix scratch (max radix <= n)
  std::vector<cd> vbig;
  auto tw = [&](I64 e) {
    const cd c = P.w[static_cast<size_t>(e % n)];
    return inverse ? std::conj(c) : c;
  };
  I64 ns = 1;
  for (int p : P.radices) {
    cd* vv = v;
    if (p > 63) {
      vbig.resize(static_cast<size_t>(2 * p));
      vv = vbig.data();
    }
    const I64 np = n / p;
    const I64 tstep = n / (ns * p);
    for (I64 j = 0; j < np; ++j) {
      const I64 k = j % ns;
      for (int r = 0; r < p; ++r) vv[r] = x[j + r * np];
      if (ns > 1)
        for (int r = 1; r < p; ++r) vv[r] *= tw(static_cast<I64>(r) * k * tstep);
      // radix-p DFT
      if (p == 2) {
        const cd a = vv[0], b = vv[1];
        vv[0] = a + b;
        vv[1] = a - b;
      } else if (p == 4) {
        const cd a0 = vv[0], a1 = vv[1], a2 = vv[2], a3 = vv[3];
        const cd s02 = a0 + a2, d02 = a0 - a2, s13 = a1 + a3, d13 = a1 - a3;
        // -i*d13 for forward, +i*d13 for inverse
        const cd rot = inverse ? cd(-d13.imag(), d13.real()) : cd(d13.imag(), -d13.real());
        vv[0] = s02 + s13;
        vv[1] = d02 + rot;
        vv[2] = s02 - s13;
        vv[3] = d02 - rot;
      } else {
        cd* o = vv + p;
        const I64 wstep = n / p;
        for (int q = 0; q < p; ++q) {
          cd acc = vv[0];
          for (int r = 1; r < p; ++r) acc += vv[r] * tw(static_cast<I64>((r * q) % p) * wstep);
          o[q] = acc;
        }
        for (int q = 0; q < p; ++q) vv[q] = o[q];
      }
      const I64 base = (j / ns) * ns * p + k;
      for (int r = 0; r < p; ++r) y[base + r * ns] = vv[r];
    }
    std::swap(x, y);
    ns *= p;
  }
  if (x != data) std::memcpy(data, x, sizeof(cd) * static_cast<size_t>(n));
}

// 3D transform of a Tensor3 (axis-1 fastest).  fft.hpp:51-71 passes FFTW the
// dims reversed; the transform itself is the plain separable 3D DFT.
void fft3(cd* t, I64 n1, I64 n2, I64 n3, bool inverse) {
  const I64 dims[3] = {n1, n2, n3};
  const I64 strides[3] = {1, n1, n1 * n2};
  for (int ax = 0; ax < 3; ++ax) {
    const I64 n = dims[ax], st = strides[ax];
    if (n <= 1) continue;
    const I64 nlines = n1 * n2 * n3 / n;
    const int nt = std::max(1, std::min<int>(g_threads, static_cast<int>(nlines)));
    std::vector<std::vector<cd>> lines(static_cast<size_t>(nt)), works(static_cast<size_t>(nt));
    parallel_for(nlines, [&](I64 li, int tid) {
      // line index -> base offset
      I64 base;
      if (ax == 0) base = li * n1;
      else if (ax == 1) base = (li % n1) + (li / n1) * n1 * n2;
      else base = li;
      auto& line = lines[static_cast<size_t>(tid)];
      line.resize(static_cast<size_t>(n));
      for (I64 e = 0; e < n; ++e) line[static_cast<size_t>(e)] = t[base + e * st];
      fft_line(line.data(), n, inverse, works[static_cast<size_t>(tid)]);
      for (I64 e = 0; e < n; ++e) t[base + e * st] = line[static_cast<size_t>(e)];
    });
  }
  if (inverse) {  // fft.hpp:36: t.flat() /= t.size()
    const double nn = static_cast<double>(n1 * n2 * n3);
    const I64 tot = n1 * n2 * n3;
    for (I64 i = 0; i < tot; ++i) t[i] /= nn;
  }
}

// ---------------------------------------------------------------------------
// Component tables: components.hpp:46-92 and operator.hpp:205-219 for PWC;
// the PWL generalisation (not in the reference, BASELINE north star) follows
// the same reciprocity/parity rules.
// ---------------------------------------------------------------------------
struct Comp {
  int q, qp, l, lp;
  int par[3];
};
struct Block {
  int t, s, c, dsign;
};

void build_table(int kind, int basis, std::vector<Comp>& comps, std::vector<Block>& blocks) {
  if (kind != 0 && kind != 1) throw invalid("component table: kind must be 0 (N) or 1 (K)");
  if (basis != 0 && basis != 1) throw invalid("component table: basis must be 0 (PWC) or 1 (PWL)");
  const int L = basis == 0 ? 1 : 4;
  comps.clear();
  blocks.clear();
  for (int q = 0; q < 3; ++q)
    for (int qp = (kind == 0 ? q : q + 1); qp < 3; ++qp)
      for (int l = 0; l < L; ++l)
        for (int lp = l; lp < L; ++lp) {
          Comp c{q, qp, l, lp, {1, 1, 1}};
          for (int a = 0; a < 3; ++a) {
            int odd = (l == a + 1) + (lp == a + 1);
            if (kind == 0) odd += (q == a) + (qp == a);
            else odd += (a == 3 - q - qp);
            c.par[a] = (odd % 2) ? -1 : 1;
          }
          comps.push_back(c);
        }
  for (int ci = 0; ci < static_cast<int>(comps.size()); ++ci) {
    const Comp& c = comps[static_cast<size_t>(ci)];
    const int kappa = kind == 0 ? 1 : -1;
    const int sigma = c.par[0] * c.par[1] * c.par[2];
    auto idx = [&](int q, int l) { return q * L + l; };
    const Block cand[4] = {{idx(c.q, c.l), idx(c.qp, c.lp), ci, 1},
                           {idx(c.qp, c.l), idx(c.q, c.lp), ci, kappa},
                           {idx(c.q, c.lp), idx(c.qp, c.l), ci, kappa * sigma},
                           {idx(c.qp, c.lp), idx(c.q, c.l), ci, sigma}};
    std::vector<Block> mine;
    for (const Block& b : cand) {
      bool dup = false;
      for (const Block& m : mine) dup |= (m.t == b.t && m.s == b.s);
      if (!dup) mine.push_back(b);
    }
    blocks.insert(blocks.end(), mine.begin(), mine.end());
  }
}

int ncur(int basis) { return basis == 0 ? 3 : 12; }

// ---------------------------------------------------------------------------
// operator.hpp restatements
// ---------------------------------------------------------------------------
// circulant_embed (operator.hpp:39-59)
void circulant_embed(const cd* t, const I64 d[3], const int sg[3], cd* e) {
  const I64 n1 = d[0], n2 = d[1], n3 = d[2];
  const I64 m1 = 2 * n1, m2 = 2 * n2, m3 = 2 * n3;
  std::fill(e, e + m1 * m2 * m3, cd(0.0));
  for (I64 k = 0; k < m3; ++k) {
    if (k == n3) continue;
    const I64 ok = k < n3 ? k : m3 - k;
    const double sk = k < n3 ? 1.0 : sg[2];
    for (I64 j = 0; j < m2; ++j) {
      if (j == n2) continue;
      const I64 oj = j < n2 ? j : m2 - j;
      const double sj = j < n2 ? 1.0 : sg[1];
      for (I64 i = 0; i < m1; ++i) {
        if (i == n1) continue;
        const I64 oi = i < n1 ? i : m1 - i;
        const double si = i < n1 ? 1.0 : sg[0];
        e[i + m1 * (j + m2 * k)] = si * sj * sk * t[oi + n1 * (oj + n2 * ok)];
      }
    }
  }
}

// embed_column + forward1 per column (operator.hpp:64-90)
void transform_factor(const cd* u, I64 n, I64 r, int sign, cd* out) {
  std::vector<cd> work;
  for (I64 c = 0; c < r; ++c) {
    cd* e = out + 2 * n * c;
    std::fill(e, e + 2 * n, cd(0.0));
    for (I64 m = 0; m < n; ++m) e[m] = u[m + n * c];
    for (I64 m = n + 1; m < 2 * n; ++m) e[m] = static_cast<double>(sign) * u[2 * n - m + n * c];
    fft_line(e, 2 * n, false, work);
  }
}

// decompress_tucker (operator.hpp:224-244): three GEMM stages.
void decompress_tucker(const I64 ed[3], const I64 rk[3], const cd* core, const cd* u1,
                       const cd* u2, const cd* u3, cd* dst) {
  const I64 m1 = ed[0], m2 = ed[1], m3 = ed[2];
  const I64 r1 = rk[0], r2 = rk[1], r3 = rk[2];
  if (r1 == 0 || r2 == 0 || r3 == 0) {
    std::fill(dst, dst + m1 * m2 * m3, cd(0.0));
    return;
  }
  // c1 = U1 * G(r1 x r2r3)
  std::vector<cd> c1(static_cast<size_t>(m1 * r2 * r3));
  parallel_for(r2 * r3, [&](I64 col, int) {
    for (I64 i = 0; i < m1; ++i) {
      cd acc = 0.0;
      for (I64 a = 0; a < r1; ++a) acc += u1[i + m1 * a] * core[a + r1 * col];
      c1[static_cast<size_t>(i + m1 * col)] = acc;
    }
  });
  // c2 slab g = c1_g (m1 x r2) * U2^T
  std::vector<cd> c2(static_cast<size_t>(m1 * m2 * r3));
  parallel_for(r3, [&](I64 g, int) {
    for (I64 j = 0; j < m2; ++j)
      for (I64 i = 0; i < m1; ++i) {
        cd acc = 0.0;
        for (I64 b = 0; b < r2; ++b) acc += c1[static_cast<size_t>(i + m1 * (b + r2 * g))] * u2[j + m2 * b];
        c2[static_cast<size_t>(i + m1 * j + m1 * m2 * g)] = acc;
      }
  });
  // dst (m1m2 x m3) = c2 * U3^T
  const I64 m12 = m1 * m2;
  parallel_for(m3, [&](I64 k, int) {
    cd* col = dst + m12 * k;
    for (I64 p = 0; p < m12; ++p) col[p] = 0.0;
    for (I64 g = 0; g < r3; ++g) {
      const cd w = u3[k + m3 * g];
      const cd* src = c2.data() + m12 * g;
      for (I64 p = 0; p < m12; ++p) col[p] += src[p] * w;
    }
  });
}

// mac_elementwise (operator.hpp:263-265): y += coeff * s * x
void mac_elementwise(cd* y, const cd* s, const cd* x, double coeff, I64 n) {
  parallel_for(std::max<I64>(1, std::min<I64>(n / 65536, 64)), [&](I64 part, int) {
    const I64 parts = std::max<I64>(1, std::min<I64>(n / 65536, 64));
    const I64 lo = n * part / parts, hi = n * (part + 1) / parts;
    for (I64 i = lo; i < hi; ++i) y[i] += coeff * s[i] * x[i];
  });
}

// apply_operator (operator.hpp:273-382) for strategies HosvdDecompress and Dense.
struct TuckerIn {
  const I64* ranks;
  const double* const* cores;
  const double* const* u1s;
  const double* const* u2s;
  const double* const* u3s;
};

// apply_operator (operator.hpp:273-382) as a staged computation: pieces 0..S-1 pad +
// forward3 of current s (:290-297), S..S+NC-1 decompress + mac of component c (:303-364),
// S+NC..2S+NC-1 inverse3 of target t (:367-375).  Running every piece in order is
// apply_operator; the CPU baseline times the pieces of one full matvec.
struct StagedMatvec {
  int kind, basis, S;
  I64 grid[3], ed[3], nv, ne;
  std::vector<Comp> comps;
  std::vector<Block> blocks;
  TuckerIn tk{};
  bool has_tk = false;
  std::vector<const double*> spectra;
  std::vector<std::vector<cd>> xhat, yhat;
  std::vector<cd> buffer, x;

  StagedMatvec(int kind_, int basis_, const I64 g[3], const TuckerIn* t, const double* const* sp, const cd* xin)
      : kind(kind_), basis(basis_) {
    build_table(kind, basis, comps, blocks);
    for (int a = 0; a < 3; ++a)
      if (g[a] < 1) throw invalid("apply_operator: dim mismatch");
    S = ncur(basis);
    for (int a = 0; a < 3; ++a) {
      grid[a] = g[a];
      ed[a] = 2 * g[a];
    }
    nv = grid[0] * grid[1] * grid[2];
    ne = ed[0] * ed[1] * ed[2];
    if (t) {
      tk = *t;
      has_tk = true;
      buffer.resize(static_cast<size_t>(ne));
    } else {
      spectra.assign(sp, sp + comps.size());
    }
    x.assign(xin, xin + S * nv);
    xhat.resize(static_cast<size_t>(S));
    yhat.assign(static_cast<size_t>(S), std::vector<cd>());
  }
  int npieces() const { return 2 * S + static_cast<int>(comps.size()); }
  void piece(int i) {
    const int nc = static_cast<int>(comps.size());
    if (i < S) {
      std::vector<cd>& xh = xhat[static_cast<size_t>(i)];
      xh.assign(static_cast<size_t>(ne), cd(0.0));
      cd* p = xh.data();
      for (I64 k = 0; k < grid[2]; ++k)
        for (I64 j = 0; j < grid[1]; ++j)
          for (I64 ii = 0; ii < grid[0]; ++ii)
            p[ii + ed[0] * (j + ed[1] * k)] = x[static_cast<size_t>(i * nv + ii + grid[0] * (j + grid[1] * k))];
      fft3(p, ed[0], ed[1], ed[2], false);
      return;
    }
    if (i < S + nc) {
      const int ci = i - S;
      const Comp& c = comps[static_cast<size_t>(ci)];
      const double sigma = c.par[0] * c.par[1] * c.par[2];
      const cd* sp;
      if (has_tk) {
        const I64* rk = tk.ranks + 3 * ci;
        decompress_tucker(ed, rk, reinterpret_cast<const cd*>(tk.cores[ci]), reinterpret_cast<const cd*>(tk.u1s[ci]),
                          reinterpret_cast<const cd*>(tk.u2s[ci]), reinterpret_cast<const cd*>(tk.u3s[ci]),
                          buffer.data());
        sp = buffer.data();
      } else {
        if (!spectra[static_cast<size_t>(ci)]) throw invalid("apply_operator: dense spectrum absent");
        sp = reinterpret_cast<const cd*>(spectra[static_cast<size_t>(ci)]);
      }
      for (const Block& bk : blocks)
        if (bk.c == ci) {
          std::vector<cd>& yh = yhat[static_cast<size_t>(bk.t)];
          if (yh.empty()) yh.assign(static_cast<size_t>(ne), cd(0.0));
          if (xhat[static_cast<size_t>(bk.s)].empty()) throw invalid("apply_operator: piece order");
          mac_elementwise(yh.data(), sp, xhat[static_cast<size_t>(bk.s)].data(), bk.dsign * sigma, ne);
        }
      return;
    }
    const int q = i - S - nc;
    std::vector<cd>& yh = yhat[static_cast<size_t>(q)];
    if (yh.empty()) yh.assign(static_cast<size_t>(ne), cd(0.0));
    fft3(yh.data(), ed[0], ed[1], ed[2], true);
  }
  void result(cd* y) const {
    for (int q = 0; q < S; ++q) {
      const cd* p = yhat[static_cast<size_t>(q)].data();
      for (I64 k = 0; k < grid[2]; ++k)
        for (I64 j = 0; j < grid[1]; ++j)
          for (I64 i = 0; i < grid[0]; ++i)
            y[q * nv + i + grid[0] * (j + grid[1] * k)] = p[i + ed[0] * (j + ed[1] * k)];
    }
  }
};

void apply_operator(int kind, int basis, const I64 grid[3], const TuckerIn* tk,
                    const double* const* spectra, const cd* x, cd* y) {
  StagedMatvec mv(kind, basis, grid, tk, spectra, x);
  for (int i = 0; i < mv.npieces(); ++i) mv.piece(i);
  mv.result(y);
}

// apply_system (solver.hpp:183-200), with the PWL Gram weights g_l.
void apply_system(int basis, const I64 grid[3], const TuckerIn& tk, const cd* eps, double inv_v,
                  const cd* x, cd* y) {
  const int S = ncur(basis);
  const I64 nv = grid[0] * grid[1] * grid[2];
  std::vector<cd> nx(static_cast<size_t>(S * nv));
  apply_operator(0, basis, grid, &tk, nullptr, x, nx.data());
  for (int q = 0; q < S; ++q) {
    const int l = basis == 0 ? 0 : q % 4;
    const double g = l == 0 ? 1.0 : 1.0 / 12.0;
    for (I64 m = 0; m < nv; ++m) {
      const cd e = eps[m];
      const cd chi = e - 1.0;
      const cd eg = basis == 0 ? e : e * g;
      y[q * nv + m] = eg * x[q * nv + m] - chi * inv_v * nx[static_cast<size_t>(q * nv + m)];
    }
  }
}

// ---------------------------------------------------------------------------
// GMRES restatement (solver.hpp:34-142)
// ---------------------------------------------------------------------------
using VecFn = std::function<void(const cd*, cd*)>;

double vnorm(const cd* v, I64 n) {
  double s = 0.0;
  for (I64 i = 0; i < n; ++i) s += std::norm(v[i]);
  return std::sqrt(s);
}
cd vdot(const cd* a, const cd* b, I64 n) {  // Eigen a.dot(b) = sum conj(a) b
  cd s = 0.0;
  for (I64 i = 0; i < n; ++i) s += std::conj(a[i]) * b[i];
  return s;
}

struct GmresOut {
  int iterations = 0;
  bool converged = false;
  double final_rel = 0.0;
  std::vector<double> history;
};

GmresOut gmres(const VecFn& apply, const VecFn* precond, I64 n, const cd* rhs, const cd* x0,
               double tol, int inner, int outer, cd* sol) {
  for (I64 i = 0; i < n; ++i)
    if (!std::isfinite(rhs[i].real()) || !std::isfinite(rhs[i].imag()))
      throw invalid("gmres: non-finite right-hand side");
  if (tol < 0 || inner < 1 || outer < 1) throw invalid("gmres: invalid configuration");
  GmresOut res;
  const double bnorm = vnorm(rhs, n);
  for (I64 i = 0; i < n; ++i) sol[i] = x0 ? x0[i] : cd(0.0);
  if (bnorm == 0.0) {
    for (I64 i = 0; i < n; ++i) sol[i] = 0.0;
    res.converged = true;
    res.history.push_back(0.0);
    return res;
  }
  const int m = inner;
  std::vector<cd> basis(static_cast<size_t>(n * (m + 1)));
  std::vector<cd> hess(static_cast<size_t>((m + 1) * m), cd(0.0));
  auto H = [&](int i, int j) -> cd& { return hess[static_cast<size_t>(i + (m + 1) * j)]; };
  std::vector<cd> g(static_cast<size_t>(m + 1)), cs(static_cast<size_t>(m)), sn(static_cast<size_t>(m));
  std::vector<cd> r(static_cast<size_t>(n)), w(static_cast<size_t>(n)), tmp(static_cast<size_t>(n));
  auto col = [&](int j) { return basis.data() + n * j; };

  for (int restart = 0; restart < outer && !res.converged; ++restart) {
    apply(sol, tmp.data());
    for (I64 i = 0; i < n; ++i) r[static_cast<size_t>(i)] = rhs[i] - tmp[static_cast<size_t>(i)];
    const double beta = vnorm(r.data(), n);
    if (beta / bnorm <= tol) {
      res.converged = true;
      break;
    }
    for (I64 i = 0; i < n; ++i) col(0)[i] = r[static_cast<size_t>(i)] / beta;
    std::fill(g.begin(), g.end(), cd(0.0));
    g[0] = beta;
    int j = 0;
    bool breakdown = false;
    for (; j < m; ++j) {
      if (precond) {
        (*precond)(col(j), tmp.data());
        apply(tmp.data(), w.data());
      } else {
        apply(col(j), w.data());
      }
      for (int i = 0; i <= j; ++i) {
        H(i, j) = vdot(col(i), w.data(), n);
        const cd h = H(i, j);
        const cd* v = col(i);
        for (I64 e = 0; e < n; ++e) w[static_cast<size_t>(e)] -= h * v[e];
      }
      const double wnorm = vnorm(w.data(), n);
      H(j + 1, j) = wnorm;
      for (int i = 0; i < j; ++i) {
        const cd t = cs[static_cast<size_t>(i)] * H(i, j) + sn[static_cast<size_t>(i)] * H(i + 1, j);
        H(i + 1, j) = -std::conj(sn[static_cast<size_t>(i)]) * H(i, j) + std::conj(cs[static_cast<size_t>(i)]) * H(i + 1, j);
        H(i, j) = t;
      }
      {
        const cd a = H(j, j), b = H(j + 1, j);
        const double denom = std::sqrt(std::norm(a) + std::norm(b));
        if (denom == 0.0) {
          cs[static_cast<size_t>(j)] = 1.0;
          sn[static_cast<size_t>(j)] = 0.0;
        } else {
          cs[static_cast<size_t>(j)] = std::conj(a) / denom;
          sn[static_cast<size_t>(j)] = std::conj(b) / denom;
        }
        H(j, j) = cs[static_cast<size_t>(j)] * a + sn[static_cast<size_t>(j)] * b;
        H(j + 1, j) = 0.0;
        const cd t = cs[static_cast<size_t>(j)] * g[static_cast<size_t>(j)];
        g[static_cast<size_t>(j + 1)] = -std::conj(sn[static_cast<size_t>(j)]) * g[static_cast<size_t>(j)];
        g[static_cast<size_t>(j)] = t;
      }
      ++res.iterations;
      const double rel = std::abs(g[static_cast<size_t>(j + 1)]) / bnorm;
      res.history.push_back(rel);
      if (rel <= tol) {
        ++j;
        res.converged = true;
        break;
      }
      if (wnorm < 1e-14 * beta) {
        ++j;
        breakdown = true;
        break;
      }
      for (I64 e = 0; e < n; ++e) col(j + 1)[e] = w[static_cast<size_t>(e)] / wnorm;
    }
    std::vector<cd> y(static_cast<size_t>(j), cd(0.0));
    for (int i = j - 1; i >= 0; --i) {
      cd s = g[static_cast<size_t>(i)];
      for (int l = i + 1; l < j; ++l) s -= H(i, l) * y[static_cast<size_t>(l)];
      y[static_cast<size_t>(i)] = s / H(i, i);
    }
    std::vector<cd> update(static_cast<size_t>(n), cd(0.0));
    for (int l = 0; l < j; ++l)
      for (I64 e = 0; e < n; ++e) update[static_cast<size_t>(e)] += col(l)[e] * y[static_cast<size_t>(l)];
    if (precond) {
      (*precond)(update.data(), tmp.data());
      for (I64 e = 0; e < n; ++e) sol[e] += tmp[static_cast<size_t>(e)];
    } else {
      for (I64 e = 0; e < n; ++e) sol[e] += update[static_cast<size_t>(e)];
    }
    if (breakdown && !res.converged) {
      apply(sol, tmp.data());
      for (I64 e = 0; e < n; ++e) r[static_cast<size_t>(e)] = rhs[e] - tmp[static_cast<size_t>(e)];
      const double rel = vnorm(r.data(), n) / bnorm;
      res.converged = rel <= tol;
      if (res.converged) break;
    }
  }
  apply(sol, tmp.data());
  for (I64 e = 0; e < n; ++e) r[static_cast<size_t>(e)] = rhs[e] - tmp[static_cast<size_t>(e)];
  res.final_rel = vnorm(r.data(), n) / bnorm;
  return res;
}

// ---------------------------------------------------------------------------
// decomp.hpp restatement: thin_svd (QR + Jacobi), truncation_rank, hosvd.
// ---------------------------------------------------------------------------
struct Mat {  // column-major complex
  I64 rows = 0, cols = 0;
  std::vector<cd> a;
  Mat() = default;
  Mat(I64 r, I64 c) : rows(r), cols(c), a(static_cast<size_t>(r * c), cd(0.0)) {}
  cd& operator()(I64 i, I64 j) { return a[static_cast<size_t>(i + rows * j)]; }
  cd operator()(I64 i, I64 j) const { return a[static_cast<size_t>(i + rows * j)]; }
};

Mat adjoint(const Mat& m) {
  Mat o(m.cols, m.rows);
  for (I64 j = 0; j < m.cols; ++j)
    for (I64 i = 0; i < m.rows; ++i) o(j, i) = std::conj(m(i, j));
  return o;
}
Mat matmul(const Mat& a, const Mat& b) {
  Mat o(a.rows, b.cols);
  for (I64 j = 0; j < b.cols; ++j)
    for (I64 k = 0; k < a.cols; ++k) {
      const cd bk = b(k, j);
      if (bk == cd(0.0)) continue;
      for (I64 i = 0; i < a.rows; ++i) o(i, j) += a(i, k) * bk;
    }
  return o;
}

// Householder QR (Eigen::HouseholderQR restated): returns thin Q (rows x n) and R (n x n)
void householder_qr(const Mat& m, Mat& q, Mat& r) {
  const I64 rows = m.rows, n = m.cols;
  Mat a = m;
  std::vector<std::vector<cd>> vs;
  std::vector<cd> taus;
  for (I64 k = 0; k < n && k < rows; ++k) {
    double xnorm = 0.0;
    for (I64 i = k; i < rows; ++i) xnorm += std::norm(a(i, k));
    xnorm = std::sqrt(xnorm);
    std::vector<cd> v(static_cast<size_t>(rows - k), cd(0.0));
    cd tau = 0.0;
    if (xnorm > 0.0) {
      const cd x0 = a(k, k);
      const cd alpha = x0 == cd(0.0) ? cd(-xnorm) : -(x0 / std::abs(x0)) * xnorm;
      for (I64 i = k; i < rows; ++i) v[static_cast<size_t>(i - k)] = a(i, k);
      v[0] -= alpha;
      double vn = 0.0;
      for (auto& e : v) vn += std::norm(e);
      if (vn > 0.0) {
        tau = 2.0 / vn;
        for (I64 j = k; j < n; ++j) {
          cd s = 0.0;
          for (I64 i = k; i < rows; ++i) s += std::conj(v[static_cast<size_t>(i - k)]) * a(i, j);
          s *= tau;
          for (I64 i = k; i < rows; ++i) a(i, j) -= s * v[static_cast<size_t>(i - k)];
        }
      }
    }
    vs.push_back(v);
    taus.push_back(tau);
  }
  const I64 kk = std::min(rows, n);
  r = Mat(kk, n);
  for (I64 j = 0; j < n; ++j)
    for (I64 i = 0; i <= std::min(j, kk - 1); ++i) r(i, j) = a(i, j);
  q = Mat(rows, kk);
  for (I64 i = 0; i < kk; ++i) q(i, i) = 1.0;
  for (I64 k = static_cast<I64>(vs.size()) - 1; k >= 0; --k) {
    const auto& v = vs[static_cast<size_t>(k)];
    const cd tau = taus[static_cast<size_t>(k)];
    if (tau == cd(0.0)) continue;
    for (I64 j = 0; j < kk; ++j) {
      cd s = 0.0;
      for (I64 i = k; i < rows; ++i) s += std::conj(v[static_cast<size_t>(i - k)]) * q(i, j);
      s *= tau;
      for (I64 i = k; i < rows; ++i) q(i, j) -= s * v[static_cast<size_t>(i - k)];
    }
  }
}

// One-sided (Hestenes) Jacobi SVD of a rows >= cols matrix: A = U S V^H.
void jacobi_svd_tall(const Mat& m, Mat& u, std::vector<double>& s, Mat& v) {
  const I64 rows = m.rows, n = m.cols;
  Mat a = m;
  v = Mat(n, n);
  for (I64 i = 0; i < n; ++i) v(i, i) = 1.0;
  for (int sweep = 0; sweep < 80; ++sweep) {
    bool rotated = false;
    for (I64 p = 0; p < n - 1; ++p)
      for (I64 qq = p + 1; qq < n; ++qq) {
        double alpha = 0.0, beta = 0.0;
        cd gamma = 0.0;
        for (I64 i = 0; i < rows; ++i) {
          alpha += std::norm(a(i, p));
          beta += std::norm(a(i, qq));
          gamma += std::conj(a(i, p)) * a(i, qq);
        }
        const double ag = std::abs(gamma);
        if (ag == 0.0 || ag <= 1e-15 * std::sqrt(alpha * beta)) continue;
        rotated = true;
        const cd ph = gamma / ag;  // a_q * conj(ph) makes the coupling real
        const double zeta = (beta - alpha) / (2.0 * ag);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
        for (I64 i = 0; i < rows; ++i) {
          const cd ap = a(i, p), aq = a(i, qq) * std::conj(ph);
          a(i, p) = c * ap - sn * aq;
          a(i, qq) = sn * ap + c * aq;
        }
        for (I64 i = 0; i < n; ++i) {
          const cd vp = v(i, p), vq = v(i, qq) * std::conj(ph);
          v(i, p) = c * vp - sn * vq;
          v(i, qq) = sn * vp + c * vq;
        }
      }
    if (!rotated) break;
  }
  std::vector<double> nrm(static_cast<size_t>(n));
  for (I64 j = 0; j < n; ++j) {
    double s2 = 0.0;
    for (I64 i = 0; i < rows; ++i) s2 += std::norm(a(i, j));
    nrm[static_cast<size_t>(j)] = std::sqrt(s2);
  }
  std::vector<I64> order(static_cast<size_t>(n));
  for (I64 j = 0; j < n; ++j) order[static_cast<size_t>(j)] = j;
  std::stable_sort(order.begin(), order.end(),
                   [&](I64 x, I64 y) { return nrm[static_cast<size_t>(x)] > nrm[static_cast<size_t>(y)]; });
  u = Mat(rows, n);
  Mat v2(n, n);
  s.assign(static_cast<size_t>(n), 0.0);
  for (I64 jj = 0; jj < n; ++jj) {
    const I64 j = order[static_cast<size_t>(jj)];
    const double sj = nrm[static_cast<size_t>(j)];
    s[static_cast<size_t>(jj)] = sj;
    for (I64 i = 0; i < rows; ++i) u(i, jj) = sj > 0 ? a(i, j) / sj : cd(0.0);
    for (I64 i = 0; i < n; ++i) v2(i, jj) = v(i, j);
  }
  v = v2;
  // Columns of numerically zero singular values carry no direction after the
  // one-sided sweep; complete U to an orthonormal set (Eigen's JacobiSVD
  // returns orthonormal thin U for rank-deficient input as well).
  const double smax = s.empty() ? 0.0 : s[0];
  for (I64 jj = 0; jj < n; ++jj) {
    if (s[static_cast<size_t>(jj)] > 1e-13 * smax && smax > 0.0) continue;
    for (I64 e = 0; e < rows; ++e) {
      std::vector<cd> w(static_cast<size_t>(rows), cd(0.0));
      w[static_cast<size_t>(e)] = 1.0;
      for (int pass = 0; pass < 2; ++pass)
        for (I64 o = 0; o < n; ++o) {
          if (o == jj) continue;
          if (o > jj && !(s[static_cast<size_t>(o)] > 1e-13 * smax && smax > 0.0)) continue;
          cd d = 0.0;
          for (I64 i = 0; i < rows; ++i) d += std::conj(u(i, o)) * w[static_cast<size_t>(i)];
          for (I64 i = 0; i < rows; ++i) w[static_cast<size_t>(i)] -= d * u(i, o);
        }
      double wn = 0.0;
      for (auto& x : w) wn += std::norm(x);
      wn = std::sqrt(wn);
      if (wn > 0.5) {
        for (I64 i = 0; i < rows; ++i) u(i, jj) = w[static_cast<size_t>(i)] / wn;
        break;
      }
    }
  }
}

void jacobi_svd(const Mat& m, Mat& u, std::vector<double>& s, Mat& v) {
  if (m.rows >= m.cols) {
    jacobi_svd_tall(m, u, s, v);
  } else {
    jacobi_svd_tall(adjoint(m), v, s, u);
  }
}

// thin_svd (decomp.hpp:40-70)
void thin_svd(const Mat& m, Mat& u, std::vector<double>& s, Mat& v) {
  const I64 rows = m.rows, cols = m.cols;
  if (rows == 0 || cols == 0) throw invalid("truncated_svd: empty matrix");
  if (cols > 2 * rows) {
    Mat q, r;
    householder_qr(adjoint(m), q, r);  // m^H = Q R, R rows x rows
    Mat su, sv;
    jacobi_svd(adjoint(r), su, s, sv);
    u = su;
    v = matmul(q, sv);
  } else if (rows > 2 * cols) {
    Mat q, r;
    householder_qr(m, q, r);
    Mat su, sv;
    jacobi_svd(r, su, s, sv);
    u = matmul(q, su);
    v = sv;
  } else {
    jacobi_svd(m, u, s, v);
  }
}

// truncation_rank (decomp.hpp:72-103)
I64 truncation_rank(const std::vector<double>& s, double tol, int rule) {
  const I64 n = static_cast<I64>(s.size());
  if (n == 0) return 0;
  const double smax = s[0];
  if (smax <= 0.0) return 0;
  if (rule == 0) {
    const double threshold = (tol / std::sqrt(3.0)) * smax;
    I64 r = 0;
    for (I64 j = 0; j < n; ++j)
      if (s[static_cast<size_t>(j)] > 0.0 && s[static_cast<size_t>(j)] >= threshold - 1e-14 * smax) r = j + 1;
    return r;
  }
  double total = 0.0;
  for (double x : s) total += x * x;
  const double budget = (tol / std::sqrt(3.0)) * std::sqrt(total);
  const double budget2 = budget * budget;
  double tail = 0.0;
  I64 r = n;
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

// unfold (tensor.hpp:81-98)
Mat unfold(const cd* t, const I64 d[3], int mode) {
  const I64 n1 = d[0], n2 = d[1], n3 = d[2];
  Mat m;
  if (mode == 1) {
    m = Mat(n1, n2 * n3);
    std::copy(t, t + n1 * n2 * n3, m.a.begin());
  } else if (mode == 2) {
    m = Mat(n2, n1 * n3);
    for (I64 k = 0; k < n3; ++k)
      for (I64 j = 0; j < n2; ++j)
        for (I64 i = 0; i < n1; ++i) m(j, i + n1 * k) = t[i + n1 * (j + n2 * k)];
  } else {
    m = Mat(n3, n1 * n2);
    for (I64 k = 0; k < n3; ++k)
      for (I64 p = 0; p < n1 * n2; ++p) m(k, p) = t[p + n1 * n2 * k];
  }
  return m;
}

// n_mode_product (tensor.hpp:128-135)
std::vector<cd> n_mode(const std::vector<cd>& t, I64 d[3], const Mat& u, int mode) {
  Mat un = unfold(t.data(), d, mode);
  Mat prod = matmul(u, un);
  I64 od[3] = {d[0], d[1], d[2]};
  od[mode - 1] = u.rows;
  std::vector<cd> out(static_cast<size_t>(od[0] * od[1] * od[2]));
  const I64 n1 = od[0], n2 = od[1], n3 = od[2];
  for (I64 k = 0; k < n3; ++k)
    for (I64 j = 0; j < n2; ++j)
      for (I64 i = 0; i < n1; ++i) {
        cd v;
        if (mode == 1) v = prod(i, j + n2 * k);
        else if (mode == 2) v = prod(j, i + n1 * k);
        else v = prod(k, i + n1 * j);
        out[static_cast<size_t>(i + n1 * (j + n2 * k))] = v;
      }
  d[0] = od[0];
  d[1] = od[1];
  d[2] = od[2];
  return out;
}

// ---- CP-ALS (decomp.hpp:184-298) and tucker_cp (decomp.hpp:336-373) ----
// khatri_rao (tensor.hpp:146-153): column l = a(:, l) (x) b(:, l), b fastest
Mat khatri_rao(const Mat& a, const Mat& b) {
  Mat o(a.rows * b.rows, a.cols);
  for (I64 l = 0; l < a.cols; ++l)
    for (I64 ia = 0; ia < a.rows; ++ia)
      for (I64 ib = 0; ib < b.rows; ++ib) o(ia * b.rows + ib, l) = a(ia, l) * b(ib, l);
  return o;
}

// cp_reconstruct (tensor.hpp:157-168): mode-1 unfolding = v1 khatri_rao(v3, v2)^T
std::vector<cd> cp_reconstruct(const Mat& v1, const Mat& v2, const Mat& v3) {
  std::vector<cd> t(static_cast<size_t>(v1.rows * v2.rows * v3.rows), cd(0.0));
  if (v1.cols == 0) return t;
  const Mat kr = khatri_rao(v3, v2);
  for (I64 p = 0; p < kr.rows; ++p)
    for (I64 l = 0; l < v1.cols; ++l) {
      const cd z = kr(p, l);
      for (I64 i = 0; i < v1.rows; ++i) t[static_cast<size_t>(i + v1.rows * p)] += v1(i, l) * z;
    }
  return t;
}

double fro(const std::vector<cd>& t) {
  double s = 0.0;
  for (const cd& x : t) s += std::norm(x);
  return std::sqrt(s);
}

// detail::cp_ls_update (decomp.hpp:200-219): v = (a_unf conj(z)) conj(pinv(gram)),
// gram = (b^H b) .* (c^H c), pinv by a Jacobi SVD with relative cutoff 1e-12
Mat cp_ls_update(const Mat& a_unf, const Mat& b, const Mat& c) {
  const Mat z = khatri_rao(c, b);
  Mat zc = z;
  for (cd& x : zc.a) x = std::conj(x);
  const Mat rhs = matmul(a_unf, zc);
  const Mat gb = matmul(adjoint(b), b), gc = matmul(adjoint(c), c);
  Mat gram(gb.rows, gb.cols);
  for (size_t e = 0; e < gram.a.size(); ++e) gram.a[e] = gb.a[e] * gc.a[e];
  Mat u, v;
  std::vector<double> s;
  jacobi_svd(gram, u, s, v);
  const double cutoff = (s.empty() ? 0.0 : s[0]) * 1e-12;
  const I64 r = gram.rows;
  Mat pinv(r, r);  // V diag(sinv) U^H
  for (size_t j = 0; j < s.size(); ++j) {
    if (!(s[j] > cutoff)) continue;
    const double inv = 1.0 / s[j];
    for (I64 col = 0; col < r; ++col) {
      const cd uc = std::conj(u(col, static_cast<I64>(j))) * inv;
      for (I64 row = 0; row < r; ++row) pinv(row, col) += v(row, static_cast<I64>(j)) * uc;
    }
  }
  for (cd& x : pinv.a) x = std::conj(x);
  return matmul(rhs, pinv);
}

// detail::cp_normalize_columns (decomp.hpp:221-230)
void cp_normalize_columns(Mat f[3]) {
  for (I64 l = 0; l < f[0].cols; ++l) {
    double n[3];
    for (int q = 0; q < 3; ++q) {
      double s = 0.0;
      for (I64 i = 0; i < f[q].rows; ++i) s += std::norm(f[q](i, l));
      n[q] = std::sqrt(s);
    }
    const double mag = std::cbrt(n[0] * n[1] * n[2]);
    for (int q = 0; q < 3; ++q)
      if (n[q] > 0)
        for (I64 i = 0; i < f[q].rows; ++i) f[q](i, l) *= mag / n[q];
  }
}

struct CpAlsOut {
  Mat f[3];
  std::vector<double> trace;
  bool converged = false, ill_posed = false;
};

// cp_als (decomp.hpp:237-298): SVD-initialised factors (seeded Gaussian columns beyond
// the unfolding's rank), ALS sweeps over the three modes, column normalisation, relative
// error per sweep, stop when the decrease falls below stall_tol
CpAlsOut cp_als(const cd* t, const I64 d[3], I64 r, int max_iters, double stall_tol, uint64_t seed) {
  if (r < 0) throw invalid("cp_als: rank must be >= 0");
  if (max_iters < 1) throw invalid("cp_als: max_iters must be >= 1");
  CpAlsOut res;
  const std::vector<cd> tv(t, t + d[0] * d[1] * d[2]);
  const double tnorm = fro(tv);
  I64 sorted[3] = {d[0], d[1], d[2]};
  std::sort(sorted, sorted + 3);
  res.ill_posed = r > sorted[0] * sorted[1];
  if (r == 0 || tnorm == 0.0) {
    for (int q = 0; q < 3; ++q) res.f[q] = Mat(d[q], r);
    res.trace.push_back(tnorm == 0.0 ? 0.0 : 1.0);
    res.converged = tnorm == 0.0;
    return res;
  }
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  Mat unf[3];
  for (int q = 0; q < 3; ++q) {
    unf[q] = unfold(t, d, q + 1);
    Mat u, v;
    std::vector<double> s;
    thin_svd(unf[q], u, s, v);
    const I64 have = std::min<I64>(u.cols, r);
    Mat f(d[q], r);
    for (I64 l = 0; l < have; ++l)
      for (I64 i = 0; i < d[q]; ++i) f(i, l) = u(i, l);
    for (I64 l = have; l < r; ++l) {
      for (I64 i = 0; i < d[q]; ++i) f(i, l) = cd(gauss(rng), gauss(rng));
      double nn = 0.0;
      for (I64 i = 0; i < d[q]; ++i) nn += std::norm(f(i, l));
      nn = std::sqrt(nn);
      if (nn > 0)
        for (I64 i = 0; i < d[q]; ++i) f(i, l) /= nn;
    }
    res.f[q] = std::move(f);
  }
  double prev = std::numeric_limits<double>::infinity();
  for (int sweep = 0; sweep < max_iters; ++sweep) {
    res.f[0] = cp_ls_update(unf[0], res.f[1], res.f[2]);
    res.f[1] = cp_ls_update(unf[1], res.f[0], res.f[2]);
    res.f[2] = cp_ls_update(unf[2], res.f[0], res.f[1]);
    cp_normalize_columns(res.f);
    std::vector<cd> rec = cp_reconstruct(res.f[0], res.f[1], res.f[2]);
    for (size_t e = 0; e < rec.size(); ++e) rec[e] -= tv[e];
    const double err = fro(rec) / tnorm;
    res.trace.push_back(err);
    if (prev - err < stall_tol) {
      res.converged = err <= prev + stall_tol;
      break;
    }
    prev = err;
  }
  return res;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
void orc_set_threads(int nthreads) { g_threads = std::max(1, nthreads); }

int orc_random_tensor(int64_t n1, int64_t n2, int64_t n3, uint64_t seed, double* out) {
  return guard([&] {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    cd* o = reinterpret_cast<cd*>(out);
    for (I64 n = 0; n < n1 * n2 * n3; ++n) o[n] = cd(gauss(rng), gauss(rng));
  });
}

int orc_random_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out) {
  return guard([&] {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    cd* o = reinterpret_cast<cd*>(out);
    for (I64 j = 0; j < cols; ++j)
      for (I64 i = 0; i < rows; ++i) o[i + rows * j] = cd(gauss(rng), gauss(rng));
  });
}

int orc_gauss_stream(uint64_t seed, int64_t count, double* out) {
  return guard([&] {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    cd* o = reinterpret_cast<cd*>(out);
    for (I64 n = 0; n < count; ++n) o[n] = cd(gauss(rng), gauss(rng));
  });
}

int orc_fft1(double* v, int64_t n, int inverse) {
  return guard([&] {
    std::vector<cd> work;
    cd* p = reinterpret_cast<cd*>(v);
    fft_line(p, n, inverse != 0, work);
    if (inverse)
      for (I64 i = 0; i < n; ++i) p[i] /= static_cast<double>(n);
  });
}

int orc_fft3(double* t, int64_t n1, int64_t n2, int64_t n3, int inverse) {
  return guard([&] { fft3(reinterpret_cast<cd*>(t), n1, n2, n3, inverse != 0); });
}

int orc_circulant_embed(const double* t, const int64_t dims[3], const int sign[3], double* out) {
  return guard([&] {
    circulant_embed(reinterpret_cast<const cd*>(t), dims, sign, reinterpret_cast<cd*>(out));
  });
}

int orc_transform_factor(const double* u, int64_t n, int64_t r, int sign, double* out) {
  return guard([&] {
    transform_factor(reinterpret_cast<const cd*>(u), n, r, sign, reinterpret_cast<cd*>(out));
  });
}

int orc_component_table(int kind, int basis, int* ncomp, int* comps, int* parity, int* nblock,
                        int* blocks) {
  return guard([&] {
    std::vector<Comp> cs;
    std::vector<Block> bs;
    build_table(kind, basis, cs, bs);
    *ncomp = static_cast<int>(cs.size());
    *nblock = static_cast<int>(bs.size());
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

int orc_decompress_tucker(const int64_t edims[3], const int64_t ranks[3], const double* core,
                          const double* u1, const double* u2, const double* u3, double* dst) {
  return guard([&] {
    decompress_tucker(edims, ranks, reinterpret_cast<const cd*>(core),
                      reinterpret_cast<const cd*>(u1), reinterpret_cast<const cd*>(u2),
                      reinterpret_cast<const cd*>(u3), reinterpret_cast<cd*>(dst));
  });
}

int orc_decompress_cp(const int64_t edims[3], int64_t rank, const double* w1, const double* w2,
                      const double* w3, double* dst) {
  return guard([&] {
    const I64 m1 = edims[0], m2 = edims[1], m3 = edims[2];
    const cd* a = reinterpret_cast<const cd*>(w1);
    const cd* b = reinterpret_cast<const cd*>(w2);
    const cd* c = reinterpret_cast<const cd*>(w3);
    cd* out = reinterpret_cast<cd*>(dst);
    if (rank == 0) {  // operator.hpp:252-255
      std::fill(out, out + m1 * m2 * m3, cd(0.0));
      return;
    }
    std::vector<cd> w1s(static_cast<size_t>(m1 * rank));
    for (I64 k = 0; k < m3; ++k) {
      for (I64 l = 0; l < rank; ++l)  // W1 diag(W3(k, :))
        for (I64 i = 0; i < m1; ++i) w1s[static_cast<size_t>(i + m1 * l)] = a[i + m1 * l] * c[k + m3 * l];
      for (I64 j = 0; j < m2; ++j)  // slab = w1s W2^T
        for (I64 i = 0; i < m1; ++i) {
          cd s = 0.0;
          for (I64 l = 0; l < rank; ++l) s += w1s[static_cast<size_t>(i + m1 * l)] * b[j + m2 * l];
          out[i + m1 * (j + m2 * k)] = s;
        }
    }
  });
}

int orc_apply_operator_tucker(int kind, int basis, const int64_t grid[3], const int64_t* ranks,
                              const double* const* cores, const double* const* u1s,
                              const double* const* u2s, const double* const* u3s,
                              const double* x, double* y) {
  return guard([&] {
    TuckerIn tk{ranks, cores, u1s, u2s, u3s};
    apply_operator(kind, basis, grid, &tk, nullptr, reinterpret_cast<const cd*>(x),
                   reinterpret_cast<cd*>(y));
  });
}

int orc_mv_create(int kind, int basis, const int64_t grid[3], const int64_t* ranks, const double* const* cores,
                  const double* const* u1s, const double* const* u2s, const double* const* u3s, const double* x,
                  void** handle) {
  return guard([&] {
    if (!handle) throw invalid("orc_mv_create: null handle");
    TuckerIn tk{ranks, cores, u1s, u2s, u3s};
    *handle = new StagedMatvec(kind, basis, grid, &tk, nullptr, reinterpret_cast<const cd*>(x));
  });
}
int orc_mv_npieces(void* handle) { return handle ? static_cast<StagedMatvec*>(handle)->npieces() : -1; }
int orc_mv_piece(void* handle, int i) {
  return guard([&] {
    auto* mv = static_cast<StagedMatvec*>(handle);
    if (!mv || i < 0 || i >= mv->npieces()) throw invalid("orc_mv_piece: bad piece");
    mv->piece(i);
  });
}
int orc_mv_result(void* handle, double* y) {
  return guard([&] { static_cast<StagedMatvec*>(handle)->result(reinterpret_cast<cd*>(y)); });
}
void orc_mv_destroy(void* handle) { delete static_cast<StagedMatvec*>(handle); }

int orc_apply_operator_dense(int kind, int basis, const int64_t grid[3],
                             const double* const* spectra, const double* x, double* y) {
  return guard([&] {
    apply_operator(kind, basis, grid, nullptr, spectra, reinterpret_cast<const cd*>(x),
                   reinterpret_cast<cd*>(y));
  });
}

int orc_dense_spectrum(const double* t, const int64_t dims[3], const int sign[3], double* out) {
  return guard([&] {
    cd* o = reinterpret_cast<cd*>(out);
    circulant_embed(reinterpret_cast<const cd*>(t), dims, sign, o);
    fft3(o, 2 * dims[0], 2 * dims[1], 2 * dims[2], false);
  });
}

int orc_dense_bttb(int kind, int basis, const int64_t dims[3], const double* const* tensors,
                   double* out) {
  return guard([&] {
    std::vector<Comp> comps;
    std::vector<Block> blocks;
    build_table(kind, basis, comps, blocks);
    const int S = ncur(basis);
    const I64 n1 = dims[0], n2 = dims[1], n3 = dims[2], nv = n1 * n2 * n3;
    const I64 ld = S * nv;
    cd* a = reinterpret_cast<cd*>(out);
    std::fill(a, a + ld * ld, cd(0.0));
    for (const Block& b : blocks) {
      const Comp& c = comps[static_cast<size_t>(b.c)];
      const cd* t = reinterpret_cast<const cd*>(tensors[b.c]);
      for (I64 k = 0; k < n3; ++k)
        for (I64 j = 0; j < n2; ++j)
          for (I64 i = 0; i < n1; ++i) {
            const I64 row = i + n1 * (j + n2 * k);
            for (I64 kp = 0; kp < n3; ++kp)
              for (I64 jp = 0; jp < n2; ++jp)
                for (I64 ip = 0; ip < n1; ++ip) {
                  const I64 coln = ip + n1 * (jp + n2 * kp);
                  I64 oi = ip - i, oj = jp - j, ok = kp - k;
                  double sign = 1.0;
                  if (oi < 0) { oi = -oi; sign *= c.par[0]; }
                  if (oj < 0) { oj = -oj; sign *= c.par[1]; }
                  if (ok < 0) { ok = -ok; sign *= c.par[2]; }
                  a[(b.t * nv + row) + ld * (b.s * nv + coln)] +=
                      static_cast<double>(b.dsign) * sign * t[oi + n1 * (oj + n2 * ok)];
                }
          }
    }
  });
}

int orc_apply_system_tucker(int basis, const int64_t grid[3], const int64_t* ranks,
                            const double* const* cores, const double* const* u1s,
                            const double* const* u2s, const double* const* u3s,
                            const double* eps_r, double inv_v, const double* x, double* y) {
  return guard([&] {
    TuckerIn tk{ranks, cores, u1s, u2s, u3s};
    apply_system(basis, grid, tk, reinterpret_cast<const cd*>(eps_r), inv_v,
                 reinterpret_cast<const cd*>(x), reinterpret_cast<cd*>(y));
  });
}

static void fill_gmres_out(const GmresOut& g, int* iterations, int* converged,
                           double* final_rel_res, double* history, int history_cap,
                           int* history_len) {
  if (iterations) *iterations = g.iterations;
  if (converged) *converged = g.converged ? 1 : 0;
  if (final_rel_res) *final_rel_res = g.final_rel;
  if (history_len) *history_len = static_cast<int>(g.history.size());
  if (history)
    for (int i = 0; i < history_cap && i < static_cast<int>(g.history.size()); ++i)
      history[i] = g.history[static_cast<size_t>(i)];
}

int orc_gmres(orc_linmap apply, void* apply_ctx, orc_linmap precond, void* precond_ctx,
              int64_t n, const double* rhs, const double* x0, double tol, int inner, int outer,
              double* x, int* iterations, int* converged, double* final_rel_res,
              double* history, int history_cap, int* history_len) {
  return guard([&] {
    VecFn ap = [&](const cd* a, cd* b) {
      apply(reinterpret_cast<const double*>(a), reinterpret_cast<double*>(b), apply_ctx);
    };
    VecFn pc = [&](const cd* a, cd* b) {
      precond(reinterpret_cast<const double*>(a), reinterpret_cast<double*>(b), precond_ctx);
    };
    GmresOut g = gmres(ap, precond ? &pc : nullptr, n, reinterpret_cast<const cd*>(rhs),
                       reinterpret_cast<const cd*>(x0), tol, inner, outer, reinterpret_cast<cd*>(x));
    fill_gmres_out(g, iterations, converged, final_rel_res, history, history_cap, history_len);
  });
}

int orc_gmres_system_tucker(int basis, const int64_t grid[3], const int64_t* ranks,
                            const double* const* cores, const double* const* u1s,
                            const double* const* u2s, const double* const* u3s,
                            const double* eps_r, double inv_v, const double* rhs,
                            const double* x0, double tol, int inner, int outer, double* x,
                            int* iterations, int* converged, double* final_rel_res,
                            double* history, int history_cap, int* history_len) {
  return guard([&] {
    TuckerIn tk{ranks, cores, u1s, u2s, u3s};
    const I64 n = static_cast<I64>(ncur(basis)) * grid[0] * grid[1] * grid[2];
    VecFn ap = [&](const cd* a, cd* b) {
      apply_system(basis, grid, tk, reinterpret_cast<const cd*>(eps_r), inv_v, a, b);
    };
    GmresOut g = gmres(ap, nullptr, n, reinterpret_cast<const cd*>(rhs),
                       reinterpret_cast<const cd*>(x0), tol, inner, outer, reinterpret_cast<cd*>(x));
    fill_gmres_out(g, iterations, converged, final_rel_res, history, history_cap, history_len);
  });
}

int orc_truncated_svd_values(const double* m, int64_t rows, int64_t cols, double tol, int rule,
                             int64_t* rank, double* sigma) {
  return guard([&] {
    if (tol < 0.0) throw invalid("truncated_svd: tol must be >= 0");
    Mat a(rows, cols);
    std::copy(reinterpret_cast<const cd*>(m), reinterpret_cast<const cd*>(m) + rows * cols,
              a.a.begin());
    Mat u, v;
    std::vector<double> s;
    thin_svd(a, u, s, v);
    *rank = truncation_rank(s, tol, rule);
    if (sigma)
      for (size_t i = 0; i < s.size(); ++i) sigma[i] = s[i];
  });
}

int orc_hosvd(const double* t, const int64_t dims[3], double tol, int rule, int64_t ranks[3],
              double* core, double* u1, double* u2, double* u3) {
  return guard([&] {
    if (dims[0] <= 0 || dims[1] <= 0 || dims[2] <= 0)
      throw invalid("hosvd: degenerate tensor dimensions");
    if (tol < 0.0) throw invalid("truncated_svd: tol must be >= 0");
    const cd* tc = reinterpret_cast<const cd*>(t);
    Mat factors[3];
    for (int q = 0; q < 3; ++q) {
      Mat m = unfold(tc, dims, q + 1);
      Mat u, v;
      std::vector<double> s;
      thin_svd(m, u, s, v);
      const I64 r = truncation_rank(s, tol, rule);
      factors[q] = Mat(u.rows, r);
      for (I64 j = 0; j < r; ++j)
        for (I64 i = 0; i < u.rows; ++i) factors[q](i, j) = u(i, j);
      ranks[q] = r;
    }
    if (!core) return;
    std::vector<cd> c(tc, tc + dims[0] * dims[1] * dims[2]);
    I64 d[3] = {dims[0], dims[1], dims[2]};
    for (int q = 0; q < 3; ++q) c = n_mode(c, d, adjoint(factors[q]), q + 1);
    std::copy(c.begin(), c.end(), reinterpret_cast<cd*>(core));
    double* us[3] = {u1, u2, u3};
    for (int q = 0; q < 3; ++q)
      if (us[q]) std::copy(factors[q].a.begin(), factors[q].a.end(), reinterpret_cast<cd*>(us[q]));
  });
}

// cp_als (decomp.hpp:237-298).  f_q: dims[q] x r column-major (may be null); trace: up to
// trace_cap entries; flags[0] = converged, flags[1] = ill_posed_rank.
int orc_cp_als(const double* t, const int64_t dims[3], int64_t r, int max_iters, double stall_tol, uint64_t seed,
               double* f1, double* f2, double* f3, double* trace, int trace_cap, int* ntrace, int flags[2]) {
  return guard([&] {
    CpAlsOut o = cp_als(reinterpret_cast<const cd*>(t), dims, r, max_iters, stall_tol, seed);
    double* fs[3] = {f1, f2, f3};
    for (int q = 0; q < 3; ++q)
      if (fs[q]) std::copy(o.f[q].a.begin(), o.f[q].a.end(), reinterpret_cast<cd*>(fs[q]));
    *ntrace = static_cast<int>(o.trace.size());
    for (int i = 0; i < std::min(trace_cap, *ntrace); ++i) trace[i] = o.trace[static_cast<size_t>(i)];
    flags[0] = o.converged;
    flags[1] = o.ill_posed;
  });
}

// tucker_cp (decomp.hpp:336-373): hosvd, cp_als on the core (rank min(r_q) unless cp_rank >= 0,
// default seed), W_q = U_q V_q.  w_q: dims[q] x rank (null: only *rank_out is set).
// errs = {hosvd_relative_error, core_cp_relative_error, achieved_relative_error}.
int orc_tucker_cp(const double* t, const int64_t dims[3], double tol, int cp_iters, int rule, int64_t cp_rank,
                  double stall_tol, int64_t* rank_out, double* w1, double* w2, double* w3, double errs[3],
                  double* trace, int trace_cap, int* ntrace) {
  return guard([&] {
    int64_t rk[3];
    if (orc_hosvd(t, dims, tol, rule, rk, nullptr, nullptr, nullptr, nullptr) != 0) throw invalid(g_err);
    std::vector<cd> core(static_cast<size_t>(rk[0] * rk[1] * rk[2]));
    Mat U[3];
    for (int q = 0; q < 3; ++q) U[q] = Mat(dims[q], rk[q]);
    if (orc_hosvd(t, dims, tol, rule, rk, reinterpret_cast<double*>(core.data()),
                  reinterpret_cast<double*>(U[0].a.data()), reinterpret_cast<double*>(U[1].a.data()),
                  reinterpret_cast<double*>(U[2].a.data())) != 0)
      throw invalid(g_err);
    const I64 r = cp_rank >= 0 ? cp_rank : std::min({rk[0], rk[1], rk[2]});
    *rank_out = r;
    if (!w1) return;
    const cd* tc = reinterpret_cast<const cd*>(t);
    const std::vector<cd> tv(tc, tc + dims[0] * dims[1] * dims[2]);
    const double tnorm = fro(tv);
    {  // ||t - tucker reconstruct|| / ||t||
      std::vector<cd> rec = core;
      I64 d[3] = {rk[0], rk[1], rk[2]};
      for (int q = 0; q < 3; ++q) rec = n_mode(rec, d, U[q], q + 1);
      for (size_t e = 0; e < rec.size(); ++e) rec[e] -= tv[e];
      errs[0] = tnorm > 0 ? fro(rec) / tnorm : 0.0;
    }
    const I64 cd3[3] = {rk[0], rk[1], rk[2]};
    CpAlsOut cp = cp_als(core.data(), cd3, r, cp_iters, stall_tol, 0x5eed);
    errs[1] = cp.trace.empty() ? 0.0 : cp.trace.back();
    Mat W[3];
    for (int q = 0; q < 3; ++q) W[q] = matmul(U[q], cp.f[q]);
    double* ws[3] = {w1, w2, w3};
    for (int q = 0; q < 3; ++q) std::copy(W[q].a.begin(), W[q].a.end(), reinterpret_cast<cd*>(ws[q]));
    if (tnorm > 0) {
      std::vector<cd> rec = cp_reconstruct(W[0], W[1], W[2]);
      for (size_t e = 0; e < rec.size(); ++e) rec[e] -= tv[e];
      errs[2] = fro(rec) / tnorm;
    } else {
      errs[2] = 0.0;
    }
    *ntrace = static_cast<int>(cp.trace.size());
    if (trace)
      for (int i = 0; i < std::min(trace_cap, *ntrace); ++i) trace[i] = cp.trace[static_cast<size_t>(i)];
  });
}

}  // extern "C"

// ---- solve_scene stages (solver.hpp:148-285; grid.hpp:14-100; quadrature.hpp:23-52)
namespace {

constexpr double kEps0 = 8.8541878128e-12, kMu0 = 1.25663706212e-6, kC0 = 299792458.0;
constexpr double kPi = 3.141592653589793238462643383279502884;

struct Scene {  // VoxelGrid + DielectricMap frequency + PlaneWave
  I64 n[3];
  double res[3], org[3], freq;
  double pol[3], dir[3], amp;
  double omega() const { return 2.0 * kPi * freq; }
  double k0() const { return omega() / kC0; }
  cd ce() const { return cd(0.0, omega() * kEps0); }
  I64 nv() const { return n[0] * n[1] * n[2]; }
  void center(I64 i, I64 j, I64 k, double r[3]) const {
    r[0] = org[0] + (static_cast<double>(i) + 0.5) * res[0];
    r[1] = org[1] + (static_cast<double>(j) + 0.5) * res[1];
    r[2] = org[2] + (static_cast<double>(k) + 0.5) * res[2];
  }
  cd phase(const double r[3]) const {
    return std::exp(cd(0.0, -k0() * (dir[0] * r[0] + dir[1] * r[1] + dir[2] * r[2])));
  }
};

Scene make_scene(const int64_t dims[3], const double geo[6], double f, const double* pw) {
  Scene s{};
  for (int a = 0; a < 3; ++a) {
    if (dims[a] < 1) throw std::invalid_argument("VoxelGrid: dims must be >= 1");
    if (!(geo[a] > 0.0)) throw std::invalid_argument("VoxelGrid: resolution must be > 0");
    s.n[a] = dims[a];
    s.res[a] = geo[a];
    s.org[a] = geo[3 + a];
  }
  s.freq = f;
  if (pw) {
    const double pn = std::sqrt(pw[0] * pw[0] + pw[1] * pw[1] + pw[2] * pw[2]);
    const double dn = std::sqrt(pw[3] * pw[3] + pw[4] * pw[4] + pw[5] * pw[5]);
    for (int a = 0; a < 3; ++a) {
      s.pol[a] = pw[a] / pn;
      s.dir[a] = pw[3 + a] / dn;
    }
    if (std::abs(s.pol[0] * s.dir[0] + s.pol[1] * s.dir[1] + s.pol[2] * s.dir[2]) > 1e-12)
      throw std::invalid_argument("PlaneWave: polarization must be orthogonal to direction");
    s.amp = pw[6];
  }
  return s;
}

void gauss01(int p, std::vector<double>& nodes, std::vector<double>& weights) {
  if (p < 1) throw std::invalid_argument("gauss_rule: need at least one point");
  nodes.assign(p, 0.0);
  weights.assign(p, 0.0);
  for (int i = 0; i < (p + 1) / 2; ++i) {
    double x = std::cos(kPi * (i + 0.75) / (p + 0.5)), deriv = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p1 = 1.0, p2 = 0.0;
      for (int k = 0; k < p; ++k) {
        const double p3 = p2;
        p2 = p1;
        p1 = ((2.0 * k + 1.0) * x * p2 - k * p3) / (k + 1.0);
      }
      deriv = p * (x * p1 - p2) / (x * x - 1.0);
      const double dx = p1 / deriv;
      x -= dx;
      if (std::abs(dx) < 1e-15) break;
    }
    const double w = 1.0 / ((1.0 - x * x) * deriv * deriv);
    nodes[i] = 0.5 * (1.0 - x);
    weights[i] = w;
    nodes[p - 1 - i] = 0.5 * (1.0 + x);
    weights[p - 1 - i] = w;
  }
}

}  // namespace

extern "C" {

int orc_build_rhs(const int64_t dims[3], const double geo[6], double frequency, const double pw[7],
                  const double* eps_r, int quad, double* rhs) {
  return guard([&] {
    if (quad < 1) throw std::invalid_argument("build_rhs: bad quadrature order");
    const Scene s = make_scene(dims, geo, frequency, pw);
    const cd* eps = reinterpret_cast<const cd*>(eps_r);
    cd* out = reinterpret_cast<cd*>(rhs);
    const I64 nv = s.nv();
    std::vector<double> qn, qw;
    if (quad > 1) gauss01(quad, qn, qw);
    for (I64 q = 0; q < 3 * nv; ++q) out[q] = cd(0.0);  // CurrentField is zero-initialised
    for (I64 k = 0; k < s.n[2]; ++k)
      for (I64 j = 0; j < s.n[1]; ++j)
        for (I64 i = 0; i < s.n[0]; ++i) {
          const I64 v = i + s.n[0] * (j + s.n[1] * k);
          const cd chi = eps[v] - 1.0;
          if (chi == cd(0.0)) continue;
          double c[3];
          s.center(i, j, k, c);
          cd ph(0.0);
          if (quad == 1) {
            ph = s.phase(c);
          } else {
            for (int a = 0; a < quad; ++a)
              for (int b = 0; b < quad; ++b)
                for (int d = 0; d < quad; ++d) {
                  const double r[3] = {c[0] + s.res[0] * (qn[a] - 0.5), c[1] + s.res[1] * (qn[b] - 0.5),
                                       c[2] + s.res[2] * (qn[d] - 0.5)};
                  ph += qw[a] * qw[b] * qw[d] * s.phase(r);
                }
          }
          for (int q = 0; q < 3; ++q) out[q * nv + v] = s.ce() * chi * (s.pol[q] * (s.amp * ph));
        }
  });
}

int orc_recover_fields(const int64_t dims[3], const double geo[6], double frequency, const double pw[7],
                       const double* eps_r, const double* j, const double* kj, double* e, double* h) {
  return guard([&] {
    const Scene s = make_scene(dims, geo, frequency, pw);
    const cd* eps = reinterpret_cast<const cd*>(eps_r);
    const cd* jj = reinterpret_cast<const cd*>(j);
    cd* eo = reinterpret_cast<cd*>(e);
    const I64 nv = s.nv();
    const double inv_v = 1.0 / (s.res[0] * s.res[1] * s.res[2]);
    const double hd[3] = {s.dir[1] * s.pol[2] - s.dir[2] * s.pol[1], s.dir[2] * s.pol[0] - s.dir[0] * s.pol[2],
                          s.dir[0] * s.pol[1] - s.dir[1] * s.pol[0]};
    const double eta0 = std::sqrt(kMu0 / kEps0);
    for (I64 k = 0; k < s.n[2]; ++k)
      for (I64 y = 0; y < s.n[1]; ++y)
        for (I64 i = 0; i < s.n[0]; ++i) {
          const I64 v = i + s.n[0] * (y + s.n[1] * k);
          double c[3];
          s.center(i, y, k, c);
          const cd chi = eps[v] - 1.0;
          if (chi == cd(0.0)) {
            const cd ph = s.phase(c);
            for (int q = 0; q < 3; ++q) eo[q * nv + v] = s.pol[q] * (s.amp * ph);
          } else {
            const cd inv = 1.0 / (s.ce() * chi);
            for (int q = 0; q < 3; ++q) eo[q * nv + v] = inv * jj[q * nv + v];
          }
          if (kj) {
            const cd ph = s.phase(c);
            const cd* kk = reinterpret_cast<const cd*>(kj);
            cd* ho = reinterpret_cast<cd*>(h);
            for (int q = 0; q < 3; ++q) ho[q * nv + v] = hd[q] * (s.amp / eta0 * ph) + inv_v * kk[q * nv + v];
          }
        }
  });
}

int orc_postprocess(const int64_t dims[3], const double geo[6], double frequency, const double* eps_r,
                    const double* e, const double* h, double* p_abs, double* b1, double* total) {
  return guard([&] {
    const Scene s = make_scene(dims, geo, frequency, nullptr);
    const cd* eps = reinterpret_cast<const cd*>(eps_r);
    const cd* ee = reinterpret_cast<const cd*>(e);
    const I64 nv = s.nv();
    double tot = 0.0;
    for (I64 v = 0; v < nv; ++v) {
      double e2 = 0.0;
      for (int q = 0; q < 3; ++q) e2 += std::norm(ee[q * nv + v]);
      const double p = 0.5 * (-eps[v].imag() * kEps0 * s.omega()) * e2;
      p_abs[v] = p;
      tot += p;
    }
    if (total) *total = tot * (s.res[0] * s.res[1] * s.res[2]);
    if (h) {
      const cd* hh = reinterpret_cast<const cd*>(h);
      for (I64 v = 0; v < nv; ++v) b1[v] = kMu0 * std::abs(hh[v] + cd(0.0, 1.0) * hh[nv + v]);
    }
  });
}

}  // extern "C"

// ============================================================================
// Green's-tensor assembly (assembly.hpp, kernels.hpp, quadrature.hpp): PWC Galerkin
// Toeplitz-defining tensors of the N, K and scalar-g kernels on a uniform grid.
// ============================================================================
namespace {

struct V3 {
  double v[3];
  double operator[](int i) const { return v[i]; }
  double& operator[](int i) { return v[i]; }
  double norm() const { return std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]); }
};
V3 sub(const V3& a, const V3& b) { return V3{{a[0] - b[0], a[1] - b[1], a[2] - b[2]}}; }

constexpr double kPiA = 3.14159265358979323846264338327950288;
constexpr double kInv4pi = 1.0 / (4.0 * kPiA);

// kernels.hpp:28-60: entire helpers of x = -i k R by series for |x| <= 1
cd phi0(cd x) {
  if (std::abs(x) > 1.0) return std::exp(x) - 1.0;
  cd term = x, sum = x;
  for (int n = 2; n < 26; ++n) {
    term *= x / static_cast<double>(n);
    sum += term;
  }
  return sum;
}
cd psi1(cd x) {
  if (std::abs(x) > 1.0) return (x - 1.0) * std::exp(x) + 1.0;
  cd xn = x, sum = 0.0;
  for (int n = 2; n < 28; ++n) {
    xn *= x / static_cast<double>(n);
    sum += xn * static_cast<double>(n - 1);
  }
  return sum;
}
cd psi2(cd x) {
  if (std::abs(x) > 1.0) return std::exp(x) * (x * x - 2.0 * x + 2.0) - 2.0;
  cd sum = 0.0;
  cd xm = x * x / 2.0;
  for (int m = 3; m < 30; ++m) {
    xm *= x / static_cast<double>(m);
    sum += xm * static_cast<double>((m - 1) * (m - 2));
  }
  return sum;
}

struct Radial {
  cd g, gp, gpp;
};
// kernels.hpp:67-76
Radial radial(double R, double k) {
  const cd e = std::exp(cd(0.0, -k * R));
  const cd ikr(0.0, k * R);
  Radial r;
  r.g = e * kInv4pi / R;
  r.gp = -(1.0 + ikr) * e * kInv4pi / (R * R);
  r.gpp = (2.0 + 2.0 * ikr - k * k * R * R) * e * kInv4pi / (R * R * R);
  return r;
}
// kernels.hpp:84-91
Radial radial_dynamic(double R, double k) {
  const cd x(0.0, -k * R);
  Radial r;
  r.g = phi0(x) * kInv4pi / R;
  r.gp = psi1(x) * kInv4pi / (R * R);
  r.gpp = psi2(x) * kInv4pi / (R * R * R);
  return r;
}
// kernels.hpp:95-99
cd hessian_entry(const Radial& h, const V3& rhat, double R, int q, int qp) {
  const cd iso = h.gp / R;
  const cd aniso = h.gpp - iso;
  return aniso * rhat[q] * rhat[qp] + (q == qp ? iso : cd(0.0));
}
V3 unit(const V3& r, double R) { return V3{{r[0] / R, r[1] / R, r[2] / R}}; }
// kernels.hpp:103-108
cd n_kernel(const V3& rv, double k, int q, int qp) {
  const double R = rv.norm();
  const Radial h = radial(R, k);
  return hessian_entry(h, unit(rv, R), R, q, qp) + (q == qp ? k * k * h.g : cd(0.0));
}
// kernels.hpp:113-119
cd n_kernel_self_remainder(const V3& rv, double k, int q, int qp) {
  const double R = rv.norm();
  const Radial hd = radial_dynamic(R, k);
  const cd g_full = hd.g + kInv4pi / R;
  return hessian_entry(hd, unit(rv, R), R, q, qp) + (q == qp ? k * k * g_full : cd(0.0));
}
int levi_civita(int a, int b, int c) {
  if (a == b || b == c || a == c) return 0;
  return ((b - a + 3) % 3 == 1) ? 1 : -1;
}
// kernels.hpp:128-134
cd k_kernel(const V3& rv, double k, int q, int qp) {
  if (q == qp) return 0.0;
  const int a = 3 - q - qp;
  const double R = rv.norm();
  const Radial h = radial(R, k);
  return static_cast<double>(levi_civita(q, a, qp)) * h.gp * rv[a] / R;
}

// quadrature.hpp:21-58 (Newton on the Legendre roots, mapped to [0, 1])
struct GaussRuleO {
  std::vector<double> nodes, weights;
};
const GaussRuleO& gauss_rule_o(int p) {
  static std::mutex mu;
  static std::map<int, GaussRuleO> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(p);
  if (it != cache.end()) return it->second;
  if (p < 1) throw invalid("gauss_rule: need at least one point");
  GaussRuleO r;
  r.nodes.resize(static_cast<size_t>(p));
  r.weights.resize(static_cast<size_t>(p));
  const int m = (p + 1) / 2;
  for (int i = 0; i < m; ++i) {
    double x = std::cos(kPiA * (i + 0.75) / (p + 0.5));
    double deriv = 0.0;
    for (int iter = 0; iter < 100; ++iter) {
      double p1 = 1.0, p2 = 0.0;
      for (int k = 0; k < p; ++k) {
        const double p3 = p2;
        p2 = p1;
        p1 = ((2.0 * k + 1.0) * x * p2 - k * p3) / (k + 1.0);
      }
      deriv = p * (x * p1 - p2) / (x * x - 1.0);
      const double dx = p1 / deriv;
      x -= dx;
      if (std::abs(dx) < 1e-15) break;
    }
    const double w = 1.0 / ((1.0 - x * x) * deriv * deriv);
    r.nodes[static_cast<size_t>(i)] = 0.5 * (1.0 - x);
    r.weights[static_cast<size_t>(i)] = w;
    r.nodes[static_cast<size_t>(p - 1 - i)] = 0.5 * (1.0 + x);
    r.weights[static_cast<size_t>(p - 1 - i)] = w;
  }
  return cache.emplace(p, std::move(r)).first->second;
}

struct Box3O {
  double lo[3], hi[3];
};
using KFn = std::function<cd(const V3&)>;
// quadrature.hpp:71-86
cd integrate_box(const KFn& f, const Box3O& box, int p) {
  const GaussRuleO& g = gauss_rule_o(p);
  const double lx = box.hi[0] - box.lo[0], ly = box.hi[1] - box.lo[1], lz = box.hi[2] - box.lo[2];
  cd sum = 0.0;
  for (int a = 0; a < p; ++a)
    for (int b = 0; b < p; ++b)
      for (int c = 0; c < p; ++c) {
        V3 u{{box.lo[0] + lx * g.nodes[a], box.lo[1] + ly * g.nodes[b], box.lo[2] + lz * g.nodes[c]}};
        sum += g.weights[a] * g.weights[b] * g.weights[c] * f(u);
      }
  return sum * (lx * ly * lz);
}
// quadrature.hpp:92-118
cd integrate_box_duffy(const KFn& f, const Box3O& box, const int corner[3], int p) {
  const GaussRuleO& g = gauss_rule_o(p);
  double base[3], span[3];
  for (int a = 0; a < 3; ++a) {
    base[a] = corner[a] ? box.hi[a] : box.lo[a];
    span[a] = (corner[a] ? box.lo[a] : box.hi[a]) - base[a];
  }
  const double jac = std::abs(span[0] * span[1] * span[2]);
  cd sum = 0.0;
  for (int radial_ax = 0; radial_ax < 3; ++radial_ax) {
    const int s1 = (radial_ax + 1) % 3, s2 = (radial_ax + 2) % 3;
    for (int a = 0; a < p; ++a) {
      const double t = g.nodes[a];
      for (int b = 0; b < p; ++b)
        for (int c = 0; c < p; ++c) {
          double v[3];
          v[radial_ax] = t;
          v[s1] = t * g.nodes[b];
          v[s2] = t * g.nodes[c];
          V3 u{{base[0] + span[0] * v[0], base[1] + span[1] * v[1], base[2] + span[2] * v[2]}};
          sum += g.weights[a] * g.weights[b] * g.weights[c] * (t * t) * f(u);
        }
    }
  }
  return sum * jac;
}
using RFn = std::function<cd(double, double)>;
// quadrature.hpp:126-136
cd integrate_rect(const RFn& f, const double lo[2], const double hi[2], int p) {
  const GaussRuleO& g = gauss_rule_o(p);
  const double lx = hi[0] - lo[0], ly = hi[1] - lo[1];
  cd sum = 0.0;
  for (int a = 0; a < p; ++a)
    for (int b = 0; b < p; ++b)
      sum += g.weights[a] * g.weights[b] * f(lo[0] + lx * g.nodes[a], lo[1] + ly * g.nodes[b]);
  return sum * (lx * ly);
}
// quadrature.hpp:139-166
cd integrate_rect_duffy(const RFn& f, const double lo[2], const double hi[2], const int corner[2], int p) {
  const GaussRuleO& g = gauss_rule_o(p);
  double base[2], span[2];
  for (int a = 0; a < 2; ++a) {
    base[a] = corner[a] ? hi[a] : lo[a];
    span[a] = (corner[a] ? lo[a] : hi[a]) - base[a];
  }
  const double jac = std::abs(span[0] * span[1]);
  cd sum = 0.0;
  for (int radial_ax = 0; radial_ax < 2; ++radial_ax) {
    const int other = 1 - radial_ax;
    for (int a = 0; a < p; ++a) {
      const double t = g.nodes[a];
      for (int b = 0; b < p; ++b) {
        double v[2];
        v[radial_ax] = t;
        v[other] = t * g.nodes[b];
        sum += g.weights[a] * g.weights[b] * t * f(base[0] + span[0] * v[0], base[1] + span[1] * v[1]);
      }
    }
  }
  return sum * jac;
}

// assembly.hpp:49-79: Galerkin voxel-pair integral as a tent-weighted 3D correlation
cd correlation_entry(const KFn& kernel, const V3& d, const double delta[3], int points, bool duffy_at_d) {
  std::vector<double> cuts[3];
  for (int a = 0; a < 3; ++a) {
    cuts[a] = {-delta[a], 0.0, delta[a]};
    if (duffy_at_d && d[a] > -delta[a] && d[a] < delta[a] && d[a] != 0.0) {
      cuts[a].push_back(d[a]);
      std::sort(cuts[a].begin(), cuts[a].end());
    }
  }
  KFn weighted = [&](const V3& u) {
    const double w = (delta[0] - std::abs(u[0])) * (delta[1] - std::abs(u[1])) * (delta[2] - std::abs(u[2]));
    return kernel(sub(u, d)) * w;
  };
  cd sum = 0.0;
  for (size_t ia = 0; ia + 1 < cuts[0].size(); ++ia)
    for (size_t ib = 0; ib + 1 < cuts[1].size(); ++ib)
      for (size_t ic = 0; ic + 1 < cuts[2].size(); ++ic) {
        Box3O box{{cuts[0][ia], cuts[1][ib], cuts[2][ic]}, {cuts[0][ia + 1], cuts[1][ib + 1], cuts[2][ic + 1]}};
        bool corner = duffy_at_d;
        int which[3] = {0, 0, 0};
        for (int a = 0; a < 3; ++a) {
          const double lo = box.lo[a], hi = box.hi[a];
          if (d[a] == lo) which[a] = 0;
          else if (d[a] == hi) which[a] = 1;
          else corner = false;
        }
        sum += corner ? integrate_box_duffy(weighted, box, which, points) : integrate_box(weighted, box, points);
      }
  return sum;
}

// assembly.hpp:84-104
double face_pair_static(double dt1, double dt2, double h, int points) {
  RFn f = [&](double u, double v) {
    const double w = (dt1 - std::abs(u)) * (dt2 - std::abs(v));
    return cd(w * kInv4pi / std::sqrt(h * h + u * u + v * v));
  };
  cd sum = 0.0;
  for (int su = 0; su < 2; ++su)
    for (int sv = 0; sv < 2; ++sv) {
      const double lo[2] = {su ? 0.0 : -dt1, sv ? 0.0 : -dt2};
      const double hi[2] = {su ? dt1 : 0.0, sv ? dt2 : 0.0};
      if (h == 0.0) {
        const int corner[2] = {su ? 0 : 1, sv ? 0 : 1};
        sum += integrate_rect_duffy(f, lo, hi, corner, points);
      } else {
        sum += integrate_rect(f, lo, hi, points);
      }
    }
  return sum.real();
}

struct QuadSpec {
  int far = 5, near = 10, near_radius = 1, surface = 12, volume = 6;
  void validate() const {
    if (far < 1 || near < 1 || surface < 1 || volume < 1)
      throw invalid("QuadratureSpec: quadrature budget of zero");
    if (near_radius < 1) throw invalid("QuadratureSpec: near_radius must be >= 1");
  }
};

// assembly.hpp:127-150 (diagonal of the static nabla-nabla dyad; off-diagonals are 0)
void self_static_term(const double delta[3], const QuadSpec& quad, double dyad[3], double* gram, double* err,
                      bool* converged) {
  quad.validate();
  *gram = delta[0] * delta[1] * delta[2];
  auto diagonal = [&](int q, int points) {
    const int t1 = (q + 1) % 3, t2 = (q + 2) % 3;
    const double same = face_pair_static(delta[t1], delta[t2], 0.0, points);
    const double opp = face_pair_static(delta[t1], delta[t2], delta[q], points);
    return 2.0 * (opp - same);
  };
  double max_change = 0.0;
  for (int q = 0; q < 3; ++q) {
    const double v = diagonal(q, quad.surface);
    const double v_refined = diagonal(q, quad.surface + 4);
    dyad[q] = v_refined;
    max_change = std::max(max_change, std::abs(v_refined - v) / *gram);
  }
  *err = max_change;
  *converged = max_change < 1e-7;
}

// assembly.hpp:159-233 (op 0 = N, 1 = K, 2 = scalar g), PWC only
void assemble_defining_tensor(const I64 dims[3], const double res[3], double k0, int op, int q, int qp,
                              const QuadSpec& quad, cd* t) {
  quad.validate();
  for (int a = 0; a < 3; ++a)
    if (dims[a] < 1 || !(res[a] > 0.0)) throw invalid("assemble_defining_tensor: bad grid");
  if (op < 0 || op > 2 || q < 0 || q > 2 || qp < 0 || qp > 2) throw invalid("assemble_defining_tensor: bad component");
  const double scale = res[0];
  const double delta[3] = {1.0, res[1] / scale, res[2] / scale};
  const double k = k0 * scale;
  // parity (components.hpp:46-65): N(q,q') odd along q and q' (q != q'), K odd along the third axis
  int par[3] = {1, 1, 1};
  if (op == 0 && q != qp) par[q] = par[qp] = -1;
  if (op == 1 && q != qp) par[3 - q - qp] = -1;
  KFn kernel;
  double si_power = 3.0;
  if (op == 0) {
    kernel = [=](const V3& r) { return n_kernel(r, k, q, qp); };
  } else if (op == 1) {
    kernel = [=](const V3& r) { return k_kernel(r, k, q, qp); };
    si_power = 4.0;
  } else {
    kernel = [=](const V3& r) { return radial(r.norm(), k).g; };
    si_power = 5.0;
  }
  const double si_scale = std::pow(scale, si_power);
  cd self_entry = 0.0;
  const V3 zero{{0.0, 0.0, 0.0}};
  if (op == 0) {
    double dyad[3], gram, err;
    bool conv;
    self_static_term(delta, quad, dyad, &gram, &err, &conv);
    KFn rem = [=](const V3& r) { return n_kernel_self_remainder(r, k, q, qp); };
    self_entry = correlation_entry(rem, zero, delta, quad.volume, true);
    self_entry += (q == qp ? gram + dyad[q] : 0.0);
  } else if (op == 2) {
    self_entry = correlation_entry(kernel, zero, delta, quad.volume, true);
  }
  const I64 n1 = dims[0], n2 = dims[1], n3 = dims[2];
  parallel_for(n3, [&](I64 kk, int) {
    for (I64 jj = 0; jj < n2; ++jj)
      for (I64 ii = 0; ii < n1; ++ii) {
        cd& out = t[ii + n1 * (jj + n2 * kk)];
        if ((par[0] < 0 && ii == 0) || (par[1] < 0 && jj == 0) || (par[2] < 0 && kk == 0)) {
          out = 0.0;
          continue;
        }
        const I64 cheb = std::max({ii, jj, kk});
        if (cheb == 0) {
          out = self_entry * si_scale;
          continue;
        }
        const V3 d{{static_cast<double>(ii) * delta[0], static_cast<double>(jj) * delta[1],
                    static_cast<double>(kk) * delta[2]}};
        const bool near = cheb <= quad.near_radius;
        out = correlation_entry(kernel, d, delta, near ? quad.near : quad.far, near) * si_scale;
      }
  });
}

QuadSpec quad_from(const int* q5) {
  QuadSpec q;
  if (q5) {
    q.far = q5[0];
    q.near = q5[1];
    q.near_radius = q5[2];
    q.surface = q5[3];
    q.volume = q5[4];
  }
  return q;
}

KFn kernel_of(int op, double k, int q, int qp) {
  if (op == 0) return [=](const V3& r) { return n_kernel(r, k, q, qp); };
  if (op == 1) return [=](const V3& r) { return k_kernel(r, k, q, qp); };
  if (op == 3) return [=](const V3& r) { return n_kernel_self_remainder(r, k, q, qp); };
  return [=](const V3& r) { return radial(r.norm(), k).g; };
}

}  // namespace

extern "C" {

int orc_assemble(const int64_t dims[3], const double res[3], double k0, int op, int q, int qp, const int* quad5,
                 double* out) {
  return guard([&] {
    const I64 d[3] = {dims[0], dims[1], dims[2]};
    assemble_defining_tensor(d, res, k0, op, q, qp, quad_from(quad5), reinterpret_cast<cd*>(out));
  });
}

int orc_self_static_term(const double delta[3], const int* quad5, double dyad_diag[3], double* gram, double* err,
                         int* converged) {
  return guard([&] {
    bool c = false;
    self_static_term(delta, quad_from(quad5), dyad_diag, gram, err, &c);
    if (converged) *converged = c ? 1 : 0;
  });
}

int orc_correlation_entry(int op, double k, int q, int qp, const double d[3], const double delta[3], int points,
                          int duffy, double* out) {
  return guard([&] {
    const cd v = correlation_entry(kernel_of(op, k, q, qp), V3{{d[0], d[1], d[2]}}, delta, points, duffy != 0);
    out[0] = v.real();
    out[1] = v.imag();
  });
}

int orc_kernel_eval(int op, double k, int q, int qp, const double r[3], double* out) {
  return guard([&] {
    const V3 rv{{r[0], r[1], r[2]}};
    if (rv.norm() <= 0.0) throw std::domain_error("green_g: singular point |R| = 0");
    const cd v = kernel_of(op, k, q, qp)(rv);
    out[0] = v.real();
    out[1] = v.imag();
  });
}

int orc_radial(double R, double k, int dynamic, double* out6) {
  return guard([&] {
    const Radial h = dynamic ? radial_dynamic(R, k) : radial(R, k);
    const cd v[3] = {h.g, h.gp, h.gpp};
    for (int i = 0; i < 3; ++i) {
      out6[2 * i] = v[i].real();
      out6[2 * i + 1] = v[i].imag();
    }
  });
}

// test_assembly.cpp:14-37: brute-force 6D Gauss over (test voxel) x (source voxel)
int orc_brute_pair_integral(int op, double k, int q, int qp, const double d[3], const double del[3], int p,
                            double* out) {
  return guard([&] {
    const GaussRuleO& g = gauss_rule_o(p);
    const KFn kern = kernel_of(op, k, q, qp);
    std::vector<cd> part(static_cast<size_t>(p));
    parallel_for(p, [&](I64 a, int) {
      cd sum = 0.0;
      for (int b = 0; b < p; ++b)
        for (int c = 0; c < p; ++c)
          for (int e = 0; e < p; ++e)
            for (int f = 0; f < p; ++f)
              for (int h = 0; h < p; ++h) {
                const V3 rt{{del[0] * (g.nodes[a] - 0.5), del[1] * (g.nodes[b] - 0.5), del[2] * (g.nodes[c] - 0.5)}};
                const V3 rs{{d[0] + del[0] * (g.nodes[e] - 0.5), d[1] + del[1] * (g.nodes[f] - 0.5),
                             d[2] + del[2] * (g.nodes[h] - 0.5)}};
                sum += g.weights[a] * g.weights[b] * g.weights[c] * g.weights[e] * g.weights[f] * g.weights[h] *
                       kern(sub(rt, rs));
              }
      part[static_cast<size_t>(a)] = sum;
    });
    cd sum = 0.0;
    for (const cd& v : part) sum += v;
    const double v = del[0] * del[1] * del[2];
    sum *= v * v;
    out[0] = sum.real();
    out[1] = sum.imag();
  });
}

}  // extern "C"
