// cp_als.cu -- CP-ALS on the HOSVD core (the CP half of tucker_cp, decomp.hpp:237-298,
// 336-373).  The core is r1 x r2 x r3 (<= 28^3 complex on the device path), so one sweep is
// ~r^4 complex MACs: this is setup work of the same size as the r x r eigenproblems of the
// HOSVD and runs on the host next to them.  The large tensors (the defining tensor, its
// unfoldings, the residual norms) stay on the device (api.cu tucker_cp_dev, kernels_hosvd.cu).
//
// Same algorithm and order as the reference: factors initialised from the leading left
// singular vectors of the unfoldings (seeded Gaussian columns beyond the unfolding's rank,
// std::mt19937_64 + std::normal_distribution, unit norm), sweeps f0, f1, f2 by the normal
// equations with an SVD pseudo-inverse (relative cutoff 1e-12) of the Hadamard-product Gram,
// column normalisation to a common magnitude, relative error per sweep, stop when the
// decrease falls below stall_tol.  The SVDs are one-sided (Hestenes) Jacobi: left singular
// vectors to full relative accuracy, as the reference's QR + JacobiSVD.
#include <algorithm>
#include <cmath>
#include <complex>
#include <limits>
#include <random>
#include <stdexcept>
#include <vector>

#include "kernels.cuh"

namespace vie {

namespace {

using cd = std::complex<double>;

struct CMat {  // column-major
  int64_t rows = 0, cols = 0;
  std::vector<cd> a;
  CMat() = default;
  CMat(int64_t r, int64_t c) : rows(r), cols(c), a(static_cast<size_t>(r * c), cd(0.0)) {}
  cd& operator()(int64_t i, int64_t j) { return a[static_cast<size_t>(i + rows * j)]; }
  cd operator()(int64_t i, int64_t j) const { return a[static_cast<size_t>(i + rows * j)]; }
};

CMat adj(const CMat& m) {
  CMat o(m.cols, m.rows);
  for (int64_t j = 0; j < m.cols; ++j)
    for (int64_t i = 0; i < m.rows; ++i) o(j, i) = std::conj(m(i, j));
  return o;
}

// One-sided Jacobi SVD of a tall m x n matrix (m >= n): A V = W, sigma_j = |W_j|,
// U_j = W_j / sigma_j; sorted by sigma descending.
void jsvd_tall(const CMat& m, CMat& u, std::vector<double>& s, CMat& v) {
  const int64_t rows = m.rows, n = m.cols;
  CMat w = m;
  CMat vv(n, n);
  for (int64_t i = 0; i < n; ++i) vv(i, i) = 1.0;
  for (int sweep = 0; sweep < 80; ++sweep) {
    bool rotated = false;
    for (int64_t p = 0; p + 1 < n; ++p)
      for (int64_t q = p + 1; q < n; ++q) {
        double al = 0.0, be = 0.0;
        cd ga = 0.0;
        for (int64_t i = 0; i < rows; ++i) {
          al += std::norm(w(i, p));
          be += std::norm(w(i, q));
          ga += std::conj(w(i, p)) * w(i, q);
        }
        const double mag = std::abs(ga);
        if (mag <= 1e-300 || mag <= 1e-15 * std::sqrt(al * be)) continue;
        rotated = true;
        const double tau = (be - al) / (2.0 * mag);
        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (std::abs(tau) + std::sqrt(1.0 + tau * tau));
        const double c = 1.0 / std::sqrt(1.0 + t * t), sn = t * c;
        const cd ph = ga / mag;
        const cd jpq = sn * ph, jqp = -sn * std::conj(ph);
        for (int64_t i = 0; i < rows; ++i) {
          const cd x = w(i, p), y = w(i, q);
          w(i, p) = c * x + jqp * y;
          w(i, q) = jpq * x + c * y;
        }
        for (int64_t i = 0; i < n; ++i) {
          const cd x = vv(i, p), y = vv(i, q);
          vv(i, p) = c * x + jqp * y;
          vv(i, q) = jpq * x + c * y;
        }
      }
    if (!rotated) break;
  }
  std::vector<double> sig(static_cast<size_t>(n));
  for (int64_t j = 0; j < n; ++j) {
    double a = 0.0;
    for (int64_t i = 0; i < rows; ++i) a += std::norm(w(i, j));
    sig[static_cast<size_t>(j)] = std::sqrt(a);
  }
  std::vector<int64_t> order(static_cast<size_t>(n));
  for (int64_t j = 0; j < n; ++j) order[static_cast<size_t>(j)] = j;
  std::stable_sort(order.begin(), order.end(),
                   [&](int64_t x, int64_t y) { return sig[static_cast<size_t>(x)] > sig[static_cast<size_t>(y)]; });
  u = CMat(rows, n);
  v = CMat(n, n);
  s.assign(static_cast<size_t>(n), 0.0);
  for (int64_t k = 0; k < n; ++k) {
    const int64_t o = order[static_cast<size_t>(k)];
    const double sg = sig[static_cast<size_t>(o)];
    s[static_cast<size_t>(k)] = sg;
    for (int64_t i = 0; i < rows; ++i) u(i, k) = sg > 0.0 ? w(i, o) / sg : cd(0.0);
    for (int64_t i = 0; i < n; ++i) v(i, k) = vv(i, o);
  }
}

// thin SVD of any shape: U (rows x k), s (k), V (cols x k), k = min(rows, cols)
void jsvd(const CMat& m, CMat& u, std::vector<double>& s, CMat& v) {
  if (m.rows >= m.cols) jsvd_tall(m, u, s, v);
  else jsvd_tall(adj(m), v, s, u);
}

double fro2(const std::vector<cd>& x) {
  double s = 0.0;
  for (const cd& e : x) s += std::norm(e);
  return s;
}

// cp_ls_update (decomp.hpp:200-219) for the factor of mode q (0..2):
// rhs(i_q, l) = sum over the other two indices of T conj(fa(., l) fb(., l)),
// gram = (fa^H fa) .* (fb^H fb), f_q = rhs conj(pinv(gram))
CMat ls_update(const std::vector<cd>& T, const int64_t d[3], int q, const CMat f[3], int64_t r) {
  const int a = q == 0 ? 1 : 0, b = q == 2 ? 1 : 2;  // the other modes, a < b
  const CMat& fa = f[a];
  const CMat& fb = f[b];
  CMat rhs(d[q], r);
  for (int64_t k = 0; k < d[2]; ++k)
    for (int64_t j = 0; j < d[1]; ++j)
      for (int64_t i = 0; i < d[0]; ++i) {
        const cd t = T[static_cast<size_t>(i + d[0] * (j + d[1] * k))];
        if (t == cd(0.0)) continue;
        const int64_t idx[3] = {i, j, k};
        const int64_t iq = idx[q], ia = idx[a], ib = idx[b];
        for (int64_t l = 0; l < r; ++l) rhs(iq, l) += t * std::conj(fa(ia, l) * fb(ib, l));
      }
  CMat gram(r, r);
  for (int64_t m = 0; m < r; ++m)
    for (int64_t l = 0; l < r; ++l) {
      cd ga = 0.0, gb = 0.0;
      for (int64_t i = 0; i < fa.rows; ++i) ga += std::conj(fa(i, l)) * fa(i, m);
      for (int64_t i = 0; i < fb.rows; ++i) gb += std::conj(fb(i, l)) * fb(i, m);
      gram(l, m) = ga * gb;
    }
  CMat u, v;
  std::vector<double> s;
  jsvd(gram, u, s, v);
  const double cutoff = (s.empty() ? 0.0 : s[0]) * 1e-12;
  CMat pc(r, r);  // conj(V diag(1/s) U^H)
  for (size_t j = 0; j < s.size(); ++j) {
    if (!(s[j] > cutoff)) continue;
    const double inv = 1.0 / s[j];
    for (int64_t col = 0; col < r; ++col) {
      const cd uc = std::conj(u(col, static_cast<int64_t>(j))) * inv;
      for (int64_t row = 0; row < r; ++row) pc(row, col) += v(row, static_cast<int64_t>(j)) * uc;
    }
  }
  for (cd& x : pc.a) x = std::conj(x);
  CMat out(d[q], r);
  for (int64_t col = 0; col < r; ++col)
    for (int64_t k = 0; k < r; ++k) {
      const cd p = pc(k, col);
      if (p == cd(0.0)) continue;
      for (int64_t i = 0; i < d[q]; ++i) out(i, col) += rhs(i, k) * p;
    }
  return out;
}

}  // namespace

CpAlsHost cp_als_host(const double2* t_in, const int64_t d[3], int64_t r, int max_iters, double stall_tol,
                      uint64_t seed) {
  if (r < 0) throw std::invalid_argument("cp_als: rank must be >= 0");
  if (max_iters < 1) throw std::invalid_argument("cp_als: max_iters must be >= 1");
  const int64_t n = d[0] * d[1] * d[2];
  std::vector<cd> T(static_cast<size_t>(n));
  for (int64_t e = 0; e < n; ++e) T[static_cast<size_t>(e)] = cd(t_in[e].x, t_in[e].y);
  CpAlsHost res;
  const double tnorm = std::sqrt(fro2(T));
  int64_t sorted[3] = {d[0], d[1], d[2]};
  std::sort(sorted, sorted + 3);
  res.ill_posed = r > sorted[0] * sorted[1];
  CMat f[3];
  auto export_factors = [&] {
    for (int q = 0; q < 3; ++q) {
      res.f[q].resize(f[q].a.size());
      for (size_t e = 0; e < f[q].a.size(); ++e) res.f[q][e] = make_double2(f[q].a[e].real(), f[q].a[e].imag());
    }
  };
  if (r == 0 || tnorm == 0.0) {
    for (int q = 0; q < 3; ++q) f[q] = CMat(d[q], r);
    export_factors();
    res.trace.push_back(tnorm == 0.0 ? 0.0 : 1.0);
    res.converged = tnorm == 0.0;
    return res;
  }
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  for (int q = 0; q < 3; ++q) {
    // mode-q unfolding (tensor.hpp:81-98); only its left singular vectors are used
    const int a = q == 0 ? 1 : 0, b = q == 2 ? 1 : 2;
    CMat unf(d[q], d[a] * d[b]);
    for (int64_t k = 0; k < d[2]; ++k)
      for (int64_t j = 0; j < d[1]; ++j)
        for (int64_t i = 0; i < d[0]; ++i) {
          const int64_t idx[3] = {i, j, k};
          unf(idx[q], idx[a] + d[a] * idx[b]) = T[static_cast<size_t>(i + d[0] * (j + d[1] * k))];
        }
    CMat u, v;
    std::vector<double> s;
    jsvd(unf, u, s, v);
    const int64_t have = std::min<int64_t>(u.cols, r);
    f[q] = CMat(d[q], r);
    for (int64_t l = 0; l < have; ++l)
      for (int64_t i = 0; i < d[q]; ++i) f[q](i, l) = u(i, l);
    for (int64_t l = have; l < r; ++l) {
      for (int64_t i = 0; i < d[q]; ++i) f[q](i, l) = cd(gauss(rng), gauss(rng));
      double nn = 0.0;
      for (int64_t i = 0; i < d[q]; ++i) nn += std::norm(f[q](i, l));
      nn = std::sqrt(nn);
      if (nn > 0)
        for (int64_t i = 0; i < d[q]; ++i) f[q](i, l) /= nn;
    }
  }
  double prev = std::numeric_limits<double>::infinity();
  std::vector<cd> rec(static_cast<size_t>(n));
  for (int sweep = 0; sweep < max_iters; ++sweep) {
    for (int q = 0; q < 3; ++q) f[q] = ls_update(T, d, q, f, r);
    for (int64_t l = 0; l < r; ++l) {  // cp_normalize_columns (decomp.hpp:221-230)
      double nq[3];
      for (int q = 0; q < 3; ++q) {
        double s = 0.0;
        for (int64_t i = 0; i < d[q]; ++i) s += std::norm(f[q](i, l));
        nq[q] = std::sqrt(s);
      }
      const double mag = std::cbrt(nq[0] * nq[1] * nq[2]);
      for (int q = 0; q < 3; ++q)
        if (nq[q] > 0)
          for (int64_t i = 0; i < d[q]; ++i) f[q](i, l) *= mag / nq[q];
    }
    double e2 = 0.0;  // ||cp_reconstruct(f) - t|| / ||t||
    for (int64_t k = 0; k < d[2]; ++k)
      for (int64_t j = 0; j < d[1]; ++j)
        for (int64_t i = 0; i < d[0]; ++i) {
          cd x = 0.0;
          for (int64_t l = 0; l < r; ++l) x += f[0](i, l) * f[1](j, l) * f[2](k, l);
          e2 += std::norm(x - T[static_cast<size_t>(i + d[0] * (j + d[1] * k))]);
        }
    const double err = std::sqrt(e2) / tnorm;
    res.trace.push_back(err);
    if (prev - err < stall_tol) {
      res.converged = err <= prev + stall_tol;
      break;
    }
    prev = err;
  }
  export_factors();
  return res;
}

}  // namespace vie
