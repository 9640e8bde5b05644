// C++ parity tests of the drop-in wrapper (include/vie_b200.hpp), written the
// way the reference's GTest suites are (test_fft_operator.cpp, test_solver.cpp),
// with the CPU oracle (oracle/vie_oracle.h, test infrastructure) as checker.
// Prints one PASS/FAIL line per test; exit code = number of failures.
#include <cmath>
#include <complex>
#include <cstdio>
#include <functional>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "vie_b200.hpp"
#include "vie_oracle.h"

using namespace vie::b200;

namespace {

int g_fail = 0;

void run(const char* name, const std::function<void()>& fn) {
  try {
    fn();
    std::printf("PASS %s\n", name);
  } catch (const std::exception& e) {
    std::printf("FAIL %s: %s\n", name, e.what());
    ++g_fail;
  }
}

void expect(bool ok, const std::string& msg) {
  if (!ok) throw std::runtime_error(msg);
}

// test_util.hpp:17-24 recipe
FactorMatrix random_matrix(Index rows, Index cols, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  FactorMatrix m(rows, cols);
  for (Index j = 0; j < cols; ++j)
    for (Index i = 0; i < rows; ++i) m(i, j) = cplx(gauss(rng), gauss(rng));
  return m;
}

// spatial Tucker form with the parity-zero rows (test_fft_operator.cpp:17-26)
TuckerForm random_form(const std::array<Index, 3>& d, Index r, const Parity& p, std::uint64_t seed) {
  TuckerForm f;
  f.core = Tensor3(r, r, r);
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  for (auto& v : f.core.data) v = cplx(gauss(rng), gauss(rng));
  for (int q = 0; q < 3; ++q) {
    f.factors[q] = random_matrix(d[q], r, seed + 1 + q);
    if (p.sign[q] < 0)
      for (Index c = 0; c < r; ++c) f.factors[q](0, c) = 0.0;
  }
  f.ranks = {r, r, r};
  return f;
}

CurrentField random_field(const std::array<Index, 3>& d, BasisOrder b, std::uint64_t seed) {
  CurrentField x(d, b);
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  for (auto& t : x.comp)
    for (auto& v : t.data) v = cplx(gauss(rng), gauss(rng));
  return x;
}

double rel(const std::vector<cplx>& a, const std::vector<cplx>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num += std::norm(a[i] - b[i]);
    den += std::norm(a[i]);
  }
  return std::sqrt(num / (den > 0 ? den : 1.0));
}

struct OracleForms {  // transformed (Fourier) factors for the oracle
  std::vector<int64_t> ranks;
  std::vector<std::vector<cplx>> cores, u1, u2, u3;
  std::vector<const double*> pc, p1, p2, p3;
};

OracleForms to_oracle(const std::vector<std::pair<KernelComponent, TuckerForm>>& forms, BasisOrder order) {
  OracleForms o;
  for (const auto& [comp, f] : forms) {
    const Parity p = component_parity(comp, order);
    o.ranks.insert(o.ranks.end(), {f.ranks[0], f.ranks[1], f.ranks[2]});
    o.cores.push_back(f.core.data);
    std::vector<cplx>* dst[3] = {nullptr, nullptr, nullptr};
    o.u1.emplace_back();
    o.u2.emplace_back();
    o.u3.emplace_back();
    dst[0] = &o.u1.back();
    dst[1] = &o.u2.back();
    dst[2] = &o.u3.back();
    for (int q = 0; q < 3; ++q) {
      const FactorMatrix& u = f.factors[q];
      dst[q]->resize(static_cast<size_t>(2 * u.rows * u.cols));
      if (orc_transform_factor(reinterpret_cast<const double*>(u.data.data()), u.rows, u.cols, p.sign[q],
                               reinterpret_cast<double*>(dst[q]->data())))
        throw std::runtime_error(orc_last_error());
    }
  }
  for (size_t c = 0; c < o.cores.size(); ++c) {
    o.pc.push_back(reinterpret_cast<const double*>(o.cores[c].data()));
    o.p1.push_back(reinterpret_cast<const double*>(o.u1[c].data()));
    o.p2.push_back(reinterpret_cast<const double*>(o.u2[c].data()));
    o.p3.push_back(reinterpret_cast<const double*>(o.u3[c].data()));
  }
  return o;
}

std::vector<std::pair<KernelComponent, TuckerForm>> make_family(OperatorKind k, BasisOrder b,
                                                                 const std::array<Index, 3>& d, Index r,
                                                                 std::uint64_t seed) {
  std::vector<std::pair<KernelComponent, TuckerForm>> out;
  for (const auto& c : unique_components(k, b)) out.emplace_back(c, random_form(d, r, component_parity(c, b), ++seed));
  return out;
}

}  // namespace

int main() {
  DftService dft(0);

  for (auto [k, b] : {std::pair{OperatorKind::N, BasisOrder::PWC}, std::pair{OperatorKind::K, BasisOrder::PWC},
                      std::pair{OperatorKind::N, BasisOrder::PWL}, std::pair{OperatorKind::K, BasisOrder::PWL}}) {
    const std::string name = std::string("ApplyOperator.MatchesOracle.") + (k == OperatorKind::N ? "N" : "K") +
                             (b == BasisOrder::PWC ? "pwc" : "pwl");
    run(name.c_str(), [&, k = k, b = b] {
      const std::array<Index, 3> d{3, 4, 5};
      auto fam = make_family(k, b, d, 3, 30);
      EmbeddedSpectrum op = build_operator_spectra(k, b, fam, dft);
      OracleForms of = to_oracle(fam, b);
      ApplyWorkspace ws;
      for (int trial = 0; trial < 3; ++trial) {
        CurrentField x = random_field(d, b, 40 + 3 * trial);
        CurrentField y = apply_operator(op, x, MatvecStrategy::HosvdDecompress, ScratchPolicy::WithBuffer, &ws, dft);
        const std::vector<cplx> xv = x.to_vector();
        std::vector<cplx> yref(xv.size());
        const int64_t g[3] = {d[0], d[1], d[2]};
        if (orc_apply_operator_tucker(static_cast<int>(k), static_cast<int>(b), g, of.ranks.data(), of.pc.data(),
                                      of.p1.data(), of.p2.data(), of.p3.data(),
                                      reinterpret_cast<const double*>(xv.data()), reinterpret_cast<double*>(yref.data())))
          throw std::runtime_error(orc_last_error());
        const double e = rel(yref, y.to_vector());
        expect(e <= 1e-10, "rel err " + std::to_string(e));
      }
    });
  }

  run("ApplyOperator.BatchEqualsSingleCalls", [&] {
    const std::array<Index, 3> d{4, 3, 5};
    auto fam = make_family(OperatorKind::N, BasisOrder::PWL, d, 2, 90);
    EmbeddedSpectrum op = build_operator_spectra(OperatorKind::N, BasisOrder::PWL, fam, dft);
    std::vector<CurrentField> xs;
    for (int i = 0; i < 3; ++i) xs.push_back(random_field(d, BasisOrder::PWL, 91 + i));
    const std::vector<CurrentField> ys = apply_operator_batch(op, xs);
    expect(ys.size() == xs.size(), "batch size");
    for (size_t i = 0; i < xs.size(); ++i) {
      CurrentField y = apply_operator(op, xs[i], MatvecStrategy::HosvdDecompress, ScratchPolicy::WithBuffer, nullptr, dft);
      const double e = rel(y.to_vector(), ys[i].to_vector());
      expect(e == 0.0, "batch vs single rel err " + std::to_string(e));
    }
  });

  run("BuildOperatorSpectra.FromTensors.ErrorTracksTolerance", [&] {  // test_fft_operator.cpp:192-209
    const std::array<Index, 3> d{4, 4, 4};
    std::vector<std::pair<KernelComponent, Tensor3>> tensors;
    std::vector<std::vector<cplx>> spec;  // oracle dense spectra
    std::uint64_t seed = 70;
    for (const auto& c : unique_components(OperatorKind::N)) {
      // rank-2 separable component with parity-zero rows (make_component_tensor)
      const Parity p = component_parity(c);
      Tensor3 t(d[0], d[1], d[2]);
      ++seed;
      FactorMatrix f[3];
      for (int q = 0; q < 3; ++q) {
        f[q] = random_matrix(d[q], 2, seed + 7 * q);
        if (p.sign[q] < 0)
          for (Index l = 0; l < 2; ++l) f[q](0, l) = 0.0;
      }
      for (Index k = 0; k < d[2]; ++k)
        for (Index j = 0; j < d[1]; ++j)
          for (Index i = 0; i < d[0]; ++i)
            for (Index l = 0; l < 2; ++l) t(i, j, k) += f[0](i, l) * f[1](j, l) * f[2](k, l);
      tensors.emplace_back(c, t);
      std::vector<cplx> sp(static_cast<size_t>(8 * t.size()));
      const int64_t dims[3] = {d[0], d[1], d[2]};
      if (orc_dense_spectrum(reinterpret_cast<const double*>(t.data.data()), dims, p.sign.data(),
                             reinterpret_cast<double*>(sp.data())))
        throw std::runtime_error(orc_last_error());
      spec.push_back(std::move(sp));
    }
    SpectrumBuildOptions opts;
    opts.tol = 1e-4;
    EmbeddedSpectrum op = build_operator_spectra(OperatorKind::N, tensors, opts, dft);
    CurrentField x = random_field(d, BasisOrder::PWC, 71);
    CurrentField y = apply_operator(op, x, MatvecStrategy::HosvdDecompress, ScratchPolicy::WithBuffer, nullptr, dft);
    std::vector<const double*> sp;
    for (auto& v : spec) sp.push_back(reinterpret_cast<const double*>(v.data()));
    const std::vector<cplx> xv = x.to_vector();
    std::vector<cplx> yref(xv.size());
    const int64_t g[3] = {d[0], d[1], d[2]};
    if (orc_apply_operator_dense(0, 0, g, sp.data(), reinterpret_cast<const double*>(xv.data()),
                                 reinterpret_cast<double*>(yref.data())))
      throw std::runtime_error(orc_last_error());
    const double e = rel(yref, y.to_vector());
    expect(e < 10 * opts.tol, "rel err " + std::to_string(e));
  });

  run("ApplyOperator.ScratchPolicyErrors", [&] {  // test_fft_operator.cpp:265-284
    const std::array<Index, 3> d{2, 2, 2};
    auto fam = make_family(OperatorKind::N, BasisOrder::PWC, d, 2, 95);
    EmbeddedSpectrum op = build_operator_spectra(OperatorKind::N, BasisOrder::PWC, fam, dft);
    CurrentField x = random_field(d, BasisOrder::PWC, 96);
    bool thrown = false;
    try {
      apply_operator(op, x, MatvecStrategy::HosvdDecompress, ScratchPolicy::NoBuffer, nullptr, dft);
    } catch (const std::invalid_argument&) {
      thrown = true;
    }
    expect(thrown, "NoBuffer with a decompress strategy must throw");
    thrown = false;
    try {
      apply_operator(op, random_field({2, 2, 3}, BasisOrder::PWC, 1), MatvecStrategy::HosvdDecompress,
                     ScratchPolicy::WithBuffer, nullptr, dft);
    } catch (const std::invalid_argument&) {
      thrown = true;
    }
    expect(thrown, "dim mismatch must throw");
  });

  run("ApplyOperator.ZeroInputGivesZero", [&] {  // test_fft_operator.cpp:121-130
    const std::array<Index, 3> d{3, 3, 4};
    auto fam = make_family(OperatorKind::N, BasisOrder::PWC, d, 2, 20);
    EmbeddedSpectrum op = build_operator_spectra(OperatorKind::N, BasisOrder::PWC, fam, dft);
    CurrentField y = apply_operator(op, CurrentField(d), MatvecStrategy::HosvdDecompress, ScratchPolicy::WithBuffer,
                                    nullptr, dft);
    double n = 0;
    for (auto v : y.to_vector()) n += std::norm(v);
    expect(n == 0.0, "nonzero output");
  });

  run("ApplySystem.MatchesOracle", [&] {  // test_solver.cpp:153-180
    const std::array<Index, 3> d{4, 3, 5};
    auto fam = make_family(OperatorKind::N, BasisOrder::PWC, d, 3, 17);
    EmbeddedSpectrum op = build_operator_spectra(OperatorKind::N, BasisOrder::PWC, fam, dft);
    OracleForms of = to_oracle(fam, BasisOrder::PWC);
    std::vector<cplx> eps(static_cast<size_t>(op.n_vox()));
    for (size_t i = 0; i < eps.size(); ++i) eps[i] = cplx(2.0 + 0.1 * static_cast<double>(i % 7), -0.3);
    CurrentField x = random_field(d, BasisOrder::PWC, 20);
    CurrentField y = apply_system(eps, 0.37, op, x);
    const std::vector<cplx> xv = x.to_vector();
    std::vector<cplx> yref(xv.size());
    const int64_t g[3] = {d[0], d[1], d[2]};
    if (orc_apply_system_tucker(0, g, of.ranks.data(), of.pc.data(), of.p1.data(), of.p2.data(), of.p3.data(),
                                reinterpret_cast<const double*>(eps.data()), 0.37,
                                reinterpret_cast<const double*>(xv.data()), reinterpret_cast<double*>(yref.data())))
      throw std::runtime_error(orc_last_error());
    expect(rel(yref, y.to_vector()) <= 1e-10, "rel err");
  });

  run("Gmres.MatchesOracle", [&] {  // iterations +-1, final residual within 1e-8
    const std::array<Index, 3> d{5, 4, 4};
    auto fam = make_family(OperatorKind::N, BasisOrder::PWC, d, 3, 77);
    for (auto& pr : fam)
      for (auto& v : pr.second.core.data) v *= 1e-4;
    EmbeddedSpectrum op = build_operator_spectra(OperatorKind::N, BasisOrder::PWC, fam, dft);
    OracleForms of = to_oracle(fam, BasisOrder::PWC);
    std::vector<cplx> eps(static_cast<size_t>(op.n_vox()));
    for (size_t i = 0; i < eps.size(); ++i) eps[i] = cplx(2.0 + 3.0 * static_cast<double>(i % 5) / 5.0, -0.5);
    const std::vector<cplx> rhs = random_field(d, BasisOrder::PWC, 78).to_vector();
    GmresConfig cfg{1e-8, 8, 20};
    GmresResult r = gmres_system(eps, 1.0, op, rhs, cfg);
    std::vector<cplx> xref(rhs.size());
    std::vector<double> hist(200);
    int it = 0, cv = 0, hl = 0;
    double fr = 0;
    const int64_t g[3] = {d[0], d[1], d[2]};
    if (orc_gmres_system_tucker(0, g, of.ranks.data(), of.pc.data(), of.p1.data(), of.p2.data(), of.p3.data(),
                                reinterpret_cast<const double*>(eps.data()), 1.0,
                                reinterpret_cast<const double*>(rhs.data()), nullptr, 1e-8, 8, 20,
                                reinterpret_cast<double*>(xref.data()), &it, &cv, &fr, hist.data(), 200, &hl))
      throw std::runtime_error(orc_last_error());
    expect(r.converged && cv, "not converged");
    expect(std::abs(r.iterations - it) <= 1, "iterations " + std::to_string(r.iterations) + " vs " + std::to_string(it));
    expect(std::abs(r.final_relative_residual - fr) <= 1e-8, "final residual");
    bool thrown = false;
    try {
      gmres_system(eps, 1.0, op, rhs, GmresConfig{1e-5, 0, 1});
    } catch (const std::invalid_argument&) {
      thrown = true;
    }
    expect(thrown, "invalid config must throw");
  });

  // solve_scene stages (solver.hpp:148-285) through the wrapper vs the oracle
  run("SceneStages.MatchOracle", [&] {
    VoxelGrid g{{5, 4, 6}, {0.004, 0.004, 0.004}, {-0.01, 0.0, 0.02}};
    DielectricMap m(g, 2.98e8);
    for (Index k = 1; k < 5; ++k)
      for (Index j = 1; j < 3; ++j)
        for (Index i = 1; i < 4; ++i) m.set_voxel(i, j, k, 40.0 + i, 0.5);
    PlaneWave inc{{0.0, 1.0, -1.0}, {0.0, 1.0, 1.0}, 2.0};
    const double geo[6] = {0.004, 0.004, 0.004, -0.01, 0.0, 0.02};
    const double pw[7] = {0.0, 1.0, -1.0, 0.0, 1.0, 1.0, 2.0};
    const int64_t dims[3] = {5, 4, 6};
    const size_t nv = m.eps_r.size();
    auto rel_err = [](const std::vector<cplx>& a, const std::vector<cplx>& b) {
      double num = 0.0, den = 0.0;
      for (size_t i = 0; i < a.size(); ++i) {
        num += std::norm(a[i] - b[i]);
        den += std::norm(b[i]);
      }
      return std::sqrt(num / den);
    };
    for (int quad : {1, 3}) {
      const std::vector<cplx> rhs = build_rhs(m, inc, quad).to_vector();
      std::vector<cplx> ref(3 * nv);
      if (orc_build_rhs(dims, geo, 2.98e8, pw, reinterpret_cast<const double*>(m.eps_r.data()), quad,
                        reinterpret_cast<double*>(ref.data())))
        throw std::runtime_error(orc_last_error());
      expect(rel_err(rhs, ref) <= 1e-13, "build_rhs quad " + std::to_string(quad));
    }
    CurrentField j(g.dims), h(g.dims);
    for (int q = 0; q < 3; ++q) {
      j.comp[q] = Tensor3(5, 4, 6);
      h.comp[q] = Tensor3(5, 4, 6);
      if (orc_random_tensor(5, 4, 6, 90 + q, reinterpret_cast<double*>(j.comp[q].data.data())) ||
          orc_random_tensor(5, 4, 6, 95 + q, reinterpret_cast<double*>(h.comp[q].data.data())))
        throw std::runtime_error(orc_last_error());
    }
    Fields f = recover_fields(j, m, inc, nullptr);
    expect(!f.has_h, "no K operator, no h");
    const std::vector<cplx> jv = j.to_vector();
    std::vector<cplx> eref(3 * nv);
    if (orc_recover_fields(dims, geo, 2.98e8, pw, reinterpret_cast<const double*>(m.eps_r.data()),
                           reinterpret_cast<const double*>(jv.data()), nullptr,
                           reinterpret_cast<double*>(eref.data()), nullptr))
      throw std::runtime_error(orc_last_error());
    expect(rel_err(f.e.to_vector(), eref) <= 1e-13, "recover_fields e");
    f.h = h;
    f.has_h = true;
    PostProcess pp = postprocess(f, m);
    const std::vector<cplx> hv = h.to_vector();
    std::vector<double> pref(nv), bref(nv);
    double tref = 0.0;
    if (orc_postprocess(dims, geo, 2.98e8, reinterpret_cast<const double*>(m.eps_r.data()),
                        reinterpret_cast<const double*>(eref.data()), reinterpret_cast<const double*>(hv.data()),
                        pref.data(), bref.data(), &tref))
      throw std::runtime_error(orc_last_error());
    for (size_t v = 0; v < nv; ++v) {
      expect(std::abs(pp.p_abs[v] - pref[v]) <= 1e-12 * std::abs(pref[v]) + 1e-300, "p_abs");
      expect(std::abs(pp.b1_plus[v] - bref[v]) <= 1e-12 * bref[v], "b1_plus");
    }
    expect(std::abs(pp.total_absorbed_power - tref) <= 1e-12 * std::abs(tref), "total power");
    bool thrown = false;
    try {
      build_rhs(m, PlaneWave{{1.0, 0.0, 1.0}, {0.0, 0.0, 1.0}, 1.0});
    } catch (const std::invalid_argument&) {
      thrown = true;
    }
    expect(thrown, "non-orthogonal plane wave must throw");
  });

  // Tucker+CP components through the wrapper: equal to the Tucker path with the
  // superdiagonal core (decomp.hpp:143-148, operator.hpp:248-261)
  run("ApplyOperator.TuckerCpEqualsSuperdiagonalTucker", [&] {
    const std::array<Index, 3> d{4, 5, 3};
    const Index R = 3;
    std::vector<std::pair<KernelComponent, TuckerCPForm>> cp;
    std::vector<std::pair<KernelComponent, TuckerForm>> tk;
    std::uint64_t seed = 500;
    for (const auto& c : unique_components(OperatorKind::N, BasisOrder::PWC)) {
      const Parity p = component_parity(c, BasisOrder::PWC);
      TuckerCPForm f;
      f.rank = R;
      TuckerForm t;
      t.core = Tensor3(R, R, R);
      for (Index l = 0; l < R; ++l) t.core(l, l, l) = 1.0;
      for (int q = 0; q < 3; ++q) {
        f.factors[q] = random_matrix(d[q], R, ++seed);
        if (p.sign[q] < 0)
          for (Index l = 0; l < R; ++l) f.factors[q](0, l) = 0.0;
        t.factors[q] = f.factors[q];
      }
      t.ranks = {R, R, R};
      cp.emplace_back(c, f);
      tk.emplace_back(c, t);
    }
    EmbeddedSpectrum a = build_operator_spectra(OperatorKind::N, BasisOrder::PWC, cp, dft);
    EmbeddedSpectrum b = build_operator_spectra(OperatorKind::N, BasisOrder::PWC, tk, dft);
    CurrentField x(d);
    for (int q = 0; q < 3; ++q) {
      x.comp[q] = Tensor3(d[0], d[1], d[2]);
      if (orc_random_tensor(d[0], d[1], d[2], 600 + q, reinterpret_cast<double*>(x.comp[q].data.data())))
        throw std::runtime_error(orc_last_error());
    }
    ApplyWorkspace ws;
    const std::vector<cplx> ya = apply_operator(a, x, MatvecStrategy::HosvdDecompress, ScratchPolicy::WithBuffer, &ws, dft).to_vector();
    const std::vector<cplx> yb = apply_operator(b, x, MatvecStrategy::HosvdDecompress, ScratchPolicy::WithBuffer, &ws, dft).to_vector();
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < ya.size(); ++i) {
      num += std::norm(ya[i] - yb[i]);
      den += std::norm(yb[i]);
    }
    expect(std::sqrt(num / den) <= 1e-13, "CP vs superdiagonal Tucker");
  });

  // tucker_cp / cp_als through the wrapper (decomp.hpp:237-373) vs the oracle restatement
  run("TuckerCp.MatchesOracle", [&] {
    const int64_t d[3] = {7, 6, 5};
    Tensor3 t(d[0], d[1], d[2]);
    if (orc_random_tensor(d[0], d[1], d[2], 77, reinterpret_cast<double*>(t.data.data())))
      throw std::runtime_error(orc_last_error());
    const TuckerCpResult a = tucker_cp(t, 0.3, 60, TruncationRule::Energy, -1, 0.0, dft);
    int64_t rk = 0;
    double errs[3];
    int nt = 0;
    if (orc_tucker_cp(reinterpret_cast<const double*>(t.data.data()), d, 0.3, 60, VIE_RULE_ENERGY, -1, 0.0, &rk,
                      nullptr, nullptr, nullptr, errs, nullptr, 0, &nt))
      throw std::runtime_error(orc_last_error());
    expect(a.form.rank == rk, "tucker_cp rank");
    std::vector<double> w(static_cast<size_t>(2 * (d[0] + d[1] + d[2]) * rk));
    std::vector<double> tr(61);
    if (orc_tucker_cp(reinterpret_cast<const double*>(t.data.data()), d, 0.3, 60, VIE_RULE_ENERGY, -1, 0.0, &rk,
                      w.data(), w.data() + 2 * d[0] * rk, w.data() + 2 * (d[0] + d[1]) * rk, errs, tr.data(), 61, &nt))
      throw std::runtime_error(orc_last_error());
    expect(static_cast<int>(a.cp_error_trace.size()) == nt, "tucker_cp sweeps");
    for (int i = 0; i < nt; ++i) expect(std::abs(a.cp_error_trace[i] - tr[i]) <= 1e-8, "tucker_cp trace");
    expect(std::abs(a.hosvd_relative_error - errs[0]) <= 1e-9, "hosvd error");
    expect(std::abs(a.stats.achieved_relative_error - errs[2]) <= 1e-9, "achieved error");
    const CpAlsResult c = cp_als(t, 3, 30, 0.0);
    expect(c.rel_error_trace.size() == 30 && !c.ill_posed_rank, "cp_als sweeps");
    SpectrumBuildOptions opts;
    opts.tucker_cp = true;
    opts.tol = 1e-6;
    opts.cp_iters = 100;
    std::vector<std::pair<KernelComponent, Tensor3>> tens;
    const std::array<Index, 3> g{4, 5, 3};
    std::uint64_t seed = 900;
    for (const auto& comp : unique_components(OperatorKind::N, BasisOrder::PWC)) {
      const Parity p = component_parity(comp, BasisOrder::PWC);
      Tensor3 x(g[0], g[1], g[2]);
      FactorMatrix f[3];
      for (int q = 0; q < 3; ++q) {
        f[q] = random_matrix(g[q], 2, ++seed);
        if (p.sign[q] < 0)
          for (Index l = 0; l < 2; ++l) f[q](0, l) = 0.0;
      }
      for (Index k = 0; k < g[2]; ++k)
        for (Index j = 0; j < g[1]; ++j)
          for (Index i = 0; i < g[0]; ++i)
            for (Index l = 0; l < 2; ++l) x(i, j, k) += f[0](i, l) * f[1](j, l) * f[2](k, l);
      tens.emplace_back(comp, x);
    }
    EmbeddedSpectrum op = build_operator_spectra(OperatorKind::N, tens, opts, dft);
    CurrentField xf(g);
    for (int q = 0; q < 3; ++q) {
      xf.comp[q] = Tensor3(g[0], g[1], g[2]);
      if (orc_random_tensor(g[0], g[1], g[2], 950 + q, reinterpret_cast<double*>(xf.comp[q].data.data())))
        throw std::runtime_error(orc_last_error());
    }
    ApplyWorkspace ws;
    const std::vector<cplx> y = apply_operator(op, xf, MatvecStrategy::TuckerCpDecompress, ScratchPolicy::WithBuffer, &ws, dft).to_vector();
    opts.tucker_cp = false;
    opts.tol = 1e-12;
    EmbeddedSpectrum opt = build_operator_spectra(OperatorKind::N, tens, opts, dft);
    const std::vector<cplx> yt = apply_operator(opt, xf, MatvecStrategy::HosvdDecompress, ScratchPolicy::WithBuffer, &ws, dft).to_vector();
    expect(rel(yt, y) <= 1e-6, "tucker_cp operator vs Tucker operator");
  });

  // solve_scene (solver.hpp:300-326) through the wrapper vs the oracle pipeline
  run("SolveScene.MatchesOraclePipeline", [&] {
    const std::array<Index, 3> d{5, 4, 4};
    auto famn = make_family(OperatorKind::N, BasisOrder::PWC, d, 3, 131);
    auto famk = make_family(OperatorKind::K, BasisOrder::PWC, d, 3, 171);
    for (auto* fam : {&famn, &famk})
      for (auto& pr : *fam)
        for (auto& v : pr.second.core.data) v *= 1e-4;
    EmbeddedSpectrum opn = build_operator_spectra(OperatorKind::N, BasisOrder::PWC, famn, dft);
    EmbeddedSpectrum opk = build_operator_spectra(OperatorKind::K, BasisOrder::PWC, famk, dft);
    OracleForms ofn = to_oracle(famn, BasisOrder::PWC), ofk = to_oracle(famk, BasisOrder::PWC);
    DielectricMap m(VoxelGrid{d, {1.0, 1.0, 1.0}, {0.0, 0.0, 0.0}}, 2.98e8);  // unit voxels: 1/V = 1
    for (size_t i = 0; i < m.eps_r.size(); ++i)
      if (i % 4) m.eps_r[i] = cplx(2.0 + 3.0 * static_cast<double>(i % 5) / 5.0, -0.5);
    PlaneWave inc{{0.0, 1.0, 0.0}, {1.0, 0.0, 0.0}, 2.0};
    SolveReport rep = solve_scene(m, inc, opn, &opk, GmresConfig{1e-10, 10, 20});

    const int64_t g[3] = {d[0], d[1], d[2]};
    const double geo[6] = {1.0, 1.0, 1.0, 0.0, 0.0, 0.0};
    const double pw[7] = {0.0, 1.0, 0.0, 1.0, 0.0, 0.0, 2.0};
    const size_t nv = m.eps_r.size();
    const double* eps = reinterpret_cast<const double*>(m.eps_r.data());
    std::vector<cplx> rhs(3 * nv), x(3 * nv), kj(3 * nv), e(3 * nv), h(3 * nv);
    std::vector<double> hist(400), p(nv), b1(nv);
    int it = 0, cv = 0, hl = 0;
    double fr = 0.0, tot = 0.0;
    if (orc_build_rhs(g, geo, 2.98e8, pw, eps, 1, reinterpret_cast<double*>(rhs.data())) ||
        orc_gmres_system_tucker(0, g, ofn.ranks.data(), ofn.pc.data(), ofn.p1.data(), ofn.p2.data(), ofn.p3.data(),
                                eps, 1.0, reinterpret_cast<const double*>(rhs.data()), nullptr, 1e-10, 10, 20,
                                reinterpret_cast<double*>(x.data()), &it, &cv, &fr, hist.data(), 400, &hl) ||
        orc_apply_operator_tucker(1, 0, g, ofk.ranks.data(), ofk.pc.data(), ofk.p1.data(), ofk.p2.data(),
                                  ofk.p3.data(), reinterpret_cast<const double*>(x.data()),
                                  reinterpret_cast<double*>(kj.data())) ||
        orc_recover_fields(g, geo, 2.98e8, pw, eps, reinterpret_cast<const double*>(x.data()),
                           reinterpret_cast<const double*>(kj.data()), reinterpret_cast<double*>(e.data()),
                           reinterpret_cast<double*>(h.data())) ||
        orc_postprocess(g, geo, 2.98e8, eps, reinterpret_cast<const double*>(e.data()),
                        reinterpret_cast<const double*>(h.data()), p.data(), b1.data(), &tot))
      throw std::runtime_error(orc_last_error());
    expect(rep.converged && cv, "not converged");
    expect(std::abs(rep.iterations - it) <= 1, "iterations");
    expect(std::abs(rep.final_relative_residual - fr) <= 1e-8, "final residual");
    expect(rel(x, rep.j.to_vector()) <= 1e-8, "j");
    expect(rel(e, rep.fields.e.to_vector()) <= 1e-8, "e");
    expect(rep.fields.has_h && rel(h, rep.fields.h.to_vector()) <= 1e-8, "h");
    expect(std::abs(rep.post.total_absorbed_power - tot) <= 1e-8 * std::abs(tot), "total power");
  });

  // ---- 64^3 at the BASELINE configs[1] grid (review round 1: the drop-in's copies were
  // unordered with the context stream; these sizes expose such races)
  run("ApplySystem.Pwl64.MatchesOracle", [&] {  // test_solver.cpp:153-180 at 64^3 PWL
    const std::array<Index, 3> d{64, 64, 64};
    auto fam = make_family(OperatorKind::N, BasisOrder::PWL, d, 4, 640);
    EmbeddedSpectrum op = build_operator_spectra(OperatorKind::N, BasisOrder::PWL, fam, dft);
    OracleForms of = to_oracle(fam, BasisOrder::PWL);
    std::vector<cplx> eps(static_cast<size_t>(op.n_vox()));
    for (size_t i = 0; i < eps.size(); ++i) eps[i] = cplx(2.0 + 0.1 * static_cast<double>(i % 7), -0.3);
    CurrentField x = random_field(d, BasisOrder::PWL, 641);
    CurrentField y = apply_system(eps, 0.37, op, x);
    const std::vector<cplx> xv = x.to_vector();
    std::vector<cplx> yref(xv.size());
    const int64_t g[3] = {d[0], d[1], d[2]};
    if (orc_apply_system_tucker(1, g, of.ranks.data(), of.pc.data(), of.p1.data(), of.p2.data(), of.p3.data(),
                                reinterpret_cast<const double*>(eps.data()), 0.37,
                                reinterpret_cast<const double*>(xv.data()), reinterpret_cast<double*>(yref.data())))
      throw std::runtime_error(orc_last_error());
    const double e = rel(yref, y.to_vector());
    expect(e <= 1e-10, "rel err " + std::to_string(e));
  });

  run("GmresSystem.Pwl64.HistoryMatchesOracle", [&] {  // solver.hpp:34-142, 6 Arnoldi steps
    const std::array<Index, 3> d{64, 64, 64};
    auto fam = make_family(OperatorKind::N, BasisOrder::PWL, d, 3, 650);
    for (auto& pr : fam)
      for (auto& v : pr.second.core.data) v *= 1e-3;
    EmbeddedSpectrum op = build_operator_spectra(OperatorKind::N, BasisOrder::PWL, fam, dft);
    OracleForms of = to_oracle(fam, BasisOrder::PWL);
    std::vector<cplx> eps(static_cast<size_t>(op.n_vox()));
    for (size_t i = 0; i < eps.size(); ++i) eps[i] = cplx(2.0 + 3.0 * static_cast<double>(i % 5) / 5.0, -0.5);
    const std::vector<cplx> rhs = random_field(d, BasisOrder::PWL, 651).to_vector();
    const GmresConfig cfg{1e-14, 6, 1};  // 6 iterations, not converged: compare the whole history
    GmresResult r = gmres_system(eps, 1.0, op, rhs, cfg);
    std::vector<cplx> xref(rhs.size());
    std::vector<double> hist(64);
    int it = 0, cv = 0, hl = 0;
    double fr = 0;
    const int64_t g[3] = {d[0], d[1], d[2]};
    if (orc_gmres_system_tucker(1, g, of.ranks.data(), of.pc.data(), of.p1.data(), of.p2.data(), of.p3.data(),
                                reinterpret_cast<const double*>(eps.data()), 1.0,
                                reinterpret_cast<const double*>(rhs.data()), nullptr, cfg.tolerance, cfg.inner,
                                cfg.outer, reinterpret_cast<double*>(xref.data()), &it, &cv, &fr, hist.data(), 64, &hl))
      throw std::runtime_error(orc_last_error());
    expect(r.iterations == it && static_cast<int>(r.residual_history.size()) == hl, "iterations");
    for (int i = 0; i < hl; ++i)
      expect(std::abs(r.residual_history[i] - hist[i]) <= 1e-10 * hist[i], "history " + std::to_string(i));
    expect(std::abs(r.final_relative_residual - fr) <= 1e-8 * fr, "final residual");
    expect(rel(xref, r.solution) <= 1e-10, "iterate");
  });

  run("RecoverFields.K64.MatchesOracle", [&] {  // solver.hpp:211-249 with the K operator, 64^3 PWC
    const std::array<Index, 3> d{64, 64, 64};
    auto famk = make_family(OperatorKind::K, BasisOrder::PWC, d, 4, 660);
    EmbeddedSpectrum opk = build_operator_spectra(OperatorKind::K, BasisOrder::PWC, famk, dft);
    OracleForms ofk = to_oracle(famk, BasisOrder::PWC);
    VoxelGrid vg{d, {0.002, 0.002, 0.002}, {-0.064, -0.064, -0.064}};
    DielectricMap m(vg, 2.98e8);
    for (Index k = 8; k < 56; ++k)
      for (Index j = 8; j < 56; ++j)
        for (Index i = 8; i < 56; ++i) m.set_voxel(i, j, k, 50.0, 0.6);
    PlaneWave inc{{1.0, 0.0, 0.0}, {0.0, 0.0, 1.0}, 1.0};
    const double geo[6] = {0.002, 0.002, 0.002, -0.064, -0.064, -0.064};
    const double pw[7] = {1.0, 0.0, 0.0, 0.0, 0.0, 1.0, 1.0};
    const int64_t g[3] = {d[0], d[1], d[2]};
    CurrentField j = random_field(d, BasisOrder::PWC, 661);
    Fields f = recover_fields(j, m, inc, &opk);
    const std::vector<cplx> jv = j.to_vector();
    const size_t nv = m.eps_r.size();
    std::vector<cplx> kj(3 * nv), e(3 * nv), h(3 * nv);
    if (orc_apply_operator_tucker(1, 0, g, ofk.ranks.data(), ofk.pc.data(), ofk.p1.data(), ofk.p2.data(),
                                  ofk.p3.data(), reinterpret_cast<const double*>(jv.data()),
                                  reinterpret_cast<double*>(kj.data())) ||
        orc_recover_fields(g, geo, 2.98e8, pw, reinterpret_cast<const double*>(m.eps_r.data()),
                           reinterpret_cast<const double*>(jv.data()), reinterpret_cast<const double*>(kj.data()),
                           reinterpret_cast<double*>(e.data()), reinterpret_cast<double*>(h.data())))
      throw std::runtime_error(orc_last_error());
    expect(f.has_h, "h with the K operator");
    expect(rel(e, f.e.to_vector()) <= 1e-12, "e");
    expect(rel(h, f.h.to_vector()) <= 1e-10, "h");
  });

  // ---- gmres(apply, rhs, cfg, x0, precond) known answers, restated from
  // test_solver.cpp:31-114 and test_scene_io.cpp:107-139 with the same seeded inputs
  // (test_util.hpp random_matrix == orc_random_matrix), on the device GMRES (vie_gmres)
  auto rmat = [](Index rows, Index cols, std::uint64_t seed) {
    std::vector<cplx> m(static_cast<size_t>(rows * cols));
    if (orc_random_matrix(rows, cols, seed, reinterpret_cast<double*>(m.data())))
      throw std::runtime_error(orc_last_error());
    return m;
  };
  auto dense = [](const std::vector<cplx>& a, Index n) {  // column-major n x n
    return [a, n](const std::vector<cplx>& v) {
      std::vector<cplx> o(static_cast<size_t>(n), cplx(0.0));
      for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i) o[i] += a[static_cast<size_t>(i + n * j)] * v[j];
      return o;
    };
  };
  auto diag_map = [](const std::vector<cplx>& d) {
    return [d](const std::vector<cplx>& v) {
      std::vector<cplx> o(v.size());
      for (size_t i = 0; i < v.size(); ++i) o[i] = d[i] * v[i];
      return o;
    };
  };
  auto norm_rel = [](const std::vector<cplx>& a, const std::vector<cplx>& b) {  // |a - b| / |b|
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < a.size(); ++i) {
      num += std::norm(a[i] - b[i]);
      den += std::norm(b[i]);
    }
    return std::sqrt(num / den);
  };
  run("Gmres.IdentityConvergesInOneIteration", [&] {  // test_solver.cpp:31-38
    const std::vector<cplx> rhs = rmat(20, 1, 1);
    GmresResult r = gmres([](const std::vector<cplx>& v) { return v; }, rhs, GmresConfig{}, nullptr, nullptr, &dft);
    expect(r.converged && r.iterations == 1, "iterations " + std::to_string(r.iterations));
    expect(norm_rel(r.solution, rhs) < 1e-12, "solution");
  });
  run("Gmres.DiagonalSystemMatchesDirectSolve", [&] {  // test_solver.cpp:40-53
    std::vector<cplx> d(10);
    for (int i = 0; i < 10; ++i) d[i] = cplx(i + 1.0, 0.5 * i);
    const std::vector<cplx> rhs = rmat(10, 1, 2);
    GmresConfig cfg;
    cfg.tolerance = 1e-12;
    GmresResult r = gmres(diag_map(d), rhs, cfg, nullptr, nullptr, &dft);
    std::vector<cplx> ex(10);
    for (int i = 0; i < 10; ++i) ex[i] = rhs[i] / d[i];
    expect(r.converged, "converged");
    expect(norm_rel(r.solution, ex) < 1e-10, "solution");
  });
  run("Gmres.RestartsReachTolerance", [&] {  // test_solver.cpp:55-68
    std::vector<cplx> a0 = rmat(30, 30, 3), a(900, cplx(0.0));
    for (int i = 0; i < 30; ++i)
      for (int j = 0; j < 30; ++j) {
        cplx acc = 0.0;
        for (int k = 0; k < 30; ++k) acc += a0[i + 30 * k] * std::conj(a0[j + 30 * k]);
        a[i + 30 * j] = acc / 30.0 + (i == j ? 4.0 : 0.0);
      }
    const std::vector<cplx> rhs = rmat(30, 1, 4);
    GmresConfig cfg{1e-9, 5, 100};
    GmresResult r = gmres(dense(a, 30), rhs, cfg, nullptr, nullptr, &dft);
    expect(r.converged, "converged");
    expect(norm_rel(dense(a, 30)(r.solution), rhs) <= 2e-9, "residual");
  });
  run("Gmres.ResidualHistoryMonotoneWithinCycle", [&] {  // test_solver.cpp:70-82
    std::vector<cplx> a = rmat(25, 25, 5);
    for (int i = 0; i < 25; ++i) a[i + 25 * i] += 6.0;
    GmresResult r = gmres(dense(a, 25), rmat(25, 1, 6), GmresConfig{1e-14, 25, 1}, nullptr, nullptr, &dft);
    for (size_t i = 1; i < r.residual_history.size(); ++i)
      expect(r.residual_history[i] <= r.residual_history[i - 1] * (1.0 + 1e-12), "monotone");
  });
  run("Gmres.ReportedResidualMatchesExternalRecomputation", [&] {  // test_solver.cpp:84-97
    std::vector<cplx> a = rmat(20, 20, 7);
    for (int i = 0; i < 20; ++i) a[i + 20 * i] += 5.0;
    const std::vector<cplx> rhs = rmat(20, 1, 8);
    GmresResult r = gmres(dense(a, 20), rhs, GmresConfig{1e-8, 50, 200}, nullptr, nullptr, &dft);
    expect(r.converged, "converged");
    const double ext = norm_rel(dense(a, 20)(r.solution), rhs);
    expect(std::abs(ext - r.final_relative_residual) <= 1e-10 * std::max(1.0, ext), "final residual");
    expect(std::abs(r.residual_history.back() - ext) <= 1e-10, "last Givens estimate");
  });
  run("Gmres.NonConvergenceReportedNotThrown", [&] {  // test_solver.cpp:99-114
    std::vector<cplx> a(1600, cplx(0.0));
    for (int i = 0; i < 39; ++i) a[(i + 1) + 40 * i] = 1.0;
    a[0 + 40 * 39] = 1.0;
    std::vector<cplx> rhs(40, cplx(0.0));
    rhs[0] = 1.0;
    GmresResult r = gmres(dense(a, 40), rhs, GmresConfig{1e-12, 3, 2}, nullptr, nullptr, &dft);
    expect(!r.converged && r.solution.size() == 40, "not converged, full-size iterate");
    bool thrown = false;
    try {
      std::vector<cplx> bad(rhs);
      bad[3] = cplx(std::nan(""), 0.0);
      gmres(dense(a, 40), bad, GmresConfig{}, nullptr, nullptr, &dft);
    } catch (const std::invalid_argument&) {
      thrown = true;
    }
    expect(thrown, "non-finite rhs must throw");
  });
  run("GmresHooks.WarmStartSkipsIterations", [&] {  // test_scene_io.cpp:107-121
    std::vector<cplx> d(8);
    for (int i = 0; i < 8; ++i) d[i] = cplx(2.0 + i, 0.3);
    const std::vector<cplx> rhs = rmat(8, 1, 1);
    GmresConfig cfg;
    cfg.tolerance = 1e-10;
    GmresResult cold = gmres(diag_map(d), rhs, cfg, nullptr, nullptr, &dft);
    expect(cold.converged, "cold");
    GmresResult warm = gmres(diag_map(d), rhs, cfg, &cold.solution, nullptr, &dft);
    expect(warm.converged && warm.iterations == 0, "warm start: 0 iterations");
  });
  run("GmresHooks.DiagonalRightPreconditionerConvergesImmediately", [&] {  // test_scene_io.cpp:123-139
    std::vector<cplx> d(12);
    for (int i = 0; i < 12; ++i) d[i] = cplx(1.0 + 3.0 * i, -0.5 * i);
    auto pre = [&](const std::vector<cplx>& v) {
      std::vector<cplx> o(v.size());
      for (size_t i = 0; i < v.size(); ++i) o[i] = v[i] / d[i];
      return o;
    };
    const std::vector<cplx> rhs = rmat(12, 1, 2);
    GmresConfig cfg;
    cfg.tolerance = 1e-12;
    GmresResult r = gmres(diag_map(d), rhs, cfg, nullptr, pre, &dft);
    expect(r.converged && r.iterations == 1, "1 iteration, got " + std::to_string(r.iterations));
    expect(norm_rel(diag_map(d)(r.solution), rhs) < 1e-12, "residual");
  });
  run("GmresSystem.DiagonalPreconditionerOnTheJvieSystem", [&] {
    // zero Tucker forms: N = 0, so apply_system is diag(eps g); M = diag(1 / (eps g)) -> 1 iteration
    const std::array<Index, 3> d{6, 5, 4};
    auto fam = make_family(OperatorKind::N, BasisOrder::PWL, d, 2, 700);
    for (auto& pr : fam)
      for (auto& v : pr.second.core.data) v = 0.0;
    EmbeddedSpectrum op = build_operator_spectra(OperatorKind::N, BasisOrder::PWL, fam, dft);
    const size_t nv = static_cast<size_t>(op.n_vox());
    std::vector<cplx> eps(nv), pdiag(12 * nv);
    for (size_t i = 0; i < nv; ++i) eps[i] = cplx(2.0 + 0.01 * static_cast<double>(i), -0.4);
    for (size_t s = 0; s < 12; ++s)
      for (size_t i = 0; i < nv; ++i) pdiag[s * nv + i] = 1.0 / (eps[i] * (s % 4 == 0 ? 1.0 : 1.0 / 12.0));
    const std::vector<cplx> rhs = random_field(d, BasisOrder::PWL, 701).to_vector();
    GmresResult plain = gmres_system(eps, 1.0, op, rhs, GmresConfig{1e-12, 50, 4});
    GmresResult pc = gmres_system(eps, 1.0, op, rhs, GmresConfig{1e-12, 50, 4}, nullptr, &pdiag);
    expect(pc.converged && pc.iterations == 1, "1 iteration, got " + std::to_string(pc.iterations));
    expect(plain.converged && plain.iterations > 1, "unpreconditioned needs more");
    expect(rel(plain.solution, pc.solution) <= 1e-10, "same solution");
  });

  run("ApplyOperator.TimingsAndMatvecBench", [&] {  // operator.hpp:189-192, 451-502
    const std::array<Index, 3> d{32, 32, 32};
    auto fam = make_family(OperatorKind::N, BasisOrder::PWL, d, 4, 710);
    EmbeddedSpectrum op = build_operator_spectra(OperatorKind::N, BasisOrder::PWL, fam, dft);
    CurrentField x = random_field(d, BasisOrder::PWL, 711);
    ApplyTimings t;
    const std::vector<cplx> a =
        apply_operator(op, x, MatvecStrategy::HosvdDecompress, ScratchPolicy::WithBuffer, nullptr, dft, &t).to_vector();
    const std::vector<cplx> b =
        apply_operator(op, x, MatvecStrategy::HosvdDecompress, ScratchPolicy::WithBuffer, nullptr, dft).to_vector();
    expect(t.fft_ms > 0.0 && t.product_ms > 0.0, "timings");
    expect(rel(a, b) == 0.0, "timed == untimed");
    MatvecBenchResult r = matvec_bench(op, x, MatvecStrategy::HosvdDecompress, 3, dft);
    expect(r.repetitions == 3 && r.median_ms > 0.0 && r.product_min_ms <= r.product_ms, "bench");
  });

  run("Lifetime.OperatorOutlivesItsDftService", [&] {  // EmbeddedSpectrum is self-contained (operator.hpp:118-119)
    const std::array<Index, 3> d{4, 4, 4};
    auto fam = make_family(OperatorKind::N, BasisOrder::PWC, d, 2, 720);
    std::unique_ptr<EmbeddedSpectrum> op;
    {
      DftService local(0);
      op.reset(new EmbeddedSpectrum(build_operator_spectra(OperatorKind::N, BasisOrder::PWC, fam, local)));
    }
    CurrentField x = random_field(d, BasisOrder::PWC, 721);
    OracleForms of = to_oracle(fam, BasisOrder::PWC);
    const std::vector<cplx> xv = x.to_vector();
    std::vector<cplx> yref(xv.size());
    const int64_t g[3] = {d[0], d[1], d[2]};
    if (orc_apply_operator_tucker(0, 0, g, of.ranks.data(), of.pc.data(), of.p1.data(), of.p2.data(), of.p3.data(),
                                  reinterpret_cast<const double*>(xv.data()), reinterpret_cast<double*>(yref.data())))
      throw std::runtime_error(orc_last_error());
    CurrentField y = apply_operator(*op, x, MatvecStrategy::HosvdDecompress, ScratchPolicy::WithBuffer, nullptr, dft);
    expect(rel(yref, y.to_vector()) <= 1e-10, "operator after its DftService");
  });

  // test_container.cpp:22-66 through the drop-in's save_container / load_container
  run("Container.RoundTripsAndRejectsGarbage", [&] {
    const std::string dir = "/tmp/";
    Tensor3 t(3, 4, 5);
    if (orc_random_tensor(3, 4, 5, 1, reinterpret_cast<double*>(t.data.data()))) throw std::runtime_error(orc_last_error());
    save_container(dir + "vie_b200_dense.bin", t);
    ContainerValue v = load_container(dir + "vie_b200_dense.bin");
    expect(std::holds_alternative<Tensor3>(v) && std::get<Tensor3>(v).data == t.data, "dense round trip");
    TuckerForm f;
    f.ranks = {2, 3, 2};
    f.core = Tensor3(2, 3, 2);
    for (int q = 0; q < 3; ++q) f.factors[q] = random_matrix(4 + q, f.ranks[static_cast<size_t>(q)], 700 + q);
    for (size_t i = 0; i < f.core.data.size(); ++i) f.core.data[i] = cplx(0.5 * i, -0.25 * i);
    f.rule = TruncationRule::Energy;
    f.tol = 1e-6;
    save_container(dir + "vie_b200_tucker.bin", f, {4, 5, 6});
    v = load_container(dir + "vie_b200_tucker.bin");
    expect(std::holds_alternative<TuckerForm>(v), "tucker kind");
    const TuckerForm& g = std::get<TuckerForm>(v);
    expect(g.ranks == f.ranks && g.rule == f.rule && g.tol == f.tol && g.core.data == f.core.data, "tucker header/core");
    for (int q = 0; q < 3; ++q) expect(g.factors[q].data == f.factors[q].data, "tucker factors");
    TuckerCPForm c;
    c.rank = 3;
    for (int q = 0; q < 3; ++q) c.factors[q] = random_matrix(5, 3, 800 + q);
    save_container(dir + "vie_b200_tcp.bin", c, {5, 5, 5});
    v = load_container(dir + "vie_b200_tcp.bin");
    expect(std::holds_alternative<TuckerCPForm>(v) && std::get<TuckerCPForm>(v).factors[2].data == c.factors[2].data,
           "tucker_cp round trip");
    {
      std::FILE* fp = std::fopen((dir + "vie_b200_garbage.bin").c_str(), "wb");
      std::fputs("not a container", fp);
      std::fclose(fp);
    }
    bool threw = false;
    try {
      load_container(dir + "vie_b200_garbage.bin");
    } catch (const std::runtime_error&) {
      threw = true;
    }
    expect(threw, "garbage must throw std::runtime_error");
    for (const char* n : {"vie_b200_dense.bin", "vie_b200_tucker.bin", "vie_b200_tcp.bin", "vie_b200_garbage.bin"})
      std::remove((dir + n).c_str());
  });

  std::printf("%d failure(s)\n", g_fail);
  return g_fail;
}
