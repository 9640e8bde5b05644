// C++ parity tests of the drop-in wrapper (include/vie_b200.hpp), written the
// way the reference's GTest suites are (test_fft_operator.cpp, test_solver.cpp),
// with the CPU oracle (oracle/vie_oracle.h, test infrastructure) as checker.
// Prints one PASS/FAIL line per test; exit code = number of failures.
#include <cmath>
#include <complex>
#include <cstdio>
#include <functional>
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

  std::printf("%d failure(s)\n", g_fail);
  return g_fail;
}
