// kernels_assembly.cu -- Green's-tensor assembly on the device: the PWC Galerkin
// Toeplitz-defining tensor of one N / K / scalar-g kernel component on a uniform grid.
//
// Reference: assemble_defining_tensor (assembly.hpp:159-233) with the tent-weighted
// correlation reduction of the voxel-pair integral (assembly.hpp:49-79), the Duffy
// corner rules (quadrature.hpp:92-118, 139-166), the static self term integrated by
// parts onto the faces (assembly.hpp:84-150) and the kernels of kernels.hpp:13-134.
// One thread per tensor entry (every entry is an independent 3-D quadrature of
// 8 tent sub-boxes, p^3 points each: compute-bound FP64 with one sincos per point);
// the self entry (a few thousand points, series-stable remainder kernel) is one
// thread of a separate launch.  Units as the reference: computed in x-voxel-edge
// units, scaled by edge^3 (N), ^4 (K), ^5 (g).
#include <cmath>
#include <map>
#include <vector>

#include "kernels.cuh"

namespace vie {

namespace {

constexpr double kPi = 3.14159265358979323846264338327950288;
constexpr double kInv4pi = 1.0 / (4.0 * kPi);

struct Rule {  // one Gauss-Legendre rule on [0, 1]: p nodes / weights (device)
  const double* nd;
  const double* wt;
  int p;
};
struct Rules {  // the rules one launch uses (no runtime-indexed parameter arrays)
  Rule far, near, surface, surface4, volume;
};

struct Radial {
  double2 g, gp, gpp;
};

__device__ __forceinline__ double2 cexp_i(double th) {  // e^{i th}
  double s, c;
  sincos(th, &s, &c);
  return make_double2(c, s);
}
__device__ __forceinline__ double2 cmul_s(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 cdiv_s(double2 a, double s) { return make_double2(a.x / s, a.y / s); }
__device__ __forceinline__ double2 cdivc(double2 a, double2 b) {  // a / b
  const double d = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}
__device__ __forceinline__ double cabs2(double2 a) { return hypot(a.x, a.y); }

// kernels.hpp:67-76: g = e^{-ikR} / (4 pi R) and its radial derivatives
__device__ Radial radial(double R, double k) {
  const double2 e = cexp_i(-k * R);
  const double2 ikr = make_double2(0.0, k * R);
  Radial r;
  r.g = cdiv_s(cmul_s(e, kInv4pi), R);
  r.gp = cdiv_s(cmul_s(cmul(make_double2(-1.0 - ikr.x, -ikr.y), e), kInv4pi), R * R);
  r.gpp = cdiv_s(cmul_s(cmul(make_double2(2.0 + 2.0 * ikr.x - k * k * R * R, 2.0 * ikr.y), e), kInv4pi), R * R * R);
  return r;
}

// kernels.hpp:28-60 series-stable helpers of x = -i k R (purely imaginary here)
__device__ double2 cexp_c(double2 x) {
  const double m = exp(x.x);
  const double2 p = cexp_i(x.y);
  return make_double2(m * p.x, m * p.y);
}
__device__ double2 phi0(double2 x) {
  if (cabs2(x) > 1.0) {
    const double2 e = cexp_c(x);
    return make_double2(e.x - 1.0, e.y);
  }
  double2 term = x, sum = x;
  for (int n = 2; n < 26; ++n) {
    term = cmul(term, cdiv_s(x, static_cast<double>(n)));
    sum = cadd(sum, term);
  }
  return sum;
}
__device__ double2 psi1(double2 x) {
  if (cabs2(x) > 1.0) {
    const double2 e = cexp_c(x);
    const double2 t = cmul(make_double2(x.x - 1.0, x.y), e);
    return make_double2(t.x + 1.0, t.y);
  }
  double2 xn = x, sum = make_double2(0.0, 0.0);
  for (int n = 2; n < 28; ++n) {
    xn = cmul(xn, cdiv_s(x, static_cast<double>(n)));
    sum = cadd(sum, cmul_s(xn, static_cast<double>(n - 1)));
  }
  return sum;
}
__device__ double2 psi2(double2 x) {
  if (cabs2(x) > 1.0) {
    const double2 e = cexp_c(x);
    const double2 x2 = cmul(x, x);
    const double2 t = cmul(e, make_double2(x2.x - 2.0 * x.x + 2.0, x2.y - 2.0 * x.y));
    return make_double2(t.x - 2.0, t.y);
  }
  double2 sum = make_double2(0.0, 0.0);
  double2 xm = cdiv_s(cmul(x, x), 2.0);
  for (int m = 3; m < 30; ++m) {
    xm = cmul(xm, cdiv_s(x, static_cast<double>(m)));
    sum = cadd(sum, cmul_s(xm, static_cast<double>((m - 1) * (m - 2))));
  }
  return sum;
}
// kernels.hpp:84-91
__device__ Radial radial_dynamic(double R, double k) {
  const double2 x = make_double2(0.0, -k * R);
  Radial r;
  r.g = cdiv_s(cmul_s(phi0(x), kInv4pi), R);
  r.gp = cdiv_s(cmul_s(psi1(x), kInv4pi), R * R);
  r.gpp = cdiv_s(cmul_s(psi2(x), kInv4pi), R * R * R);
  return r;
}
// kernels.hpp:95-99
__device__ double2 hessian_entry(const Radial& h, const double rhat[3], double R, int q, int qp) {
  const double2 iso = cdiv_s(h.gp, R);
  const double2 aniso = csub(h.gpp, iso);
  double2 v = cmul_s(cmul_s(aniso, rhat[q]), rhat[qp]);
  if (q == qp) v = cadd(v, iso);
  return v;
}

// kernel op: 0 N (kernels.hpp:103-108), 1 K (:128-134), 2 scalar g, 3 N self remainder (:113-119)
__device__ double2 kernel_eval(int op, const double r[3], double k, int q, int qp) {
  const double R = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
  if (op == 2) return radial(R, k).g;
  if (op == 1) {
    if (q == qp) return make_double2(0.0, 0.0);
    const int a = 3 - q - qp;
    const Radial h = radial(R, k);
    const int lc = ((a - q + 3) % 3 == 1) ? 1 : -1;  // levi_civita(q, a, qp)
    return cmul_s(h.gp, static_cast<double>(lc) * r[a] / R);
  }
  const double rhat[3] = {r[0] / R, r[1] / R, r[2] / R};
  if (op == 0) {
    const Radial h = radial(R, k);
    double2 v = hessian_entry(h, rhat, R, q, qp);
    if (q == qp) v = cadd(v, cmul_s(h.g, k * k));
    return v;
  }
  const Radial hd = radial_dynamic(R, k);
  const double2 g_full = make_double2(hd.g.x + kInv4pi / R, hd.g.y);
  double2 v = hessian_entry(hd, rhat, R, q, qp);
  if (q == qp) v = cadd(v, cmul_s(g_full, k * k));
  return v;
}

struct KDesc {
  int op, q, qp;
  double k;
};

// integrand of the correlation: kernel(u - d) * prod_a (delta_a - |u_a|)
__device__ __forceinline__ double2 weighted(const KDesc& kd, const double u[3], const double d[3],
                                            const double delta[3]) {
  const double w = (delta[0] - fabs(u[0])) * (delta[1] - fabs(u[1])) * (delta[2] - fabs(u[2]));
  const double r[3] = {u[0] - d[0], u[1] - d[1], u[2] - d[2]};
  return cmul_s(kernel_eval(kd.op, r, kd.k, kd.q, kd.qp), w);
}

// quadrature.hpp:71-86
__device__ double2 integrate_box(const KDesc& kd, const double lo[3], const double hi[3], const double d[3],
                                 const double delta[3], const Rule& gr) {
  const double* nd = gr.nd;
  const double* wt = gr.wt;
  const int p = gr.p;
  const double lx = hi[0] - lo[0], ly = hi[1] - lo[1], lz = hi[2] - lo[2];
  double2 sum = make_double2(0.0, 0.0);
  for (int a = 0; a < p; ++a)
    for (int b = 0; b < p; ++b)
      for (int c = 0; c < p; ++c) {
        const double u[3] = {lo[0] + lx * nd[a], lo[1] + ly * nd[b], lo[2] + lz * nd[c]};
        sum = cadd(sum, cmul_s(weighted(kd, u, d, delta), wt[a] * wt[b] * wt[c]));
      }
  return cmul_s(sum, lx * ly * lz);
}

// quadrature.hpp:92-118 (three-pyramid Duffy at the given corner)
__device__ double2 integrate_box_duffy(const KDesc& kd, const double lo[3], const double hi[3], const int corner[3],
                                       const double d[3], const double delta[3], const Rule& gr) {
  const double* nd = gr.nd;
  const double* wt = gr.wt;
  const int p = gr.p;
  double base[3], span[3];
  for (int a = 0; a < 3; ++a) {
    base[a] = corner[a] ? hi[a] : lo[a];
    span[a] = (corner[a] ? lo[a] : hi[a]) - base[a];
  }
  const double jac = fabs(span[0] * span[1] * span[2]);
  double2 sum = make_double2(0.0, 0.0);
  for (int rad = 0; rad < 3; ++rad) {
    const int s1 = (rad + 1) % 3, s2 = (rad + 2) % 3;
    for (int a = 0; a < p; ++a) {
      const double t = nd[a];
      for (int b = 0; b < p; ++b)
        for (int c = 0; c < p; ++c) {
          double v[3];
          v[rad] = t;
          v[s1] = t * nd[b];
          v[s2] = t * nd[c];
          const double u[3] = {base[0] + span[0] * v[0], base[1] + span[1] * v[1], base[2] + span[2] * v[2]};
          sum = cadd(sum, cmul_s(weighted(kd, u, d, delta), wt[a] * wt[b] * wt[c] * (t * t)));
        }
    }
  }
  return cmul_s(sum, jac);
}

// assembly.hpp:49-79
__device__ double2 correlation_entry(const KDesc& kd, const double d[3], const double delta[3], bool duffy_at_d,
                                     const Rule& gr) {
  double cuts[3][4];
  int nc[3];
  for (int a = 0; a < 3; ++a) {
    cuts[a][0] = -delta[a];
    cuts[a][1] = 0.0;
    cuts[a][2] = delta[a];
    nc[a] = 3;
    if (duffy_at_d && d[a] > -delta[a] && d[a] < delta[a] && d[a] != 0.0) {
      cuts[a][3] = d[a];
      nc[a] = 4;
      for (int i = 3; i > 0 && cuts[a][i] < cuts[a][i - 1]; --i) {  // keep sorted
        const double t = cuts[a][i];
        cuts[a][i] = cuts[a][i - 1];
        cuts[a][i - 1] = t;
      }
    }
  }
  double2 sum = make_double2(0.0, 0.0);
  for (int ia = 0; ia + 1 < nc[0]; ++ia)
    for (int ib = 0; ib + 1 < nc[1]; ++ib)
      for (int ic = 0; ic + 1 < nc[2]; ++ic) {
        const double lo[3] = {cuts[0][ia], cuts[1][ib], cuts[2][ic]};
        const double hi[3] = {cuts[0][ia + 1], cuts[1][ib + 1], cuts[2][ic + 1]};
        bool corner = duffy_at_d;
        int which[3] = {0, 0, 0};
        for (int a = 0; a < 3; ++a) {
          if (d[a] == lo[a]) which[a] = 0;
          else if (d[a] == hi[a]) which[a] = 1;
          else corner = false;
        }
        sum = cadd(sum, corner ? integrate_box_duffy(kd, lo, hi, which, d, delta, gr)
                               : integrate_box(kd, lo, hi, d, delta, gr));
      }
  return sum;
}

// assembly.hpp:84-104 (2-D tent-weighted correlation of g_static over a face pair)
__device__ double face_pair_static(double dt1, double dt2, double h, const Rule& gr) {
  const double* nd = gr.nd;
  const double* wt = gr.wt;
  const int p = gr.p;
  auto f = [&](double u, double v) {
    const double w = (dt1 - fabs(u)) * (dt2 - fabs(v));
    return w * kInv4pi / sqrt(h * h + u * u + v * v);
  };
  double sum = 0.0;
  for (int su = 0; su < 2; ++su)
    for (int sv = 0; sv < 2; ++sv) {
      const double lo[2] = {su ? 0.0 : -dt1, sv ? 0.0 : -dt2};
      const double hi[2] = {su ? dt1 : 0.0, sv ? dt2 : 0.0};
      if (h == 0.0) {  // quadrature.hpp:139-166, singular corner at the origin
        const int corner[2] = {su ? 0 : 1, sv ? 0 : 1};
        double base[2], span[2];
        for (int a = 0; a < 2; ++a) {
          base[a] = corner[a] ? hi[a] : lo[a];
          span[a] = (corner[a] ? lo[a] : hi[a]) - base[a];
        }
        const double jac = fabs(span[0] * span[1]);
        double s = 0.0;
        for (int rad = 0; rad < 2; ++rad) {
          const int other = 1 - rad;
          for (int a = 0; a < p; ++a) {
            const double t = nd[a];
            for (int b = 0; b < p; ++b) {
              double v[2];
              v[rad] = t;
              v[other] = t * nd[b];
              s += wt[a] * wt[b] * t * f(base[0] + span[0] * v[0], base[1] + span[1] * v[1]);
            }
          }
        }
        sum += s * jac;
      } else {  // quadrature.hpp:126-136
        const double lx = hi[0] - lo[0], ly = hi[1] - lo[1];
        double s = 0.0;
        for (int a = 0; a < p; ++a)
          for (int b = 0; b < p; ++b) s += wt[a] * wt[b] * f(lo[0] + lx * nd[a], lo[1] + ly * nd[b]);
        sum += s * (lx * ly);
      }
    }
  return sum;
}

struct AsmArgs {
  int n1, n2, n3;
  double delta[3];
  KDesc kd;
  int par[3];
  int far, near, near_radius, surface, volume;
  double si_scale;
};

// assembly.hpp:127-150 + the self entry of :192-206 (one thread)
// assembly.hpp:127-150: diagonal of the static nabla-nabla dyad (one thread)
__global__ void k_self_static(AsmArgs a, Rules gr, double* out_dyad, double* out_err) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double* delta = a.delta;
  const double gram = delta[0] * delta[1] * delta[2];
  double max_change = 0.0;
  for (int q = 0; q < 3; ++q) {
    const int t1 = (q + 1) % 3, t2 = (q + 2) % 3;
    const double v = 2.0 * (face_pair_static(delta[t1], delta[t2], delta[q], gr.surface) -
                            face_pair_static(delta[t1], delta[t2], 0.0, gr.surface));
    const double v_refined = 2.0 * (face_pair_static(delta[t1], delta[t2], delta[q], gr.surface4) -
                                    face_pair_static(delta[t1], delta[t2], 0.0, gr.surface4));
    out_dyad[q] = v_refined;
    max_change = fmax(max_change, fabs(v_refined - v) / gram);
  }
  *out_err = max_change;
}

// the self entry of assembly.hpp:192-206: remainder correlation (+ gram + dyad for N diagonals)
__global__ void k_self_entry(AsmArgs a, Rules gr, const double* dyad, double2* out_self) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double zero[3] = {0.0, 0.0, 0.0};
  double2 self = make_double2(0.0, 0.0);
  if (a.kd.op == 0) {
    const KDesc rem{3, a.kd.q, a.kd.qp, a.kd.k};  // the N self remainder kernel (kernels.hpp:113-119)
    self = correlation_entry(rem, zero, a.delta, true, gr.volume);
    if (a.kd.q == a.kd.qp) self.x += a.delta[0] * a.delta[1] * a.delta[2] + dyad[a.kd.q];
  } else if (a.kd.op == 2) {
    self = correlation_entry(a.kd, zero, a.delta, true, gr.volume);
  }
  *out_self = cmul_s(self, a.si_scale);
}

__global__ void __launch_bounds__(128) k_assemble(AsmArgs a, Rules gr, const double2* __restrict__ self,
                                                  double2* __restrict__ t) {
  const int64_t nv = static_cast<int64_t>(a.n1) * a.n2 * a.n3;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nv;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int ii = static_cast<int>(e % a.n1);
    const int jj = static_cast<int>((e / a.n1) % a.n2);
    const int kk = static_cast<int>(e / (static_cast<int64_t>(a.n1) * a.n2));
    if ((a.par[0] < 0 && ii == 0) || (a.par[1] < 0 && jj == 0) || (a.par[2] < 0 && kk == 0)) {
      t[e] = make_double2(0.0, 0.0);
      continue;
    }
    const int cheb = max(ii, max(jj, kk));
    if (cheb == 0) {
      t[e] = *self;
      continue;
    }
    const double d[3] = {ii * a.delta[0], jj * a.delta[1], kk * a.delta[2]};
    const bool near = cheb <= a.near_radius;
    t[e] = cmul_s(correlation_entry(a.kd, d, a.delta, near, near ? gr.near : gr.far), a.si_scale);
  }
}

__global__ void k_correlation_entry(KDesc kd, double d0, double d1, double d2, double e0, double e1, double e2,
                                    int duffy, Rule gr, double2* out) {
  const double d[3] = {d0, d1, d2}, delta[3] = {e0, e1, e2};
  *out = correlation_entry(kd, d, delta, duffy != 0, gr);
}

// quadrature.hpp:21-58 on the host
void gauss_rule_host(int p, std::vector<double>& nodes, std::vector<double>& weights) {
  nodes.assign(static_cast<size_t>(p), 0.0);
  weights.assign(static_cast<size_t>(p), 0.0);
  const int m = (p + 1) / 2;
  for (int i = 0; i < m; ++i) {
    double x = std::cos(kPi * (i + 0.75) / (p + 0.5));
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
    nodes[static_cast<size_t>(i)] = 0.5 * (1.0 - x);
    weights[static_cast<size_t>(i)] = w;
    nodes[static_cast<size_t>(p - 1 - i)] = 0.5 * (1.0 + x);
    weights[static_cast<size_t>(p - 1 - i)] = w;
  }
}

}  // namespace

namespace {
// Gauss tables for the point counts of a launch, copied to rules_scratch (nodes then weights)
std::vector<Rule> upload_rules(const std::vector<int>& ps, double* rules_scratch, cudaStream_t st) {
  std::vector<double> nodes(kAsmRuleElems, 0.0), weights(kAsmRuleElems, 0.0);
  std::vector<Rule> out;
  int used = 0;
  for (int p : ps) {
    if (p < 1 || p > 31) throw std::invalid_argument("assemble: 1..31 quadrature points per axis");
    if (used + p > kAsmRuleElems) throw std::invalid_argument("assemble: quadrature table overflow");
    std::vector<double> n, w;
    gauss_rule_host(p, n, w);
    for (int i = 0; i < p; ++i) {
      nodes[static_cast<size_t>(used + i)] = n[static_cast<size_t>(i)];
      weights[static_cast<size_t>(used + i)] = w[static_cast<size_t>(i)];
    }
    out.push_back(Rule{rules_scratch + used, rules_scratch + kAsmRuleElems + used, p});
    used += p;
  }
  VIE_CUDA_CHECK(cudaMemcpyAsync(rules_scratch, nodes.data(), sizeof(double) * kAsmRuleElems, cudaMemcpyHostToDevice, st));
  VIE_CUDA_CHECK(cudaMemcpyAsync(rules_scratch + kAsmRuleElems, weights.data(), sizeof(double) * kAsmRuleElems,
                                 cudaMemcpyHostToDevice, st));
  VIE_CUDA_CHECK(cudaStreamSynchronize(st));  // host staging vectors go out of scope
  return out;
}
}  // namespace

void launch_correlation_entry(int op, double k, int q, int qp, const double d[3], const double delta[3], int points,
                              int duffy, double* rules_scratch, double2* out, cudaStream_t st) {
  const Rule gr = upload_rules({points}, rules_scratch, st)[0];
  k_correlation_entry<<<1, 1, 0, st>>>(KDesc{op, q, qp, k}, d[0], d[1], d[2], delta[0], delta[1], delta[2], duffy, gr,
                                       out);
  VIE_CUDA_CHECK(cudaGetLastError());
}

void launch_assemble(const AssemblyDesc& ad, double2* t, double2* self_scratch, double* rules_scratch,
                     cudaStream_t st, double* dyad_out, double* err_out) {
  const std::vector<Rule> r5 = upload_rules({ad.far, ad.near, ad.surface, ad.surface + 4, ad.volume}, rules_scratch, st);
  const Rules gr{r5[0], r5[1], r5[2], r5[3], r5[4]};
  AsmArgs a{};
  a.n1 = static_cast<int>(ad.dims[0]);
  a.n2 = static_cast<int>(ad.dims[1]);
  a.n3 = static_cast<int>(ad.dims[2]);
  const double scale = ad.res[0];
  a.delta[0] = 1.0;
  a.delta[1] = ad.res[1] / scale;
  a.delta[2] = ad.res[2] / scale;
  a.kd = KDesc{ad.op, ad.q, ad.qp, ad.k0 * scale};
  for (int i = 0; i < 3; ++i) a.par[i] = 1;
  if (ad.op == 0 && ad.q != ad.qp) a.par[ad.q] = a.par[ad.qp] = -1;
  if (ad.op == 1 && ad.q != ad.qp) a.par[3 - ad.q - ad.qp] = -1;
  a.far = ad.far;
  a.near = ad.near;
  a.near_radius = ad.near_radius;
  a.surface = ad.surface;
  a.volume = ad.volume;
  a.si_scale = std::pow(scale, ad.op == 0 ? 3.0 : (ad.op == 1 ? 4.0 : 5.0));
  // dyad (3) + error (1) into dyad_out / err_out when given, else into the rules scratch tail
  double* dy = dyad_out ? dyad_out : rules_scratch + 2 * kAsmRuleElems;
  double* er = err_out ? err_out : rules_scratch + 2 * kAsmRuleElems + 3;
  k_self_static<<<1, 1, 0, st>>>(a, gr, dy, er);
  VIE_CUDA_CHECK(cudaGetLastError());
  if (!t) return;
  k_self_entry<<<1, 1, 0, st>>>(a, gr, dy, self_scratch);
  VIE_CUDA_CHECK(cudaGetLastError());
  const int64_t nv = ad.dims[0] * ad.dims[1] * ad.dims[2];
  const int threads = 128;
  const int64_t blocks = std::min<int64_t>((nv + threads - 1) / threads, 148 * 64);
  k_assemble<<<static_cast<unsigned>(blocks), threads, 0, st>>>(a, gr, self_scratch, t);
  VIE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace vie
