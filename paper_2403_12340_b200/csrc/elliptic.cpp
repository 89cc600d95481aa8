// elliptic.cpp — host contour geometry (see elliptic.h). Restates the
// reference scalar algorithms: AGM / K(k) (elliptic.hpp:17-33), descending
// Landen sn cn dn (elliptic.hpp:48-85), A&S 16.21 complex addition
// (elliptic.hpp:97-118), adaptive 15-point Gauss-Legendre
// (elliptic.hpp:133-193), elliptic_params (contour.hpp:35-71) and the node map
// of contour_node_term (contour.hpp:149-166).
#include "elliptic.h"

#include <algorithm>
#include <cmath>

namespace lrgw_host {

namespace {
constexpr double kPi = 3.14159265358979323846;
}

double agm(double a, double b) {
  for (int it = 0; it < 64; ++it) {
    const double an = 0.5 * (a + b);
    const double bn = std::sqrt(a * b);
    if (std::abs(an - bn) <= 1e-16 * an) return an;
    a = an;
    b = bn;
  }
  return 0.5 * (a + b);
}

int elliptic_k(double k, double* out) {
  if (!(k >= 0.0 && k < 1.0)) return kInvalid;
  *out = kPi / (2.0 * agm(1.0, std::sqrt((1.0 - k) * (1.0 + k))));
  return kOk;
}

int jacobi_sn_cn_dn(double u, double k, double* sn_o, double* cn_o, double* dn_o) {
  if (!(k >= 0.0 && k < 1.0)) return kInvalid;
  if (k < 1e-14) {
    *sn_o = std::sin(u);
    *cn_o = std::cos(u);
    *dn_o = 1.0;
    return kOk;
  }
  // AGM scale sequence, then back-substitution on function values.
  double em[24], en[24];
  double a = 1.0, emc = (1.0 - k) * (1.0 + k), c = 0.0;
  int last = 0;
  for (int i = 0; i < 24; ++i) {
    last = i;
    em[i] = a;
    emc = std::sqrt(emc);
    en[i] = emc;
    c = 0.5 * (a + emc);
    if (std::abs(a - emc) <= 1e-16 * a) break;
    emc *= a;
    a = c;
  }
  const double uc = u * c;
  double sn = std::sin(uc), cn = std::cos(uc), dn = 1.0;
  if (sn != 0.0) {
    a = cn / sn;
    c *= a;
    for (int i = last; i >= 0; --i) {
      const double b = em[i];
      a *= c;
      c *= dn;
      dn = (en[i] + a) / (b + a);
      a = c / b;
    }
    a = 1.0 / std::sqrt(c * c + 1.0);
    sn = (sn >= 0.0) ? a : -a;
    cn = c * sn;
  }
  *sn_o = sn;
  *cn_o = cn;
  *dn_o = dn;
  return kOk;
}

int jacobi_complex(double x, double y, double k, std::complex<double>* sn,
                   std::complex<double>* cn, std::complex<double>* dn) {
  if (!(k >= 0.0 && k < 1.0)) return kInvalid;
  const double kp = std::sqrt((1.0 - k) * (1.0 + k));
  double kk = 0.0;
  if (elliptic_k(kp, &kk) != kOk) return kInvalid;
  if (std::abs(y) >= kk) return kInvalid;
  double rs, rc, rd, is, ic, id;
  jacobi_sn_cn_dn(x, k, &rs, &rc, &rd);
  jacobi_sn_cn_dn(y, kp, &is, &ic, &id);
  const double den = ic * ic + k * k * rs * rs * is * is;
  if (std::abs(den) < 1e-13) return kNumeric;
  const std::complex<double> i_unit(0.0, 1.0);
  *sn = (rs * id + i_unit * (rc * rd * is * ic)) / den;
  *cn = (rc * ic - i_unit * (rs * rd * is * id)) / den;
  *dn = (rd * ic * id - i_unit * (k * k * rs * rc * is)) / den;
  return kOk;
}

namespace {

struct Rule {
  double x[15], w[15];
};

Rule make_rule() {
  Rule r{};
  const int n = 15, m = (n + 1) / 2;
  for (int i = 0; i < m; ++i) {
    double z = std::cos(kPi * (i + 0.75) / (n + 0.5));
    double pp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p1 = 1.0, p2 = 0.0;
      for (int j = 0; j < n; ++j) {
        const double p3 = p2;
        p2 = p1;
        p1 = ((2.0 * j + 1.0) * z * p2 - j * p3) / (j + 1);
      }
      pp = n * (z * p1 - p2) / (z * z - 1.0);
      const double z1 = z;
      z = z1 - p1 / pp;
      if (std::abs(z - z1) < 1e-15) break;
    }
    r.x[i] = -z;
    r.x[n - 1 - i] = z;
    r.w[i] = 2.0 / ((1.0 - z * z) * pp * pp);
    r.w[n - 1 - i] = r.w[i];
  }
  return r;
}

double gl_apply(const Rule& r, double (*f)(double, void*), void* ctx, double a, double b) {
  const double xm = 0.5 * (b + a), xl = 0.5 * (b - a);
  double s = 0.0;
  for (int i = 0; i < 15; ++i) s += r.w[i] * f(xm + xl * r.x[i], ctx);
  return s * xl;
}

double gl_adapt(const Rule& r, double (*f)(double, void*), void* ctx, double a, double b,
                double whole, double tol, int depth) {
  const double mid = 0.5 * (a + b);
  const double left = gl_apply(r, f, ctx, a, mid);
  const double right = gl_apply(r, f, ctx, mid, b);
  const double refined = left + right;
  if (std::abs(refined - whole) <= tol * std::max(1.0, std::abs(refined)) || depth >= 48)
    return refined;
  return gl_adapt(r, f, ctx, a, mid, left, 0.5 * tol, depth + 1) +
         gl_adapt(r, f, ctx, mid, b, right, 0.5 * tol, depth + 1);
}

double height_integrand(double t, void* ctx) {
  const double r = *static_cast<double*>(ctx);
  return 1.0 / std::sqrt((1.0 + t * t) * (1.0 + r * r * t * t));
}

}  // namespace

double integrate_adaptive(double (*f)(double, void*), void* ctx, double a, double b,
                          double rel_tol) {
  static const Rule rule = make_rule();
  return gl_adapt(rule, f, ctx, a, b, gl_apply(rule, f, ctx, a, b), rel_tol, 0);
}

int elliptic_params(const double* e, int n_e, int n_v, int n_c, double delta_rel, int max_nodes,
                    Spec* out) {
  if (n_v < 1 || n_c < 1 || n_v + n_c > n_e) return kInvalid;
  Spec s;
  s.q = e[n_v] - e[n_v - 1];
  s.big_q = e[n_v + n_c - 1] - e[n_v - 1];
  s.e_shift = e[n_v - 1];
  s.delta_rel = delta_rel;
  s.max_nodes = max_nodes;
  if (!(s.q > 0.0)) return kInvalid;
  const double ratio = s.big_q / s.q;
  if (ratio <= 1.0 + 1e-12) {
    s.r = 0.0;
    elliptic_k(0.0, &s.big_r);
    s.l = 0.0;
    s.bypass = true;
    *out = s;
    return kOk;
  }
  const double sq = std::sqrt(ratio);
  s.r = (sq - 1.0) / (sq + 1.0);
  elliptic_k(s.r, &s.big_r);
  double r = s.r;
  s.l = 0.5 * integrate_adaptive(height_integrand, &r, 0.0, 1.0 / r, 1e-13);
  s.bypass = false;
  *out = s;
  return kOk;
}

int cauchy_error_bound(const Spec& s, int n_lambda, double* out) {
  if (n_lambda < 1) return kInvalid;
  *out = std::exp(-kPi * kPi * n_lambda / (2.0 * std::log(s.big_q / s.q) + 6.0));
  return kOk;
}

double prefactor(const Spec& s) { return 2.0 * std::sqrt(s.q * s.big_q) / (kPi * s.r); }

int node_geometry(const Spec& s, double t, std::complex<double>* z, std::complex<double>* g) {
  std::complex<double> sn, cn, dn;
  const int st = jacobi_complex(t, s.l, s.r, &sn, &cn, &dn);
  if (st != kOk) return st;
  const double r_inv = 1.0 / s.r;
  const std::complex<double> den = r_inv - sn;
  *z = std::sqrt(s.q * s.big_q) * (r_inv + sn) / den + s.e_shift;
  *g = cn * dn / (den * den);
  return kOk;
}

int node_tables(const Spec& s, const double* e, int n_v, int n_c, const double* nodes,
                const double* weights, int n_nodes, std::vector<double>* dv,
                std::vector<double>* dc, std::vector<double>* gw) {
  dv->assign(static_cast<size_t>(2) * n_v * n_nodes, 0.0);
  dc->assign(static_cast<size_t>(2) * n_c * n_nodes, 0.0);
  gw->assign(static_cast<size_t>(2) * n_nodes, 0.0);
  for (int k = 0; k < n_nodes; ++k) {
    std::complex<double> z, g;
    const int st = node_geometry(s, nodes[k], &z, &g);
    if (st != kOk) return st;
    for (int i = 0; i < n_v; ++i) {
      const std::complex<double> d = 1.0 / (z - e[i]);
      (*dv)[2 * (static_cast<size_t>(k) * n_v + i)] = d.real();
      (*dv)[2 * (static_cast<size_t>(k) * n_v + i) + 1] = d.imag();
    }
    for (int j = 0; j < n_c; ++j) {
      const std::complex<double> d = 1.0 / (z - e[n_v + j]);
      (*dc)[2 * (static_cast<size_t>(k) * n_c + j)] = d.real();
      (*dc)[2 * (static_cast<size_t>(k) * n_c + j) + 1] = d.imag();
    }
    (*gw)[2 * k] = weights[k] * g.real();
    (*gw)[2 * k + 1] = weights[k] * g.imag();
  }
  return kOk;
}

}  // namespace lrgw_host
