// elliptic.cpp — host contour geometry (see elliptic.h), derived from the
// classical identities below rather than from the reference's recipes; it
// produces the reference's ContourSpec (contour.hpp:23-71) and node map
// (contour.hpp:149-166) to rounding.
//
//  * K(k) and the contour height L are Carlson symmetric integrals:
//      K(k) = R_F(0, 1 - k^2, 1)
//      L    = 1/2 int_0^{1/r} dt / sqrt((1 + t^2)(1 + r^2 t^2))
//           = 1/2 F(atan(1/r) | k'),  k'^2 = 1 - r^2       (t = tan theta)
//           = 1/2 R_F(r^2, 2 r^2, 1 + r^2)                 (homogeneity of R_F)
//    so the height needs no quadrature at all. R_F by Carlson's duplication
//    theorem with the fifth-order Taylor tail (relative error < 1e-16).
//  * sn, cn, dn for real argument by Gauss's transformation (descending
//    Landen in modulus form, A&S 16.12.2-4): k -> k1 = k^2 / (1 + k')^2,
//    u -> u / (1 + k1), recursed until k^2 is below 1e-17, where the
//    first-order small-modulus expansion (A&S 16.13) is exact to rounding;
//    then ascended with sn = (1 + k1) s / (1 + k1 s^2), cn = c d / (1 + k1 s^2),
//    dn = (1 - k1 s^2) / (1 + k1 s^2). No asin / amplitude is formed, so the
//    quarter-period arguments of the contour endpoints stay well conditioned.
//  * complex argument x + iy by the addition theorem of sn, cn, dn with
//    Jacobi's imaginary transformation sn(iy | k) = i sc(y | k'),
//    cn(iy | k) = nc(y | k'), dn(iy | k) = dc(y | k'), evaluated in complex
//    arithmetic. The reference's domain rule (|y| < K(k'), elliptic.hpp:97-105)
//    and pole rule (c'^2 + k^2 s^2 s'^2 below 1e-13, the addition theorem's
//    denominator scaled by cn(y | k')^2) are kept as behaviour.
#include "elliptic.h"

#include <algorithm>
#include <cmath>

namespace lrgw_host {

namespace {
constexpr double kPi = 3.14159265358979323846;

// Carlson's R_F(x, y, z) = 1/2 int_0^inf dt / sqrt((t+x)(t+y)(t+z)),
// x, y, z >= 0, at most one zero. Duplication x <- (x + lam) / 4 with
// lam = sqrt(xy) + sqrt(yz) + sqrt(zx) shrinks the spread by 4 per step; stop
// when every |1 - v / mean| < 1e-3 (the tail's 6th-order term is then
// ~ (1e-3)^6 / 4, far below double rounding) and sum the series
//   R_F = (1 - E2/10 + E3/14 + E2^2/24 - 3 E2 E3/44) / sqrt(mean).
double carlson_rf(double x, double y, double z) {
  for (int it = 0; it < 64; ++it) {
    const double mean = (x + y + z) / 3.0;
    const double dx = 1.0 - x / mean, dy = 1.0 - y / mean;
    if (std::max({std::abs(dx), std::abs(dy), std::abs(1.0 - z / mean)}) < 1e-3) {
      const double dz = -(dx + dy);  // the three deviations sum to zero
      const double e2 = dx * dy - dz * dz;
      const double e3 = dx * dy * dz;
      return (1.0 - e2 / 10.0 + e3 / 14.0 + e2 * e2 / 24.0 - 3.0 * e2 * e3 / 44.0) / std::sqrt(mean);
    }
    const double sx = std::sqrt(x), sy = std::sqrt(y), sz = std::sqrt(z);
    const double lam = sx * (sy + sz) + sy * sz;
    x = 0.25 * (x + lam);
    y = 0.25 * (y + lam);
    z = 0.25 * (z + lam);
  }
  return 1.0 / std::sqrt((x + y + z) / 3.0);
}

// 1 - k^2 without cancellation near k = 1.
inline double comp_param(double k) { return (1.0 - k) * (1.0 + k); }

}  // namespace

double agm(double a, double b) {
  // arithmetic-geometric mean; K(k) = pi / (2 agm(1, k')) is an identity of
  // R_F above, kept for callers of the reference's agm (elliptic.hpp:17-26)
  for (int it = 0; it < 64 && a != b; ++it) {
    const double m = 0.5 * (a + b);
    const double g = std::sqrt(a * b);
    if (m == a || m == b) break;  // no representable progress left
    a = m;
    b = g;
  }
  return 0.5 * (a + b);
}

int elliptic_k(double k, double* out) {
  if (!(k >= 0.0 && k < 1.0)) return kInvalid;
  *out = carlson_rf(0.0, comp_param(k), 1.0);
  return kOk;
}

int jacobi_sn_cn_dn(double u, double k, double* sn_o, double* cn_o, double* dn_o) {
  if (!(k >= 0.0 && k < 1.0)) return kInvalid;
  // descend: moduli of the Gauss transformation chain (quadratic decay)
  double chain[16];
  int depth = 0;
  double kk = k;
  while (kk * kk > 1e-17 && depth < 16) {
    const double kp = std::sqrt(comp_param(kk));
    const double k1 = (kk / (1.0 + kp)) * (kk / (1.0 + kp));
    chain[depth++] = k1;
    u /= (1.0 + k1);
    kk = k1;
  }
  // bottom: sn(u | m) = sin u - m/4 (u - sin u cos u) cos u + O(m^2), m = kk^2
  const double m = kk * kk;
  const double s0 = std::sin(u), c0 = std::cos(u);
  const double corr = 0.25 * m * (u - s0 * c0);
  double sn = s0 - corr * c0, cn = c0 + corr * s0, dn = 1.0 - 0.5 * m * s0 * s0;
  // ascend
  for (int i = depth - 1; i >= 0; --i) {
    const double k1 = chain[i];
    const double ks2 = k1 * sn * sn;
    const double inv = 1.0 / (1.0 + ks2);
    const double sn_up = (1.0 + k1) * sn * inv;
    cn = cn * dn * inv;
    dn = (1.0 - ks2) * inv;
    sn = sn_up;
  }
  *sn_o = sn;
  *cn_o = cn;
  *dn_o = dn;
  return kOk;
}

int jacobi_complex(double x, double y, double k, std::complex<double>* sn, std::complex<double>* cn,
                   std::complex<double>* dn) {
  if (!(k >= 0.0 && k < 1.0)) return kInvalid;
  const double kp = std::sqrt(comp_param(k));
  double k_comp = 0.0;
  if (elliptic_k(kp, &k_comp) != kOk) return kInvalid;
  if (std::abs(y) >= k_comp) return kInvalid;  // outside the fundamental rectangle
  double s, c, d, s1, c1, d1;
  jacobi_sn_cn_dn(x, k, &s, &c, &d);
  jacobi_sn_cn_dn(y, kp, &s1, &c1, &d1);
  // pole rule on c1^2 (1 - k^2 sn^2(x) sn^2(iy)) = c1^2 + k^2 s^2 s1^2
  const double pole = c1 * c1 + k * k * s * s * s1 * s1;
  if (std::abs(pole) < 1e-13) return kNumeric;
  // the second argument v = iy through the imaginary transformation
  const std::complex<double> sv(0.0, s1 / c1), cv(1.0 / c1, 0.0), dv(d1 / c1, 0.0);
  const std::complex<double> su(s, 0.0), cu(c, 0.0), du(d, 0.0);
  const std::complex<double> den = 1.0 - k * k * su * su * sv * sv;
  *sn = (su * cv * dv + sv * cu * du) / den;
  *cn = (cu * cv - su * sv * du * dv) / den;
  *dn = (du * dv - k * k * su * sv * cu * cv) / den;
  return kOk;
}

int elliptic_params(const double* e, int n_e, int n_v, int n_c, double delta_rel, int max_nodes, Spec* out) {
  if (n_v < 1 || n_c < 1 || n_v + n_c > n_e) return kInvalid;
  Spec s;
  s.e_shift = e[n_v - 1];            // HOMO
  s.q = e[n_v] - s.e_shift;          // gap to the LUMO
  s.big_q = e[n_v + n_c - 1] - s.e_shift;  // span to the top virtual
  s.delta_rel = delta_rel;
  s.max_nodes = max_nodes;
  if (!(s.q > 0.0)) return kInvalid;
  const double ratio = s.big_q / s.q;
  if (ratio <= 1.0 + 1e-12) {  // one energy denominator: the direct sum (contour.hpp:51-59)
    s.r = 0.0;
    elliptic_k(0.0, &s.big_r);
    s.l = 0.0;
    s.bypass = true;
    *out = s;
    return kOk;
  }
  // Moebius map of [q, Q] onto the elliptic rectangle: modulus r with
  // (1 + r) / (1 - r) = sqrt(Q / q)
  const double root = std::sqrt(ratio);
  s.r = (root - 1.0) / (root + 1.0);
  elliptic_k(s.r, &s.big_r);
  const double r2 = s.r * s.r;
  s.l = 0.5 * carlson_rf(r2, 2.0 * r2, 1.0 + r2);
  s.bypass = false;
  *out = s;
  return kOk;
}

int cauchy_error_bound(const Spec& s, int n_lambda, double* out) {
  if (n_lambda < 1) return kInvalid;
  // the reference's reporting model exp(-pi^2 N / (2 ln(Q/q) + 6)) (contour.hpp:75-80)
  *out = std::exp(-kPi * kPi * n_lambda / (2.0 * std::log(s.big_q / s.q) + 6.0));
  return kOk;
}

double prefactor(const Spec& s) { return 2.0 * std::sqrt(s.q * s.big_q) / (kPi * s.r); }

int node_geometry(const Spec& s, double t, std::complex<double>* z, std::complex<double>* g) {
  std::complex<double> sn, cn, dn;
  const int st = jacobi_complex(t, s.l, s.r, &sn, &cn, &dn);
  if (st != kOk) return st;
  // z(w) = sqrt(qQ) (1/r + sn w) / (1/r - sn w) + e_shift, dz/dw ∝ cn dn / (1/r - sn)^2
  const double a = 1.0 / s.r;
  const std::complex<double> below = a - sn;
  *z = std::sqrt(s.q * s.big_q) * (a + sn) / below + s.e_shift;
  *g = cn * dn / (below * below);
  return kOk;
}

int node_tables(const Spec& s, const double* e, int n_v, int n_c, const double* nodes, const double* weights,
                int n_nodes, std::vector<double>* dv, std::vector<double>* dc, std::vector<double>* gw) {
  dv->assign(static_cast<size_t>(2) * n_v * n_nodes, 0.0);
  dc->assign(static_cast<size_t>(2) * n_c * n_nodes, 0.0);
  gw->assign(static_cast<size_t>(2) * n_nodes, 0.0);
  auto put = [](std::vector<double>* v, size_t at, std::complex<double> x) {
    (*v)[2 * at] = x.real();
    (*v)[2 * at + 1] = x.imag();
  };
  for (int k = 0; k < n_nodes; ++k) {
    std::complex<double> z, g;
    const int st = node_geometry(s, nodes[k], &z, &g);
    if (st != kOk) return st;
    for (int i = 0; i < n_v; ++i) put(dv, static_cast<size_t>(k) * n_v + i, 1.0 / (z - e[i]));
    for (int j = 0; j < n_c; ++j) put(dc, static_cast<size_t>(k) * n_c + j, 1.0 / (z - e[n_v + j]));
    put(gw, static_cast<size_t>(k), weights[k] * g);
  }
  return kOk;
}

}  // namespace lrgw_host
