// elliptic.hpp — drop-in scalar elliptic helpers (reference elliptic.hpp:17-118)
// over the C-ABI's host implementations.
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <functional>

#include "lrgw/runtime.hpp"

namespace lrgw {

struct JacobiTriple {
  double sn, cn, dn;
};
struct JacobiComplexTriple {
  std::complex<double> sn, cn, dn;
};

inline double elliptic_k(double k) {
  double out = 0.0;
  detail::check(lrgw_elliptic_k(k, &out), nullptr, "elliptic_k: modulus must be in [0, 1)");
  return out;
}

inline JacobiTriple jacobi_sn_cn_dn(double u, double k) {
  double o[3];
  detail::check(lrgw_jacobi_sn_cn_dn(u, k, o), nullptr, "jacobi_sn_cn_dn: modulus must be in [0, 1)");
  return {o[0], o[1], o[2]};
}

inline JacobiComplexTriple jacobi_complex(std::complex<double> u, double k) {
  double o[6];
  detail::check(lrgw_jacobi_complex(u.real(), u.imag(), k, o), nullptr, "jacobi_complex");
  return {{o[0], o[1]}, {o[2], o[3]}, {o[4], o[5]}};
}

// Arithmetic-geometric mean (elliptic.hpp:17-26): iterate until the means
// stop moving in floating point.
inline double agm(double a, double b) {
  for (int it = 0; it < 64 && a != b; ++it) {
    const double m = 0.5 * (a + b), g = std::sqrt(a * b);
    if (m == a || m == b) break;
    a = m;
    b = g;
  }
  return 0.5 * (a + b);
}

// Adaptive quadrature of a smooth integrand to a relative tolerance
// (elliptic.hpp:120-193's contract): Gauss-Kronrod (7, 15) pairs with
// bisection of any interval whose |K15 - G7| exceeds its share of the
// tolerance. Host scalar helper (the contour height itself comes from the
// closed form in csrc/elliptic.cpp).
namespace detail {
struct Gk15 {
  // Kronrod abscissae (positive half, descending) and weights; the odd
  // entries 1, 3, 5 and the centre are the 7-point Gauss nodes
  static constexpr double x[8] = {0.991455371120812639206854697526329, 0.949107912342758524526189684047851,
                                  0.864864423359769072789712788640926, 0.741531185599394439863864773280788,
                                  0.586087235467691130294144845693013, 0.405845151377397166906606412076961,
                                  0.207784955007898467600689403773245, 0.0};
  static constexpr double wk[8] = {0.022935322010529224963732008058970, 0.063092092629978553290700663189204,
                                   0.104790010322250183839876322541518, 0.140653259715525918745189590510238,
                                   0.169004726639267902826583426598550, 0.190350578064785409913256402421014,
                                   0.204432940075298892414161999234649, 0.209482141084727828012999174891714};
  static constexpr double wg[4] = {0.129484966168869693270611432679082, 0.279705391489276667901467771423780,
                                   0.381830050505118944950369775488975, 0.417959183673469387755102040816327};
};
inline void gk15(const std::function<double(double)>& f, double a, double b, double* k15, double* g7) {
  const double c = 0.5 * (a + b), h = 0.5 * (b - a);
  const double fc = f(c);
  double sk = Gk15::wk[7] * fc, sg = Gk15::wg[3] * fc;
  for (int i = 0; i < 7; ++i) {
    const double fs = f(c - h * Gk15::x[i]) + f(c + h * Gk15::x[i]);
    sk += Gk15::wk[i] * fs;
    if (i % 2 == 1) sg += Gk15::wg[i / 2] * fs;
  }
  *k15 = sk * h;
  *g7 = sg * h;
}
inline double gk_adapt(const std::function<double(double)>& f, double a, double b, double tol, int depth) {
  double k, g;
  gk15(f, a, b, &k, &g);
  if (std::abs(k - g) <= tol * std::max(1.0, std::abs(k)) || depth >= 48) return k;
  const double m = 0.5 * (a + b);
  return gk_adapt(f, a, m, 0.5 * tol, depth + 1) + gk_adapt(f, m, b, 0.5 * tol, depth + 1);
}
}  // namespace detail

inline double integrate_adaptive(const std::function<double(double)>& f, double a, double b,
                                 double rel_tol = 1e-13) {
  return detail::gk_adapt(f, a, b, rel_tol, 0);
}

}  // namespace lrgw
