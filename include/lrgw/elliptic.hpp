// elliptic.hpp — drop-in scalar elliptic helpers (reference elliptic.hpp:17-118)
// over the C-ABI's host implementations.
#pragma once

#include <complex>

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

}  // namespace lrgw
