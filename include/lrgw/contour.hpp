// contour.hpp — drop-in Cauchy/elliptic-contour quadrature of
// T = C Omega^-1 C^H (reference contour.hpp:23-329). Node geometry is host
// scalar code; every node term runs in the fused K3 DMMA kernel on the GPU.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "lrgw/elliptic.hpp"
#include "lrgw/matrix.hpp"
#include "lrgw/runtime.hpp"

namespace lrgw {

struct ContourSpec {
  double q = 0.0, big_q = 0.0, r = 0.0, big_r = 0.0, l = 0.0, e_shift = 0.0;
  double delta_rel = 1e-7;
  int max_nodes = 1025;
  bool bypass = false;
};

struct CoupledCoefficients {
  Matrix t;
  int nodes_used = 0;
  double est_rel_error = 0.0;
};

struct contour_convergence_error : numeric_error {
  contour_convergence_error(const std::string& msg, CoupledCoefficients b) : numeric_error(msg), best(std::move(b)) {}
  CoupledCoefficients best;
};

namespace detail {
inline void to7(const ContourSpec& s, double* o) {
  o[0] = s.q;
  o[1] = s.big_q;
  o[2] = s.r;
  o[3] = s.big_r;
  o[4] = s.l;
  o[5] = s.e_shift;
  o[6] = s.bypass ? 1.0 : 0.0;
}
inline void check_coupled(const Matrix& v, const Matrix& c, const std::vector<double>& e) {
  if (v.rows() != c.rows()) throw invalid_input("coupled_coefficients: point-row mismatch");
  if (static_cast<std::size_t>(v.cols() + c.cols()) > e.size())
    throw invalid_input("coupled_coefficients: not enough energies");
}
}  // namespace detail

inline ContourSpec elliptic_params(const std::vector<double>& energies, int n_v, int n_c, double delta_rel,
                                   int max_nodes = 1025) {
  double o[7];
  detail::check(lrgw_elliptic_params(energies.data(), static_cast<int>(energies.size()), n_v, n_c, delta_rel,
                                     max_nodes, o),
                nullptr, "elliptic_params");
  ContourSpec s;
  s.q = o[0];
  s.big_q = o[1];
  s.r = o[2];
  s.big_r = o[3];
  s.l = o[4];
  s.e_shift = o[5];
  s.bypass = o[6] != 0.0;
  s.delta_rel = delta_rel;
  s.max_nodes = max_nodes;
  return s;
}

inline double cauchy_error_bound(const ContourSpec& spec, int n_lambda) {
  double s7[7], out = 0.0;
  detail::to7(spec, s7);
  detail::check(lrgw_cauchy_error_bound(s7, n_lambda, &out), nullptr, "cauchy_error_bound: N_lambda < 1");
  return out;
}

inline CoupledCoefficients coupled_coefficients_direct(const Matrix& psi_v_pts, const Matrix& psi_c_pts,
                                                       const std::vector<double>& energies) {
  detail::check_coupled(psi_v_pts, psi_c_pts, energies);
  CoupledCoefficients out;
  out.t = Matrix(psi_v_pts.rows(), psi_v_pts.rows());
  lrgw_ctx c = context();
  detail::check(lrgw_coupled_coefficients_direct(c, psi_v_pts.data(), psi_c_pts.data(), psi_v_pts.rows(),
                                                 psi_v_pts.cols(), psi_c_pts.cols(), energies.data(),
                                                 static_cast<int>(energies.size()), out.t.data()),
                c, "coupled_coefficients_direct");
  return out;
}

// Fixed closed trapezoid of n_lambda intervals (the BASELINE configs' rule).
inline CoupledCoefficients coupled_coefficients_fixed(const Matrix& psi_v_pts, const Matrix& psi_c_pts,
                                                      const std::vector<double>& energies, int n_lambda) {
  detail::check_coupled(psi_v_pts, psi_c_pts, energies);
  CoupledCoefficients out;
  out.t = Matrix(psi_v_pts.rows(), psi_v_pts.rows());
  out.nodes_used = n_lambda + 1;
  lrgw_ctx c = context();
  detail::check(lrgw_coupled_coefficients_fixed(c, psi_v_pts.data(), psi_c_pts.data(), psi_v_pts.rows(),
                                                psi_v_pts.cols(), psi_c_pts.cols(), energies.data(),
                                                static_cast<int>(energies.size()), n_lambda, out.t.data()),
                c, "coupled_coefficients_fixed");
  return out;
}

inline CoupledCoefficients coupled_coefficients_contour(const Matrix& psi_v_pts, const Matrix& psi_c_pts,
                                                        const std::vector<double>& energies, const ContourSpec& spec,
                                                        int threads = 1) {
  (void)threads;
  detail::check_coupled(psi_v_pts, psi_c_pts, energies);
  if (spec.bypass) throw invalid_input("contour quadrature: spec is bypass-flagged; use the direct sum");
  CoupledCoefficients out;
  out.t = Matrix(psi_v_pts.rows(), psi_v_pts.rows());
  lrgw_ctx c = context();
  const int st = lrgw_coupled_coefficients_contour(
      c, psi_v_pts.data(), psi_c_pts.data(), psi_v_pts.rows(), psi_v_pts.cols(), psi_c_pts.cols(), energies.data(),
      static_cast<int>(energies.size()), spec.delta_rel, spec.max_nodes, out.t.data(), &out.nodes_used,
      &out.est_rel_error);
  if (st == LRGW_ERR_CONTOUR_CONVERGENCE)
    throw contour_convergence_error("coupled_coefficients_contour: did not reach delta_rel within max_nodes",
                                    std::move(out));
  detail::check(st, c, "coupled_coefficients_contour");
  return out;
}

inline std::vector<std::pair<int, Matrix>> contour_refinement_levels(const Matrix& psi_v_pts, const Matrix& psi_c_pts,
                                                                     const std::vector<double>& energies,
                                                                     const ContourSpec& spec, int max_level_nodes,
                                                                     int threads = 1) {
  (void)threads;
  (void)spec;
  detail::check_coupled(psi_v_pts, psi_c_pts, energies);
  const int n_mu = psi_v_pts.rows(), max_levels = 16;
  std::vector<double> buf(static_cast<std::size_t>(max_levels) * n_mu * n_mu);
  std::vector<int> counts(max_levels);
  int n_levels = 0;
  lrgw_ctx c = context();
  detail::check(lrgw_contour_refinement_levels(c, psi_v_pts.data(), psi_c_pts.data(), n_mu, psi_v_pts.cols(),
                                               psi_c_pts.cols(), energies.data(), static_cast<int>(energies.size()),
                                               max_level_nodes, max_levels, buf.data(), counts.data(), &n_levels),
                c, "contour_refinement_levels");
  std::vector<std::pair<int, Matrix>> out;
  for (int i = 0; i < n_levels; ++i) {
    Matrix t(n_mu, n_mu);
    std::copy(buf.begin() + static_cast<std::ptrdiff_t>(i) * n_mu * n_mu,
              buf.begin() + static_cast<std::ptrdiff_t>(i + 1) * n_mu * n_mu, t.data());
    out.emplace_back(counts[i], std::move(t));
  }
  return out;
}

}  // namespace lrgw
