// contour.hpp — drop-in Cauchy/elliptic-contour quadrature of
// T = C Omega^-1 C^H (reference contour.hpp:23-329). Node geometry is host
// scalar code; every node term runs in the fused K3 DMMA kernel on the GPU.
#pragma once

#include <cmath>
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

namespace detail {

// acc = sum_k w_k term_k on the device (the fused K3 kernel; contour.hpp:185-222).
inline Matrix sum_node_terms(const Matrix& psi_v_pts, const Matrix& psi_c_pts, const std::vector<double>& energies,
                             const ContourSpec& spec, const std::vector<double>& nodes,
                             const std::vector<double>& weights, int threads = 1) {
  (void)threads;
  check_coupled(psi_v_pts, psi_c_pts, energies);
  if (nodes.size() != weights.size()) throw invalid_input("sum_node_terms: nodes / weights length mismatch");
  Matrix acc(psi_v_pts.rows(), psi_v_pts.rows());
  if (nodes.empty()) return acc;
  double s7[7];
  to7(spec, s7);
  lrgw_ctx c = context();
  detail::check(lrgw_sum_node_terms(c, psi_v_pts.data(), psi_c_pts.data(), psi_v_pts.rows(), psi_v_pts.cols(),
                                    psi_c_pts.cols(), energies.data(), static_cast<int>(energies.size()), s7,
                                    nodes.data(), weights.data(), static_cast<int>(nodes.size()), acc.data()),
                c, "sum_node_terms");
  return acc;
}

// Im(g J(z(t + iL))) at one parameter node (contour.hpp:140-183).
inline Matrix contour_node_term(const Matrix& psi_v_pts, const Matrix& psi_c_pts, const std::vector<double>& energies,
                                const ContourSpec& spec, double t_node) {
  return sum_node_terms(psi_v_pts, psi_c_pts, energies, spec, {t_node}, {1.0});
}

}  // namespace detail

// Nested trapezoid levels of 2^m + 1 nodes, m = 4, 5, ... on [-R, R] of the
// given spec; each level evaluates only its new midpoints on the device
// (running = running / 2 + new, T = pref running, symmetrised); the visitor
// gets (node count, T) and returns false to stop (contour.hpp:224-279).
template <typename Visitor>
void visit_contour_levels(const Matrix& psi_v_pts, const Matrix& psi_c_pts, const std::vector<double>& energies,
                          const ContourSpec& spec, int max_level_nodes, int threads, Visitor&& visit) {
  detail::check_coupled(psi_v_pts, psi_c_pts, energies);
  if (spec.bypass) throw invalid_input("contour quadrature: spec is bypass-flagged; use the direct sum");
  if ((1 << 4) + 1 > max_level_nodes) throw invalid_input("contour quadrature: node cap below one level");
  const double pref = 2.0 * std::sqrt(spec.q * spec.big_q) / (3.14159265358979323846 * spec.r);
  Matrix running;
  for (int m = 4;; ++m) {
    const int n_nodes = (1 << m) + 1;
    if (n_nodes > max_level_nodes) break;
    const double h = 2.0 * spec.big_r / (n_nodes - 1);
    std::vector<double> nodes, weights;
    const bool first = running.empty();
    for (int k = first ? 0 : 1; k < n_nodes; k += first ? 1 : 2) {
      nodes.push_back(-spec.big_r + k * h);
      weights.push_back((first && (k == 0 || k == n_nodes - 1)) ? 0.5 * h : h);
    }
    Matrix add = detail::sum_node_terms(psi_v_pts, psi_c_pts, energies, spec, nodes, weights, threads);
    running = first ? std::move(add) : 0.5 * running + add;
    Matrix t = pref * running;
    symmetrize(t);
    if (!visit(n_nodes, std::move(t))) break;
  }
}

// Every level's estimate up to the node cap, on the given spec (contour.hpp:281-294).
inline std::vector<std::pair<int, Matrix>> contour_refinement_levels(const Matrix& psi_v_pts, const Matrix& psi_c_pts,
                                                                     const std::vector<double>& energies,
                                                                     const ContourSpec& spec, int max_level_nodes,
                                                                     int threads = 1) {
  std::vector<std::pair<int, Matrix>> levels;
  visit_contour_levels(psi_v_pts, psi_c_pts, energies, spec, max_level_nodes, threads, [&](int n, Matrix t) {
    levels.emplace_back(n, std::move(t));
    return true;
  });
  return levels;
}

// Adaptive refinement to spec.delta_rel within spec.max_nodes; on failure
// contour_convergence_error carries the best estimate (contour.hpp:296-329).
inline CoupledCoefficients coupled_coefficients_contour(const Matrix& psi_v_pts, const Matrix& psi_c_pts,
                                                        const std::vector<double>& energies, const ContourSpec& spec,
                                                        int threads = 1) {
  CoupledCoefficients best;
  bool converged = false;
  Matrix prev;
  visit_contour_levels(psi_v_pts, psi_c_pts, energies, spec, spec.max_nodes, threads, [&](int n_nodes, Matrix t) {
    if (prev.empty()) {
      best = CoupledCoefficients{t, n_nodes, 1.0};
      prev = std::move(t);
      return true;
    }
    const double rel = frobenius_norm(t - prev) / std::max(frobenius_norm(t), 1e-300);
    best = CoupledCoefficients{t, n_nodes, rel};
    prev = std::move(t);
    if (rel <= spec.delta_rel) {
      converged = true;
      return false;
    }
    return true;
  });
  if (!converged)
    throw contour_convergence_error("coupled_coefficients_contour: did not reach delta_rel within max_nodes",
                                    std::move(best));
  return best;
}

}  // namespace lrgw
