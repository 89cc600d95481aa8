// isdf.hpp — drop-in ISDF for the vc pair set (reference isdf.hpp:16-183):
// point selection (K1) and the auxiliary-basis fit (K2) on the GPU.
#pragma once

#include <algorithm>
#include <cstdint>
#include <utility>
#include <vector>

#include "lrgw/matrix.hpp"
#include "lrgw/model.hpp"
#include "lrgw/runtime.hpp"

namespace lrgw {

enum class PairSetLabel { vc, vn, nn };
enum class PointSelector { qrcp_direct, qrcp_sketched };

inline const char* to_string(PairSetLabel l) {
  switch (l) {
    case PairSetLabel::vc: return "vc";
    case PairSetLabel::vn: return "vn";
    default: return "nn";
  }
}

struct IsdfDecomposition {
  PairSetLabel label = PairSetLabel::vc;
  double k_mu = 0.0;
  int n_mu = 0;
  std::vector<int> point_indices;  // strictly increasing grid indices
  Matrix p;                        // N_r x N_mu
};

inline int num_aux(double k_mu, int n1, int n2) {
  int out = 0;
  detail::check(lrgw_num_aux(k_mu, n1, n2, &out), nullptr, "num_aux: k_mu must be > 0");
  return out;
}

inline std::vector<int> select_interpolation_points(const Matrix& psi_a, const Matrix& psi_b, int n_mu,
                                                    PointSelector method = PointSelector::qrcp_direct) {
  if (psi_a.rows() != psi_b.rows()) throw invalid_input("pair_matrix_transposed: row mismatch");
  std::vector<int32_t> pts(std::max(n_mu, 0));
  lrgw_ctx c = context();
  detail::check(lrgw_select_interpolation_points(
                    c, psi_a.data(), psi_b.data(), psi_a.rows(), psi_a.cols(), psi_b.cols(), n_mu,
                    method == PointSelector::qrcp_sketched ? LRGW_QRCP_SKETCHED : LRGW_QRCP_DIRECT, pts.data()),
                c, "select_interpolation_points");
  return std::vector<int>(pts.begin(), pts.end());
}

inline IsdfDecomposition fit_auxiliary_basis(const Matrix& psi_a, const Matrix& psi_b, const std::vector<int>& points,
                                             PairSetLabel label = PairSetLabel::vc, double k_mu = 0.0) {
  if (psi_a.rows() != psi_b.rows()) throw invalid_input("fit_auxiliary_basis: row mismatch");
  IsdfDecomposition d;
  d.label = label;
  d.k_mu = k_mu;
  d.n_mu = static_cast<int>(points.size());
  d.point_indices = points;
  d.p = Matrix(psi_a.rows(), d.n_mu);
  std::vector<int32_t> pts(points.begin(), points.end());
  lrgw_ctx c = context();
  detail::check(lrgw_fit_auxiliary_basis(c, psi_a.data(), psi_b.data(), psi_a.rows(), psi_a.cols(), psi_b.cols(),
                                         pts.empty() ? nullptr : pts.data(), d.n_mu, d.p.data()),
                c, "fit_auxiliary_basis");
  return d;
}

inline std::pair<Matrix, Matrix> pair_factors(const ElectronicStructure& es, PairSetLabel label) {
  switch (label) {
    case PairSetLabel::vc: return {es.occupied(), es.unoccupied()};
    case PairSetLabel::vn: return {es.occupied(), es.psi};
    default: return {es.psi, es.psi};
  }
}

inline IsdfDecomposition build_isdf(const ElectronicStructure& es, PairSetLabel label, double k_mu,
                                    PointSelector method = PointSelector::qrcp_direct) {
  auto [a, b] = pair_factors(es, label);
  const int n_mu = std::clamp(num_aux(k_mu, a.cols(), b.cols()), 1, es.grid.n_r());
  return fit_auxiliary_basis(a, b, select_interpolation_points(a, b, n_mu, method), label, k_mu);
}

}  // namespace lrgw
