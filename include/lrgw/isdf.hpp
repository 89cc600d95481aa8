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

inline constexpr long long kPairMatrixGuard = 1LL << 26;

// Pair matrix M (N_r x N1 N2, column i + N1 j = psi_a(:, i) .* psi_b(:, j))
// and its transpose (isdf.hpp:49-88), materialised on the device behind the
// reference's 2^26-entry guard.
inline Matrix pair_matrix(const Matrix& psi_a, const Matrix& psi_b) {
  if (psi_a.rows() != psi_b.rows()) throw invalid_input("pair_matrix: row mismatch");
  Matrix m(psi_a.rows(), psi_a.cols() * psi_b.cols());
  lrgw_ctx c = context();
  detail::check(lrgw_pair_matrix(c, psi_a.data(), psi_b.data(), psi_a.rows(), psi_a.cols(), psi_b.cols(), 0,
                                 m.data()),
                c, "pair_matrix");
  return m;
}

inline Matrix pair_matrix_transposed(const Matrix& psi_a, const Matrix& psi_b) {
  if (psi_a.rows() != psi_b.rows()) throw invalid_input("pair_matrix_transposed: row mismatch");
  Matrix z(psi_a.cols() * psi_b.cols(), psi_a.rows());
  lrgw_ctx c = context();
  detail::check(lrgw_pair_matrix(c, psi_a.data(), psi_b.data(), psi_a.rows(), psi_a.cols(), psi_b.cols(), 1,
                                 z.data()),
                c, "pair_matrix_transposed");
  return z;
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

// The C factor: the pair matrix at the interpolation rows (isdf.hpp:185-191).
inline Matrix isdf_coefficients(const Matrix& psi_a, const Matrix& psi_b, const IsdfDecomposition& dec) {
  return pair_matrix(rows_at(psi_a, dec.point_indices), rows_at(psi_b, dec.point_indices));
}

// ||M - P C||_F / ||M||_F with M materialised (guarded; isdf.hpp:193-202).
inline double isdf_reconstruction_error(const Matrix& psi_a, const Matrix& psi_b, const IsdfDecomposition& dec) {
  const Matrix m = pair_matrix(psi_a, psi_b);
  const Matrix diff = m - matmul(dec.p, rows_at(m, dec.point_indices));
  return frobenius_norm(diff) / frobenius_norm(m);
}

// Descending singular values of the pair matrix from the eigenvalues of its
// smaller Gram matrix, truncated to max_terms (isdf.hpp:204-220).
inline std::vector<double> singular_value_report(const Matrix& psi_a, const Matrix& psi_b, int max_terms) {
  const Matrix m = pair_matrix(psi_a, psi_b);
  Matrix gram = (m.cols() <= m.rows()) ? matmul_tn(m, m) : matmul_nt(m, m);
  symmetrize(gram);
  const SymEigResult ev = sym_eig(gram);
  std::vector<double> sv;
  sv.reserve(ev.values.size());
  for (auto it = ev.values.rbegin(); it != ev.values.rend(); ++it) sv.push_back(std::sqrt(std::max(*it, 0.0)));
  if (max_terms >= 0 && static_cast<int>(sv.size()) > max_terms) sv.resize(max_terms);
  return sv;
}

}  // namespace lrgw
