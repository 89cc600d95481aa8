// linalg.hpp — drop-in dense linear algebra (reference linalg.hpp:17-351) over
// the device: QRCP with the path's greedy pivots (swap-mirrored ties) and
// Householder Q / R leaves, partial-pivot LU with the reference's
// 1e-14 max|A| singularity rule, symmetric eigensolver (ascending).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "lrgw/matrix.hpp"
#include "lrgw/runtime.hpp"

namespace lrgw {

struct QrcpResult {
  Matrix q;               // m x k, orthonormal columns, k = min(m, n)
  Matrix r;               // k x n, upper triangular
  std::vector<int> perm;  // columns of A in selection order, length n
};

inline QrcpResult qrcp(const Matrix& a) {
  const int m = a.rows(), n = a.cols();
  if (m < 1 || n < 1) throw invalid_input("qrcp: empty matrix");
  const int k = std::min(m, n);
  QrcpResult out;
  out.q = Matrix(m, k);
  out.r = Matrix(k, n);
  std::vector<int32_t> perm(n);
  lrgw_ctx c = context();
  detail::check(lrgw_qrcp(c, a.data(), m, n, perm.data(), out.q.data(), out.r.data()), c, "qrcp");
  out.perm.assign(perm.begin(), perm.end());
  return out;
}

struct LuFactors {
  Matrix lu;             // unit-lower L and U
  std::vector<int> piv;  // row swapped with row i at step i
  double max_abs_input;  // the pivot threshold's scale
};

inline LuFactors lu_factor(const Matrix& a) {
  if (a.rows() != a.cols()) throw invalid_input("lu_factor: not square");
  const int n = a.rows();
  LuFactors f{Matrix(n, n), std::vector<int>(n), 0.0};
  if (n == 0) return f;
  std::vector<int32_t> piv(n);
  lrgw_ctx c = context();
  detail::check(lrgw_lu_factor(c, a.data(), n, f.lu.data(), piv.data(), &f.max_abs_input), c, "lu_factor");
  f.piv.assign(piv.begin(), piv.end());
  return f;
}

inline Matrix lu_solve_factored(const LuFactors& f, const Matrix& b) {
  const int n = f.lu.rows();
  if (b.rows() != n) throw invalid_input("lu_solve: rhs row mismatch");
  Matrix x(n, b.cols());
  if (n == 0 || b.cols() == 0) return x;
  std::vector<int32_t> piv(f.piv.begin(), f.piv.end());
  lrgw_ctx c = context();
  detail::check(lrgw_lu_solve_factored(c, f.lu.data(), piv.data(), n, b.data(), b.cols(), x.data()), c, "lu_solve");
  return x;
}

inline Matrix lu_solve(const Matrix& a, const Matrix& b) { return lu_solve_factored(lu_factor(a), b); }

inline Matrix lu_invert(const Matrix& a) { return lu_solve(a, Matrix::identity(a.rows())); }

struct SymEigResult {
  std::vector<double> values;  // ascending
  Matrix q;                    // eigenvectors in the columns
};

// Symmetrises; refuses a symmetry defect above 1e-8 ||A||_F (a caller bug,
// not roundoff) like the reference (linalg.hpp:307-316).
inline SymEigResult sym_eig(const Matrix& a) {
  if (a.rows() != a.cols()) throw invalid_input("sym_eig: not square");
  const int n = a.rows();
  if (n == 0) throw invalid_input("sym_eig: empty matrix");
  if (symmetry_defect(a) > 1e-8 * std::max(frobenius_norm(a), 1e-300))
    throw invalid_input("sym_eig: matrix is not symmetric");
  Matrix s = a;
  symmetrize(s);
  SymEigResult r{std::vector<double>(n), Matrix(n, n)};
  lrgw_ctx c = context();
  detail::check(lrgw_sym_eig(c, s.data(), n, r.values.data(), r.q.data()), c, "sym_eig");
  return r;
}

// Spectral norm of a symmetric matrix.
inline double sym_norm2(const Matrix& a) {
  SymEigResult ev = sym_eig(a);
  return std::max(std::abs(ev.values.front()), std::abs(ev.values.back()));
}

}  // namespace lrgw
