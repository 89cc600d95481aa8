// model.hpp — drop-in electronic-structure container and Coulomb operator
// (reference model.hpp:27-50, 151-223) and the WFN1 file format
// (model.hpp:236-339). apply_coulomb runs on the GPU (cuFFT
// leaf + the fused v(G)/N_r scale kernel).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "lrgw/dft.hpp"
#include "lrgw/grid.hpp"
#include "lrgw/linalg.hpp"
#include "lrgw/matrix.hpp"
#include "lrgw/rng.hpp"
#include "lrgw/runtime.hpp"

namespace lrgw {

struct ElectronicStructure {
  Grid grid;
  Matrix psi;                    // N_r x (N_v + N_c)
  std::vector<double> energies;  // ascending
  std::vector<double> vxc;
  int n_v = 0;
  int n_c = 0;
  int n_bands() const { return n_v + n_c; }
  double gap() const { return energies[n_v] - energies[n_v - 1]; }
  Matrix occupied() const { return cols_block(psi, 0, n_v); }
  Matrix unoccupied() const { return cols_block(psi, n_v, n_c); }
  // ||psi^T psi dV - I||_F (model.hpp:41-49)
  double orthonormality_defect() const {
    Matrix g = matmul_tn(psi, psi);
    const double dv = grid.dv();
    for (int j = 0; j < g.cols(); ++j) {
      for (int i = 0; i < g.rows(); ++i) g(i, j) *= dv;
      g(j, j) -= 1.0;
    }
    return frobenius_norm(g);
  }
};

// Seeded synthetic stand-in for KS-DFT output (model.hpp:52-116): band-limited
// Gaussian random fields (Gaussian envelope of width a third of the smallest
// Nyquist |G| on complex normal coefficients, the real part of the inverse
// unitary DFT), orthonormalised by QRCP against the dV-weighted inner product;
// occupied energies equispaced on [-bandwidth, 0], unoccupied on
// [gap, gap + bandwidth]. The transforms and the QR run on the device.
inline ElectronicStructure build_synthetic_system(std::uint64_t seed, const Grid& grid, int n_v, int n_c, double gap,
                                                  double bandwidth) {
  if (!(gap > 0.0)) throw invalid_input("build_synthetic_system: gap must be > 0");
  if (!(bandwidth >= gap)) throw invalid_input("build_synthetic_system: bandwidth must be >= gap");
  if (n_v < 1 || n_c < 1) throw invalid_input("build_synthetic_system: need n_v >= 1 and n_c >= 1");
  const int n_r = grid.n_r(), nb = n_v + n_c;
  if (nb > n_r) throw invalid_input("build_synthetic_system: grid too small for band count");
  Rng rng(seed);
  double g_nyq = 1e300;
  for (int k = 0; k < 3; ++k) g_nyq = std::min(g_nyq, 3.14159265358979323846 * grid.dims[k] / grid.cell[k]);
  const double sigma2 = (g_nyq / 3.0) * (g_nyq / 3.0);
  std::vector<double> env(n_r);
  for (int idx = 0; idx < n_r; ++idx) env[idx] = std::exp(-grid.g_norm2(idx) / (2.0 * sigma2));
  Matrix fields(n_r, nb);
  std::vector<cplx> coef(n_r);
  for (int b = 0; b < nb; ++b) {
    for (int idx = 0; idx < n_r; ++idx) {
      // the same expression as model.hpp:84: C++ leaves the order of the two
      // draws to the compiler (GCC evaluates the imaginary argument first),
      // so the drop-in inherits whatever order the reference's build gets
      coef[idx] = env[idx] * cplx(rng.gaussian(), rng.gaussian());
    }
    const std::vector<cplx> field = dft(grid, coef, DftDirection::inverse);
    for (int idx = 0; idx < n_r; ++idx) fields(idx, b) = field[idx].real();
  }
  QrcpResult qr = qrcp(fields);
  for (int j = 0; j < nb; ++j)
    if (std::abs(qr.r(j, j)) < 1e-12)
      throw numeric_error("build_synthetic_system: random fields are rank deficient; grid too small for band count");
  const double inv_sqrt_dv = 1.0 / std::sqrt(grid.dv());
  ElectronicStructure es;
  es.grid = grid;
  es.psi = Matrix(n_r, nb);
  for (int j = 0; j < nb; ++j)
    for (int i = 0; i < n_r; ++i) es.psi(i, j) = qr.q(i, j) * inv_sqrt_dv;
  es.n_v = n_v;
  es.n_c = n_c;
  es.energies.resize(nb);
  for (int i = 0; i < n_v; ++i) es.energies[i] = (n_v == 1) ? 0.0 : -bandwidth * (n_v - 1 - i) / double(n_v - 1);
  for (int j = 0; j < n_c; ++j) es.energies[n_v + j] = gap + ((n_c == 1) ? 0.0 : bandwidth * j / double(n_c - 1));
  es.vxc.assign(nb, 0.0);
  return es;
}

// Occupied-unoccupied energy differences, pair (i, j) at i + n_v j (model.hpp:118-145).
struct OmegaDiagonal {
  std::vector<double> entries;
  double min_abs() const {
    double m = 1e300;
    for (double v : entries) m = std::min(m, std::abs(v));
    return m;
  }
};

inline OmegaDiagonal build_omega(const ElectronicStructure& es) {
  OmegaDiagonal w;
  w.entries.resize(static_cast<std::size_t>(es.n_v) * es.n_c);
  for (int j = 0; j < es.n_c; ++j)
    for (int i = 0; i < es.n_v; ++i) {
      const double d = es.energies[i] - es.energies[es.n_v + j];
      if (!(d < 0.0)) throw invalid_input("build_omega: system is not gapped");
      w.entries[i + static_cast<std::size_t>(es.n_v) * j] = d;
    }
  return w;
}

enum class CoulombMode { reciprocal_diagonal, dense };

struct CoulombOperator {
  Grid grid;
  CoulombMode mode = CoulombMode::reciprocal_diagonal;
  std::vector<double> kernel;  // v(G), length N_r
  Matrix dense;                // only populated for dense mode
  bool zero = false;           // made by zero_coulomb()
};

inline constexpr int kDenseCoulombGuard = 4096;

// V X column by column (model.hpp:208-223): dense mode multiplies; otherwise
// F^-1 diag(v.kernel) F on the device with the operator's OWN kernel array
// (a caller may edit it), the analytic 4 pi / |G|^2 kernel through its fused
// on-device path.
inline Matrix apply_coulomb(const CoulombOperator& v, const Matrix& x, int threads = 1);

inline CoulombOperator build_coulomb(const Grid& grid, CoulombMode mode) {
  CoulombOperator v;
  v.grid = grid;
  v.mode = mode;
  v.kernel.resize(grid.n_r());
  detail::check(lrgw_coulomb_kernel(grid.dims.data(), grid.cell.data(), v.kernel.data()), nullptr,
                "build_coulomb");
  if (mode == CoulombMode::dense) {
    if (grid.n_r() > kDenseCoulombGuard)
      throw guard_exceeded("build_coulomb: dense mode refused for N_r > " + std::to_string(kDenseCoulombGuard));
    CoulombOperator r = v;
    r.mode = CoulombMode::reciprocal_diagonal;
    v.dense = apply_coulomb(r, Matrix::identity(grid.n_r()));
    symmetrize(v.dense);
  }
  return v;
}

inline CoulombOperator zero_coulomb(const Grid& grid) {
  CoulombOperator v;
  v.grid = grid;
  v.kernel.assign(grid.n_r(), 0.0);
  v.zero = true;
  return v;
}

namespace detail {
// The fused device paths take (dims, cell, zero): valid when the kernel is
// the analytic one of the grid (or all zero).
inline bool analytic_kernel(const CoulombOperator& v) {
  if (v.mode == CoulombMode::dense) return false;
  if (static_cast<int>(v.kernel.size()) != v.grid.n_r()) return false;
  bool all_zero = true;
  for (double k : v.kernel) all_zero = all_zero && k == 0.0;
  if (all_zero) return true;
  if (v.zero) return false;
  std::vector<double> ref(v.grid.n_r());
  detail::check(lrgw_coulomb_kernel(v.grid.dims.data(), v.grid.cell.data(), ref.data()), nullptr, "build_coulomb");
  return ref == v.kernel;
}
inline int zero_flag(const CoulombOperator& v) {
  for (double k : v.kernel)
    if (k != 0.0) return 0;
  return 1;
}
}  // namespace detail

inline Matrix apply_coulomb(const CoulombOperator& v, const Matrix& x, int threads) {
  (void)threads;
  if (x.rows() != v.grid.n_r()) throw invalid_input("apply_coulomb: row count != N_r");
  if (v.mode == CoulombMode::dense) return matmul(v.dense, x);
  Matrix y(x.rows(), x.cols());
  if (x.cols() == 0) return y;
  if (static_cast<int>(v.kernel.size()) != v.grid.n_r()) throw invalid_input("apply_coulomb: kernel length != N_r");
  lrgw_ctx c = context();
  if (detail::analytic_kernel(v))
    detail::check(lrgw_apply_coulomb(c, v.grid.dims.data(), v.grid.cell.data(), detail::zero_flag(v), x.data(),
                                     x.cols(), y.data()),
                  c, "apply_coulomb");
  else
    detail::check(lrgw_apply_coulomb_kernel(c, v.grid.dims.data(), v.kernel.data(), x.data(), x.cols(), y.data()), c,
                  "apply_coulomb");
  return y;
}

// Dense V regardless of mode, guarded (model.hpp:225-234).
inline Matrix coulomb_dense_matrix(const CoulombOperator& v) {
  if (v.mode == CoulombMode::dense) return v.dense;
  if (v.grid.n_r() > kDenseCoulombGuard) throw guard_exceeded("coulomb_dense_matrix: N_r exceeds dense guard");
  Matrix d = apply_coulomb(v, Matrix::identity(v.grid.n_r()));
  symmetrize(d);
  return d;
}

// WFN1 files (model.hpp:236-339): the same bytes and io_error messages as the
// reference; I/O in liblrgw_cuda (csrc/wfn1.cpp).
inline void save_system(const std::string& path, const ElectronicStructure& es) {
  if (es.psi.rows() != es.grid.n_r() || es.psi.cols() != es.n_bands() ||
      static_cast<int>(es.energies.size()) != es.n_bands() || static_cast<int>(es.vxc.size()) != es.n_bands())
    throw invalid_input("save_system: array shapes do not match the header");
  if (lrgw_wfn1_save(path.c_str(), es.grid.dims.data(), es.grid.cell.data(), es.n_v, es.n_c, es.psi.data(),
                     es.energies.data(), es.vxc.data()) != LRGW_OK)
    throw io_error(lrgw_last_error());
}

inline ElectronicStructure load_system(const std::string& path) {
  std::array<int, 3> dims{};
  std::array<double, 3> cell{};
  int n_v = 0, n_c = 0;
  if (lrgw_wfn1_info(path.c_str(), dims.data(), cell.data(), &n_v, &n_c) != LRGW_OK) throw io_error(lrgw_last_error());
  ElectronicStructure es;
  es.grid = Grid(dims, cell);
  es.n_v = n_v;
  es.n_c = n_c;
  es.psi = Matrix(es.grid.n_r(), n_v + n_c);
  es.energies.resize(n_v + n_c);
  es.vxc.resize(n_v + n_c);
  if (lrgw_wfn1_load(path.c_str(), es.psi.data(), es.energies.data(), es.vxc.data()) != LRGW_OK)
    throw io_error(lrgw_last_error());
  return es;
}

}  // namespace lrgw
