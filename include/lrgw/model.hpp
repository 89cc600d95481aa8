// model.hpp — drop-in electronic-structure container and Coulomb operator
// (reference model.hpp:27-50, 151-223). apply_coulomb runs on the GPU (cuFFT
// leaf + the fused v(G)/N_r scale kernel).
#pragma once

#include <vector>

#include "lrgw/grid.hpp"
#include "lrgw/matrix.hpp"
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
};

enum class CoulombMode { reciprocal_diagonal, dense };

struct CoulombOperator {
  Grid grid;
  CoulombMode mode = CoulombMode::reciprocal_diagonal;
  std::vector<double> kernel;  // v(G), length N_r
  Matrix dense;                // unused on the B200 path
  bool zero = false;           // zero_coulomb()
};

inline constexpr int kDenseCoulombGuard = 4096;

inline CoulombOperator build_coulomb(const Grid& grid, CoulombMode mode) {
  if (mode == CoulombMode::dense && grid.n_r() > kDenseCoulombGuard)
    throw guard_exceeded("build_coulomb: dense mode refused for N_r > 4096");
  CoulombOperator v;
  v.grid = grid;
  v.mode = mode;
  v.kernel.resize(grid.n_r());
  detail::check(lrgw_coulomb_kernel(grid.dims.data(), grid.cell.data(), v.kernel.data()), nullptr,
                "build_coulomb");
  return v;
}

inline CoulombOperator zero_coulomb(const Grid& grid) {
  CoulombOperator v;
  v.grid = grid;
  v.kernel.assign(grid.n_r(), 0.0);
  v.zero = true;
  return v;
}

// V X column by column; `threads` is kept for signature parity (host-only).
inline Matrix apply_coulomb(const CoulombOperator& v, const Matrix& x, int threads = 1) {
  (void)threads;
  if (x.rows() != v.grid.n_r()) throw invalid_input("apply_coulomb: row count != N_r");
  Matrix y(x.rows(), x.cols());
  if (x.cols() == 0) return y;
  lrgw_ctx c = context();
  detail::check(lrgw_apply_coulomb(c, v.grid.dims.data(), v.grid.cell.data(), v.zero ? 1 : 0, x.data(), x.cols(),
                                   y.data()),
                c, "apply_coulomb");
  return y;
}

}  // namespace lrgw
