// model.hpp — drop-in electronic-structure container and Coulomb operator
// (reference model.hpp:27-50, 151-223) and the WFN1 file format
// (model.hpp:236-339). apply_coulomb runs on the GPU (cuFFT
// leaf + the fused v(G)/N_r scale kernel).
#pragma once

#include <string>
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
