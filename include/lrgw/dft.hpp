// dft.hpp — drop-in unitary 3-D DFT on the periodic grid (reference
// dft.hpp:18-68): forward exp(-2 pi i k.r / n), inverse exp(+...), each
// scaled by 1 / sqrt(N_r); a cuFFT Z2Z leaf on the device.
#pragma once

#include <cmath>
#include <complex>
#include <vector>

#include "lrgw/grid.hpp"
#include "lrgw/runtime.hpp"

namespace lrgw {

using cplx = std::complex<double>;

enum class DftDirection { forward, inverse };

// The n x n unitary DFT matrix of one axis, row-major (dft.hpp:18-35).
inline std::vector<cplx> dft_twiddles(int n, DftDirection dir) {
  std::vector<cplx> w(static_cast<std::size_t>(n) * n);
  const double sign = dir == DftDirection::forward ? -1.0 : 1.0, scale = 1.0 / std::sqrt(double(n));
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j) {
      const double ang = sign * 6.283185307179586476925286766559 * double((long long)k * j % n) / n;
      w[static_cast<std::size_t>(k) * n + j] = scale * cplx(std::cos(ang), std::sin(ang));
    }
  return w;
}

inline std::vector<cplx> dft(const Grid& grid, const std::vector<cplx>& x, DftDirection dir) {
  if (static_cast<int>(x.size()) != grid.n_r()) throw invalid_input("dft: size mismatch");
  std::vector<cplx> y(x.size());
  lrgw_ctx c = context();
  detail::check(lrgw_dft(c, grid.dims.data(), reinterpret_cast<const double*>(x.data()),
                         dir == DftDirection::inverse ? 1 : 0, reinterpret_cast<double*>(y.data())),
                c, "dft");
  return y;
}

}  // namespace lrgw
