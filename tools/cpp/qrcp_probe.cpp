// Diagnostic: the synthetic-system fields of build_synthetic_system
// (model.hpp:56-116) for the si8-shaped gw test system and their QRCP
// pivots / R diagonal, printed for a reference-vs-drop-in diff.
#include <cstdio>

#include "lrgw/gw.hpp"

using namespace lrgw;

int main(int argc, char** argv) {
  const int nb = 32;
  Grid grid({8, 8, 8}, {6.0, 6.0, 6.0});
  const int n_r = grid.n_r();
  Rng rng(1);
  double g_nyq = 1e300;
  for (int k = 0; k < 3; ++k) g_nyq = std::min(g_nyq, 3.14159265358979323846 * grid.dims[k] / grid.cell[k]);
  const double sigma2 = (g_nyq / 3.0) * (g_nyq / 3.0);
  Matrix fields(n_r, nb);
  std::vector<cplx> coef(n_r);
  for (int b = 0; b < nb; ++b) {
    for (int idx = 0; idx < n_r; ++idx) {
      const double env = std::exp(-grid.g_norm2(idx) / (2.0 * sigma2));
      const double re = rng.gaussian(), im = rng.gaussian();
      coef[idx] = env * cplx(re, im);
    }
    std::vector<cplx> f = dft(grid, coef, DftDirection::inverse);
    for (int idx = 0; idx < n_r; ++idx) fields(idx, b) = f[idx].real();
  }
  for (int b = 0; b < nb; ++b) {
    double s = 0.0;
    for (int i = 0; i < n_r; ++i) s += fields(i, b) * fields(i, b);
    std::printf("col %2d norm2 %.17g first %.17g\n", b, s, fields(0, b));
  }
  QrcpResult qr = qrcp(fields);
  for (int j = 0; j < nb; ++j) std::printf("piv %2d -> %2d r %.17g q00 %.17g\n", j, qr.perm[j], qr.r(j, j), qr.q(0, j));
  return 0;
}
