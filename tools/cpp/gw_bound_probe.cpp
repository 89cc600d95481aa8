// Diagnostic: the quantities behind the reference test "error bound holds on
// the si8-shaped system at k = 8" (test_gw.cpp:292-300), printed so the same
// source compiled against the reference headers (CPU) and against the
// drop-in (include/lrgw over liblrgw_cuda.so) can be diffed stage by stage.
#include <cstdio>
#include <functional>

#include "lrgw/gw.hpp"

using namespace lrgw;

static unsigned long long hash_idx(const std::vector<int>& v) {
  unsigned long long h = 1469598103934665603ULL;
  for (int x : v) h = (h ^ (unsigned)x) * 1099511628211ULL;
  return h;
}

int main() {
  Grid grid({8, 8, 8}, {6.0, 6.0, 6.0});
  ElectronicStructure es = build_synthetic_system(1, grid, 16, 16, 1.0, 4.0);
  CoulombOperator v = build_coulomb(grid, CoulombMode::reciprocal_diagonal);
  {
    double e = 0.0;
    for (double x : es.energies) e += x;
    std::printf("psi fro %.17g energies sum %.17g\n", frobenius_norm(es.psi), e);
    Matrix vd = coulomb_dense_matrix(v);
    std::printf("v dense fro %.17g v00 %.17g v10 %.17g\n", frobenius_norm(vd), vd(0, 0), vd(1, 0));
    OmegaDiagonal om = build_omega(es);
    Matrix m = pair_matrix(es.occupied(), es.unoccupied());
    Matrix chi = chi_dense_exact(es, om);
    Matrix vchi = apply_coulomb(v, chi);
    Matrix vm = apply_coulomb(v, m);
    std::printf("pair fro %.17g chi fro %.17g chi00 %.17g vchi fro %.17g vchi00 %.17g vchi01 %.17g vm fro %.17g\n",
                frobenius_norm(m), frobenius_norm(chi), chi(0, 0), frobenius_norm(vchi), vchi(0, 0), vchi(0, 1),
                frobenius_norm(vm));
    Matrix eye = Matrix::identity(grid.n_r());
    Matrix veye = apply_coulomb(v, eye);
    std::printf("V I fro %.17g V00 %.17g V10 %.17g\n", frobenius_norm(veye), veye(0, 0), veye(1, 0));
    EpsilonDense d = epsilon_dense_oracle(es, v, nullptr);
    double tr = 0.0;
    for (int i = 0; i < d.eps_inv.rows(); ++i) tr += d.eps_inv(i, i);
    std::printf("eps_inv fro %.17g trace %.17g e00 %.17g e10 %.17g\n", frobenius_norm(d.eps_inv), tr, d.eps_inv(0, 0),
                d.eps_inv(1, 0));
  }
  IsdfDecomposition vc = build_isdf(es, PairSetLabel::vc, 8.0);
  IsdfDecomposition vn = build_isdf(es, PairSetLabel::vn, 8.0);
  IsdfDecomposition nn = build_isdf(es, PairSetLabel::nn, 8.0);
  std::printf("points vc %zu %016llx vn %zu %016llx nn %zu %016llx\n", vc.point_indices.size(),
              hash_idx(vc.point_indices), vn.point_indices.size(), hash_idx(vn.point_indices),
              nn.point_indices.size(), hash_idx(nn.point_indices));
  std::printf("theta fro vc %.17g vn %.17g nn %.17g\n", frobenius_norm(vc.p), frobenius_norm(vn.p),
              frobenius_norm(nn.p));
  SelfEnergies exact = self_energies_bruteforce(es, v);
  SelfEnergies isdf = self_energies_isdf_conventional(es, v, vc, vn, nn);
  for (int n = 0; n < es.n_bands(); ++n)
    std::printf("band %2d exact %.17g isdf %.17g\n", n, exact.sigma_total[n], isdf.sigma_total[n]);
  ErrorBoundReport rep = isdf_error_bound_check(es, v, vc, vn, nn);
  std::printf("dx_norm %.17g dm_fro %.17g all_within %d\n", rep.delta_x_norm, rep.delta_m_fro, (int)rep.all_within);
  for (std::size_t n = 0; n < rep.bands.size(); ++n)
    std::printf("bound %2zu observed %.6e bound %.6e slack %.6e within %d\n", n, rep.bands[n].observed,
                rep.bands[n].bound, rep.bands[n].slack, (int)rep.bands[n].within);
  return 0;
}
