// test_dropin.cpp — the reference's own known-answer tests, restated as plain
// assertions against the DROP-IN headers (include/lrgw/*.hpp) over
// liblrgw_cuda.so: a caller of the reference API recompiles unchanged.
// Sources of the KATs: proj/tests/test_isdf.cpp, test_contour.cpp,
// test_smw.cpp, test_model.cpp, test_elliptic.cpp.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <string>

#include "lrgw/lrgw.hpp"

using namespace lrgw;

static int failures = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

// Orthonormal orbitals from a seeded Gaussian (modified Gram-Schmidt, host).
static Matrix orbitals(int n_r, int nb, std::uint64_t seed) {
  Rng rng(seed);
  Matrix q = Matrix::gaussian(n_r, nb, rng);
  for (int j = 0; j < nb; ++j) {
    for (int i = 0; i < j; ++i) {
      double d = 0.0;
      for (int r = 0; r < n_r; ++r) d += q(r, i) * q(r, j);
      for (int r = 0; r < n_r; ++r) q(r, j) -= d * q(r, i);
    }
    double nn = 0.0;
    for (int r = 0; r < n_r; ++r) nn += q(r, j) * q(r, j);
    nn = std::sqrt(nn);
    for (int r = 0; r < n_r; ++r) q(r, j) /= nn;
  }
  return q;
}

int main() {
  // num_aux (test_isdf.cpp:21-34)
  CHECK(num_aux(8.0, 16, 16) == 128);
  CHECK(num_aux(8.0, 128, 128) == 1024);
  CHECK(throws<invalid_input>([] { num_aux(0.0, 4, 4); }));

  // elliptic_params closed form (test_contour.cpp:35-52)
  ContourSpec s = elliptic_params({0.0, 1.0, 4.0}, 1, 2, 1e-7);
  CHECK(std::abs(s.r - 1.0 / 3.0) <= 1e-15);
  CHECK(std::abs(s.big_r - elliptic_k(1.0 / 3.0)) <= 1e-14 * s.big_r);
  CHECK(!s.bypass && s.l > 0.0);
  CHECK(elliptic_params({0.0, 2.0}, 1, 1, 1e-7).bypass);
  CHECK(throws<invalid_input>([] { elliptic_params({0.0, 0.0, 1.0}, 1, 2, 1e-7); }));

  // the two-denominator toy pins the contour constant: T = -0.75 (test_contour.cpp:84-95)
  {
    Matrix v(1, 1), c(1, 2);
    v(0, 0) = 1.0;
    c(0, 0) = c(0, 1) = 1.0;
    std::vector<double> e = {0.0, 2.0, 4.0};
    CoupledCoefficients t = coupled_coefficients_contour(v, c, e, elliptic_params(e, 1, 2, 1e-10));
    CHECK(std::abs(t.t(0, 0) + 0.75) <= 0.75e-9);
    CHECK(t.nodes_used >= 17 && t.est_rel_error <= 1e-10);
    Matrix one(1, 1);
    one(0, 0) = 1.0;
    CHECK(std::abs(coupled_coefficients_direct(one, one, {0.0, 2.0}).t(0, 0) + 0.5) <= 1e-15);
  }

  // select / fit / contour / SMW on a seeded desk system
  const Grid grid({8, 8, 8}, {6.0, 6.0, 6.0});
  const int n_r = grid.n_r();
  Matrix psi = orbitals(n_r, 32, 1);
  Matrix a = cols_block(psi, 0, 16), b = cols_block(psi, 16, 16);
  std::vector<int> all(n_r);
  std::iota(all.begin(), all.end(), 0);
  CHECK(throws<invalid_input>([&] { select_interpolation_points(a, b, n_r + 1); }));
  std::vector<int> pts = select_interpolation_points(a, b, 128);
  CHECK(pts.size() == 128);
  for (std::size_t i = 1; i < pts.size(); ++i) CHECK(pts[i] > pts[i - 1]);
  IsdfDecomposition dec = fit_auxiliary_basis(a, b, pts);
  // Theta reproduces the pair functions at the interpolation points: P(pts, :) = I
  Matrix pp = rows_at(dec.p, pts);
  double defect = 0.0;
  for (int j = 0; j < 128; ++j)
    for (int i = 0; i < 128; ++i) defect = std::max(defect, std::abs(pp(i, j) - (i == j ? 1.0 : 0.0)));
  CHECK(defect <= 1e-10);
  CHECK(throws<numeric_error>([] { fit_auxiliary_basis(Matrix(8, 2), Matrix(8, 2), {1, 3}); }));

  std::vector<double> e(32);
  for (int i = 0; i < 16; ++i) e[i] = -4.0 + 4.0 * i / 15.0;
  for (int j = 0; j < 16; ++j) e[16 + j] = 1.0 + 4.0 * j / 15.0;
  Matrix pv = rows_at(a, pts), pc = rows_at(b, pts);
  CoupledCoefficients t_dir = coupled_coefficients_direct(pv, pc, e);
  CoupledCoefficients t_quad = coupled_coefficients_contour(pv, pc, e, elliptic_params(e, 16, 16, 1e-7));
  CHECK(frobenius_norm(t_quad.t - t_dir.t) <= 1e-7 * frobenius_norm(t_dir.t));  // test_contour.cpp:97-109
  CHECK(symmetry_defect(t_quad.t) <= 1e-10 * frobenius_norm(t_quad.t));

  CoulombOperator v = build_coulomb(grid, CoulombMode::reciprocal_diagonal);
  CHECK(v.kernel[0] == 0.0);
  Matrix ones(n_r, 1);
  for (int i = 0; i < n_r; ++i) ones(i, 0) = 1.0;
  CHECK(max_abs(apply_coulomb(v, ones)) <= 1e-12);  // test_model.cpp:68-80
  // V = 0 => K = 2T (test_smw.cpp:58-64)
  Matrix k0 = assemble_K(t_dir.t, dec.p, zero_coulomb(grid));
  CHECK(frobenius_norm(k0 - 2.0 * t_dir.t) <= 1e-9 * frobenius_norm(k0));
  // K symmetric negative definite; K = 0 => identity apply (test_smw.cpp:66-97)
  EpsilonInverseLowRank eps = build_epsilon_inverse(t_dir.t, dec.p, v);
  CHECK(symmetry_defect(eps.k) <= 1e-10 * frobenius_norm(eps.k));
  Rng rng(11);
  Matrix x = Matrix::gaussian(n_r, 3, rng);
  EpsilonInverseLowRank id;
  id.p_vc = dec.p;
  id.k = Matrix(128, 128);
  id.v = v;
  CHECK(epsilon_inverse_apply(id, x) == x);
  // linearity (test_smw.cpp:99-111)
  Matrix x1 = Matrix::gaussian(n_r, 1, rng), x2 = Matrix::gaussian(n_r, 1, rng);
  Matrix lhs = epsilon_inverse_apply(eps, 1.7 * x1 - 0.4 * x2);
  Matrix rhs = 1.7 * epsilon_inverse_apply(eps, x1) - 0.4 * epsilon_inverse_apply(eps, x2);
  CHECK(frobenius_norm(lhs - rhs) <= 1e-12 * frobenius_norm(lhs));
  // rank-deficient T is rejected (test_smw.cpp:74-85)
  {
    const Grid g4({4, 4, 4}, {6.0, 6.0, 6.0});
    Matrix q = orbitals(64, 4, 2);
    Matrix qa = cols_block(q, 0, 2), qb = cols_block(q, 2, 2);
    std::vector<int> p8 = select_interpolation_points(qa, qb, 8);
    IsdfDecomposition d8 = fit_auxiliary_basis(qa, qb, p8);
    Matrix t8 = coupled_coefficients_direct(rows_at(qa, p8), rows_at(qb, p8), {-1.0, -0.5, 0.5, 1.0}).t;
    CHECK(throws<numeric_error>([&] { assemble_K(t8, d8.p, build_coulomb(g4, CoulombMode::reciprocal_diagonal)); }));
  }
  // GW consumers (test_gw.cpp:66-90, 174-233): vn / nn ISDF, projections, Sigma
  {
    ElectronicStructure es;
    es.grid = grid;
    es.psi = psi;
    es.n_v = 16;
    es.n_c = 16;
    es.energies = e;
    es.vxc.assign(32, 0.0);
    IsdfDecomposition vn = build_isdf(es, PairSetLabel::vn, 4.0);
    IsdfDecomposition nn = build_isdf(es, PairSetLabel::nn, 4.0);
    CHECK(vn.n_mu == num_aux(4.0, 16, 32) && nn.n_mu == num_aux(4.0, 32, 32));
    ScreenedProjections proj = project_screened_interactions(eps, vn, nn);
    CHECK(symmetry_defect(proj.w_vn) == 0.0 && symmetry_defect(proj.v_vn) == 0.0);
    SelfEnergies sig = self_energies_lowrank(es, proj.w_vn, proj.w_nn, proj.v_vn, vn, nn);
    CHECK(sig.pipeline_tag == PipelineTag::lowrank);
    for (int n = 0; n < 32; ++n) {
      CHECK(sig.sigma_x[n] <= 1e-12);
      CHECK(sig.sigma_total[n] == sig.sigma_sex_x[n] + sig.sigma_x[n] + sig.sigma_coh[n]);
    }
    EpsilonInverseLowRank e0 = build_epsilon_inverse(t_dir.t, dec.p, zero_coulomb(grid));
    ScreenedProjections p0 = project_screened_interactions(e0, vn, nn);
    CHECK(frobenius_norm(p0.w_vn) <= 1e-12 && frobenius_norm(p0.v_vn) <= 1e-12);
    SelfEnergies s0 = self_energies_lowrank(es, p0.w_vn, p0.w_nn, p0.v_vn, vn, nn);
    for (int n = 0; n < 32; ++n) CHECK(std::abs(s0.sigma_total[n]) <= 1e-14);
    es.vxc.assign(32, 0.05);
    QuasiparticleEnergies qp = quasiparticle_energies(es, sig);
    for (int n = 0; n < 32; ++n) CHECK(qp.eps_gw[n] == es.energies[n] + sig.sigma_total[n] - 0.05);
    es.vxc.assign(31, 0.0);
    CHECK(throws<invalid_input>([&] { quasiparticle_energies(es, sig); }));
  }
  // WFN1 round trip and error messages (test_model.cpp:125-193)
  {
    ElectronicStructure es;
    es.grid = grid;
    es.psi = psi;
    es.n_v = 16;
    es.n_c = 16;
    es.energies = e;
    es.vxc.assign(32, 0.01);
    const std::string path = "/tmp/lrgw_dropin_test.wfn1";
    save_system(path, es);
    ElectronicStructure back = load_system(path);
    CHECK(back.grid == es.grid && back.n_v == 16 && back.n_c == 16);
    CHECK(back.psi == es.psi && back.energies == es.energies && back.vxc == es.vxc);
    {
      std::FILE* f = std::fopen(path.c_str(), "r+b");
      std::fputc('X', f);
      std::fclose(f);
    }
    bool msg_ok = false;
    try {
      load_system(path);
    } catch (const io_error& ex) {
      msg_ok = std::string(ex.what()) == "load_system: bad magic";
    }
    CHECK(msg_ok);
    CHECK(throws<io_error>([] { load_system("lrgw_test_does_not_exist.wfn1"); }));
    std::remove(path.c_str());
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "ok", failures);
  return failures ? 1 : 0;
}
