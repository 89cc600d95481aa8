// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// extern "C" wrapper over the UNMODIFIED reference library `lrgw`
// (header-only C++20, /root/reference/proj/include/lrgw). Compiled by
// oracle/Makefile straight from the reference headers where they lie into
// oracle/_ref/libref_lrgw.so; no reference source is copied into this repo.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs load the result.
//
// Every entry point returns an lrgw status code (same numbering as
// include/lrgw_cuda.h) mapped 1:1 from the reference exception taxonomy
// (errors.hpp:10-36, contour.hpp:92-96).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "lrgw/contour.hpp"
#include "lrgw/driver.hpp"
#include "lrgw/elliptic.hpp"
#include "lrgw/gw.hpp"
#include "lrgw/isdf.hpp"
#include "lrgw/linalg.hpp"
#include "lrgw/model.hpp"
#include "lrgw/rng.hpp"
#include "lrgw/smw.hpp"

using namespace lrgw;

namespace {

enum {
  kOk = 0,
  kInvalid = 1,
  kGuard = 2,
  kNumeric = 3,
  kSingular = 4,
  kContour = 5,
  kIo = 6,
  kOther = 9,
};

thread_local int g_pivot = -1;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return kOk;
  } catch (const contour_convergence_error&) {
    return kContour;
  } catch (const singular_matrix& e) {
    g_pivot = e.pivot_index;
    return kSingular;
  } catch (const numeric_error&) {
    return kNumeric;
  } catch (const guard_exceeded&) {
    return kGuard;
  } catch (const io_error&) {
    return kIo;
  } catch (const invalid_input&) {
    return kInvalid;
  } catch (...) {
    return kOther;
  }
}

Matrix from_ptr(const double* p, int rows, int cols) {
  Matrix m(rows, cols);
  if (rows * static_cast<std::size_t>(cols) > 0)
    std::memcpy(m.data(), p, sizeof(double) * m.size());
  return m;
}

void to_ptr(const Matrix& m, double* p) {
  if (m.size() > 0) std::memcpy(p, m.data(), sizeof(double) * m.size());
}

Grid make_grid(const int* dims, const double* cell) {
  return Grid({dims[0], dims[1], dims[2]}, {cell[0], cell[1], cell[2]});
}

ContourSpec spec_from(const double* s) {
  ContourSpec c;
  c.q = s[0];
  c.big_q = s[1];
  c.r = s[2];
  c.big_r = s[3];
  c.l = s[4];
  c.e_shift = s[5];
  c.bypass = s[6] != 0.0;
  return c;
}

}  // namespace

extern "C" {

int ref_last_pivot() { return g_pivot; }

// rng.hpp:13-48 + matrix.hpp:29-33 — seeded column-major N(0,1) fill.
int ref_gaussian(std::uint64_t seed, int rows, int cols, double* out) {
  return guarded([&] {
    Rng rng(seed);
    to_ptr(Matrix::gaussian(rows, cols, rng), out);
  });
}

// rng.hpp:27-30 — n uniforms in (lo, hi].
int ref_uniform(std::uint64_t seed, int n, double lo, double hi, double* out) {
  return guarded([&] {
    Rng rng(seed);
    for (int i = 0; i < n; ++i) out[i] = rng.uniform(lo, hi);
  });
}

// model.hpp:56-116 — the reference's synthetic system (KAT fixtures).
int ref_build_synthetic(std::uint64_t seed, const int* dims, const double* cell,
                        int n_v, int n_c, double gap, double bandwidth,
                        double* psi, double* energies) {
  return guarded([&] {
    ElectronicStructure es = build_synthetic_system(
        seed, make_grid(dims, cell), n_v, n_c, gap, bandwidth);
    to_ptr(es.psi, psi);
    for (int i = 0; i < n_v + n_c; ++i) energies[i] = es.energies[i];
  });
}

// isdf.hpp:42-46
int ref_num_aux(double k, int n1, int n2, int* out) {
  return guarded([&] { *out = num_aux(k, n1, n2); });
}

// linalg.hpp:26-111 — pivot order of Householder QRCP (and |R_kk|).
int ref_qrcp(const double* a, int m, int n, int* perm, double* rdiag) {
  return guarded([&] {
    QrcpResult r = qrcp(from_ptr(a, m, n));
    for (int j = 0; j < n; ++j) perm[j] = r.perm[j];
    const int k = m < n ? m : n;
    if (rdiag)
      for (int j = 0; j < k; ++j) rdiag[j] = r.r(j, j);
  });
}

// isdf.hpp:95-112
int ref_select_points(const double* a, const double* b, int n_r, int n1,
                      int n2, int n_mu, int sketched, int* pts) {
  return guarded([&] {
    std::vector<int> p = select_interpolation_points(
        from_ptr(a, n_r, n1), from_ptr(b, n_r, n2), n_mu,
        sketched ? PointSelector::qrcp_sketched : PointSelector::qrcp_direct);
    for (int i = 0; i < n_mu; ++i) pts[i] = p[i];
  });
}

// isdf.hpp:118-163 — Theta (N_r x N_mu, column-major).
int ref_fit(const double* a, const double* b, int n_r, int n1, int n2,
            const int* pts, int n_mu, double* theta) {
  return guarded([&] {
    std::vector<int> p(pts, pts + n_mu);
    IsdfDecomposition d =
        fit_auxiliary_basis(from_ptr(a, n_r, n1), from_ptr(b, n_r, n2), p);
    to_ptr(d.p, theta);
  });
}

// isdf.hpp:195-202
int ref_isdf_error(const double* a, const double* b, int n_r, int n1, int n2,
                   const int* pts, int n_mu, const double* theta, double* err) {
  return guarded([&] {
    IsdfDecomposition d;
    d.n_mu = n_mu;
    d.point_indices.assign(pts, pts + n_mu);
    d.p = from_ptr(theta, n_r, n_mu);
    *err = isdf_reconstruction_error(from_ptr(a, n_r, n1), from_ptr(b, n_r, n2), d);
  });
}

// elliptic.hpp:28-33
int ref_elliptic_k(double k, double* out) {
  return guarded([&] { *out = elliptic_k(k); });
}

// elliptic.hpp:48-85
int ref_jacobi(double u, double k, double* out3) {
  return guarded([&] {
    JacobiTriple t = jacobi_sn_cn_dn(u, k);
    out3[0] = t.sn;
    out3[1] = t.cn;
    out3[2] = t.dn;
  });
}

// elliptic.hpp:97-118 — out6 = sn, cn, dn as (re, im) pairs.
int ref_jacobi_complex(double x, double y, double k, double* out6) {
  return guarded([&] {
    JacobiComplexTriple t = jacobi_complex({x, y}, k);
    out6[0] = t.sn.real();
    out6[1] = t.sn.imag();
    out6[2] = t.cn.real();
    out6[3] = t.cn.imag();
    out6[4] = t.dn.real();
    out6[5] = t.dn.imag();
  });
}

// contour.hpp:35-71 — out7 = q, Q, r, R, L, e_shift, bypass.
int ref_elliptic_params(const double* e, int n_e, int n_v, int n_c,
                        double delta_rel, int max_nodes, double* out7) {
  return guarded([&] {
    ContourSpec s = elliptic_params(std::vector<double>(e, e + n_e), n_v, n_c,
                                    delta_rel, max_nodes);
    out7[0] = s.q;
    out7[1] = s.big_q;
    out7[2] = s.r;
    out7[3] = s.big_r;
    out7[4] = s.l;
    out7[5] = s.e_shift;
    out7[6] = s.bypass ? 1.0 : 0.0;
  });
}

// contour.hpp:75-80
int ref_cauchy_error_bound(double q, double big_q, int n_lambda, double* out) {
  return guarded([&] {
    ContourSpec s;
    s.q = q;
    s.big_q = big_q;
    *out = cauchy_error_bound(s, n_lambda);
  });
}

// contour.hpp:114-137
int ref_coupled_direct(const double* pv, const double* pc, int n_mu, int n_v,
                       int n_c, const double* e, int n_e, double* t) {
  return guarded([&] {
    CoupledCoefficients c = coupled_coefficients_direct(
        from_ptr(pv, n_mu, n_v), from_ptr(pc, n_mu, n_c),
        std::vector<double>(e, e + n_e));
    to_ptr(c.t, t);
  });
}

// contour.hpp:144-183 — one unweighted node term.
int ref_node_term(const double* pv, const double* pc, int n_mu, int n_v,
                  int n_c, const double* e, int n_e, const double* spec7,
                  double t_node, double* out) {
  return guarded([&] {
    Matrix m = detail::contour_node_term(
        from_ptr(pv, n_mu, n_v), from_ptr(pc, n_mu, n_c),
        std::vector<double>(e, e + n_e), spec_from(spec7), t_node);
    to_ptr(m, out);
  });
}

// contour.hpp:185-222 — weighted node sum at explicit nodes (no prefactor).
int ref_sum_node_terms(const double* pv, const double* pc, int n_mu, int n_v,
                       int n_c, const double* e, int n_e, const double* spec7,
                       const double* nodes, const double* weights, int n_nodes,
                       int threads, double* acc) {
  return guarded([&] {
    Matrix m = detail::sum_node_terms(
        from_ptr(pv, n_mu, n_v), from_ptr(pc, n_mu, n_c),
        std::vector<double>(e, e + n_e), spec_from(spec7),
        std::vector<double>(nodes, nodes + n_nodes),
        std::vector<double>(weights, weights + n_nodes), threads);
    to_ptr(m, acc);
  });
}

// contour.hpp:298-329 — adaptive quadrature; on kContour `t` holds the best
// estimate carried by the exception.
int ref_coupled_contour(const double* pv, const double* pc, int n_mu, int n_v,
                        int n_c, const double* e, int n_e, double delta_rel,
                        int max_nodes, int threads, double* t, int* nodes_used,
                        double* est_rel) {
  std::vector<double> ev(e, e + n_e);
  Matrix mv = from_ptr(pv, n_mu, n_v), mc = from_ptr(pc, n_mu, n_c);
  try {
    ContourSpec s = elliptic_params(ev, n_v, n_c, delta_rel, max_nodes);
    CoupledCoefficients c = coupled_coefficients_contour(mv, mc, ev, s, threads);
    to_ptr(c.t, t);
    *nodes_used = c.nodes_used;
    *est_rel = c.est_rel_error;
    return kOk;
  } catch (const contour_convergence_error& ex) {
    to_ptr(ex.best.t, t);
    *nodes_used = ex.best.nodes_used;
    *est_rel = ex.best.est_rel_error;
    return kContour;
  } catch (...) {
    return guarded([] { throw; });
  }
}

// contour.hpp:282-294 — every level estimate up to the cap; out holds
// n_levels * n_mu^2 doubles, level node counts in `counts`.
int ref_contour_levels(const double* pv, const double* pc, int n_mu, int n_v,
                       int n_c, const double* e, int n_e, int max_level_nodes,
                       int max_levels, double* out, int* counts, int* n_levels) {
  return guarded([&] {
    std::vector<double> ev(e, e + n_e);
    ContourSpec s = elliptic_params(ev, n_v, n_c, 1e-7);
    auto lv = contour_refinement_levels(from_ptr(pv, n_mu, n_v),
                                        from_ptr(pc, n_mu, n_c), ev, s,
                                        max_level_nodes, 1);
    int n = static_cast<int>(lv.size());
    if (n > max_levels) n = max_levels;
    for (int i = 0; i < n; ++i) {
      counts[i] = lv[i].first;
      to_ptr(lv[i].second, out + static_cast<std::size_t>(i) * n_mu * n_mu);
    }
    *n_levels = n;
  });
}

// model.hpp:165-195 — reciprocal kernel 4 pi / |G|^2, v(0) = 0.
int ref_coulomb_kernel(const int* dims, const double* cell, double* kern) {
  return guarded([&] {
    CoulombOperator v =
        build_coulomb(make_grid(dims, cell), CoulombMode::reciprocal_diagonal);
    for (std::size_t i = 0; i < v.kernel.size(); ++i) kern[i] = v.kernel[i];
  });
}

// model.hpp:208-223; zero_kernel != 0 selects zero_coulomb (model.hpp:198-204).
int ref_apply_coulomb(const int* dims, const double* cell, int zero_kernel,
                      const double* x, int m, int threads, double* y) {
  return guarded([&] {
    Grid g = make_grid(dims, cell);
    CoulombOperator v = zero_kernel
                            ? zero_coulomb(g)
                            : build_coulomb(g, CoulombMode::reciprocal_diagonal);
    to_ptr(apply_coulomb(v, from_ptr(x, g.n_r(), m), threads), y);
  });
}

// smw.hpp:42-73
int ref_assemble_K(const double* t, const double* p, int n_r, int n_mu,
                   const int* dims, const double* cell, int zero_kernel,
                   int threads, double* k) {
  return guarded([&] {
    Grid g = make_grid(dims, cell);
    if (g.n_r() != n_r) throw invalid_input("shim: grid / N_r mismatch");
    CoulombOperator v = zero_kernel
                            ? zero_coulomb(g)
                            : build_coulomb(g, CoulombMode::reciprocal_diagonal);
    to_ptr(assemble_K(from_ptr(t, n_mu, n_mu), from_ptr(p, n_r, n_mu), v, threads), k);
  });
}

// smw.hpp:84-103 — build the factored inverse, apply it to X (N_r x m).
// k_out (N_mu^2) and vp_out (N_r x N_mu) are optional.
int ref_build_and_apply(const double* t, const double* p, int n_r, int n_mu,
                        const int* dims, const double* cell, int threads,
                        const double* x, int m, double* y, double* k_out,
                        double* vp_out) {
  return guarded([&] {
    Grid g = make_grid(dims, cell);
    if (g.n_r() != n_r) throw invalid_input("shim: grid / N_r mismatch");
    CoulombOperator v = build_coulomb(g, CoulombMode::reciprocal_diagonal);
    EpsilonInverseLowRank e = build_epsilon_inverse(
        from_ptr(t, n_mu, n_mu), from_ptr(p, n_r, n_mu), v, threads);
    if (x && y) to_ptr(epsilon_inverse_apply(e, from_ptr(x, n_r, m)), y);
    if (k_out) to_ptr(e.k, k_out);
    if (vp_out) to_ptr(e.vp, vp_out);
  });
}

// gw.hpp:73-88 — projected screened interactions from the factored inverse
// built on (T, P_vc) (smw.hpp:84-95) and the vn / nn interpolation vectors.
int ref_project_screened(const double* t, const double* p, int n_r, int n_mu, const int* dims,
                         const double* cell, int zero_kernel, const double* p_vn, int n_vn,
                         const double* p_nn, int n_nn, double* w_vn, double* w_nn, double* v_vn) {
  return guarded([&] {
    Grid g = make_grid(dims, cell);
    if (g.n_r() != n_r) throw invalid_input("shim: grid / N_r mismatch");
    CoulombOperator v = zero_kernel ? zero_coulomb(g) : build_coulomb(g, CoulombMode::reciprocal_diagonal);
    EpsilonInverseLowRank e = build_epsilon_inverse(from_ptr(t, n_mu, n_mu), from_ptr(p, n_r, n_mu), v);
    IsdfDecomposition vn, nn;
    vn.p = from_ptr(p_vn, n_r, n_vn);
    nn.p = from_ptr(p_nn, n_r, n_nn);
    ScreenedProjections out = project_screened_interactions(e, vn, nn);
    to_ptr(out.w_vn, w_vn);
    to_ptr(out.w_nn, w_nn);
    to_ptr(out.v_vn, v_vn);
  });
}

ElectronicStructure make_es(const double* psi, int n_r, int n_v, int n_c, const int* dims, const double* cell,
                            const double* energies) {
  ElectronicStructure es;
  es.grid = make_grid(dims, cell);
  if (es.grid.n_r() != n_r) throw invalid_input("shim: grid / N_r mismatch");
  es.psi = from_ptr(psi, n_r, n_v + n_c);
  es.n_v = n_v;
  es.n_c = n_c;
  es.energies.assign(energies, energies + n_v + n_c);
  es.vxc.assign(n_v + n_c, 0.0);
  return es;
}

IsdfDecomposition dec_at(const ElectronicStructure& es, PairSetLabel label, const int* pts, int n) {
  Matrix a = label == PairSetLabel::nn ? es.psi : es.occupied();
  Matrix b = label == PairSetLabel::vc ? es.unoccupied() : es.psi;
  return fit_auxiliary_basis(a, b, std::vector<int>(pts, pts + n), label);
}

void put_sigma(const SelfEnergies& s, int nb, double* out4) {
  for (int n = 0; n < nb; ++n) {
    out4[n] = s.sigma_sex_x[n];
    out4[nb + n] = s.sigma_x[n];
    out4[2 * nb + n] = s.sigma_coh[n];
    out4[3 * nb + n] = s.sigma_total[n];
  }
}

// gw.hpp:143-153 — self_energies_lowrank on caller-supplied projections
// (the leaf the GPU's lrgw_self_energies_lowrank replaces).
int ref_sigma_lowrank(const double* psi, int n_r, int n_v, int n_c, const int* pts_vn, int n_vn,
                      const int* pts_nn, int n_nn, const double* w_vn, const double* w_nn,
                      const double* v_vn, double* out4) {
  return guarded([&] {
    ElectronicStructure es;
    es.psi = from_ptr(psi, n_r, n_v + n_c);
    es.n_v = n_v;
    es.n_c = n_c;
    IsdfDecomposition vn, nn;
    vn.point_indices.assign(pts_vn, pts_vn + n_vn);
    nn.point_indices.assign(pts_nn, pts_nn + n_nn);
    SelfEnergies s = self_energies_lowrank(es, from_ptr(w_vn, n_vn, n_vn), from_ptr(w_nn, n_nn, n_nn),
                                           from_ptr(v_vn, n_vn, n_vn), vn, nn);
    put_sigma(s, n_v + n_c, out4);
  });
}

// The three self-energy pipelines of gw.hpp on fixed point sets, composed as
// test_gw.cpp:13-41 does: which = 0 low-rank (T direct, build_epsilon_inverse,
// project_screened_interactions, self_energies_lowrank), 1 conventional ISDF
// (dense eps, gw.hpp:158-181), 2 brute force (gw.hpp:189-222).
int ref_self_energies(const double* psi, int n_r, int n_v, int n_c, const int* dims, const double* cell,
                      const double* energies, const int* pts_vc, int n_vc, const int* pts_vn, int n_vn,
                      const int* pts_nn, int n_nn, int which, double* out4) {
  return guarded([&] {
    ElectronicStructure es = make_es(psi, n_r, n_v, n_c, dims, cell, energies);
    CoulombOperator v = build_coulomb(es.grid, CoulombMode::reciprocal_diagonal);
    SelfEnergies s;
    if (which == 2) {
      s = self_energies_bruteforce(es, v);
    } else {
      IsdfDecomposition vc = dec_at(es, PairSetLabel::vc, pts_vc, n_vc);
      IsdfDecomposition vn = dec_at(es, PairSetLabel::vn, pts_vn, n_vn);
      IsdfDecomposition nn = dec_at(es, PairSetLabel::nn, pts_nn, n_nn);
      if (which == 1) {
        s = self_energies_isdf_conventional(es, v, vc, vn, nn);
      } else {
        Matrix t = coupled_coefficients_direct(rows_at(es.occupied(), vc.point_indices),
                                               rows_at(es.unoccupied(), vc.point_indices), es.energies)
                       .t;
        EpsilonInverseLowRank e = build_epsilon_inverse(t, vc.p, v);
        ScreenedProjections proj = project_screened_interactions(e, vn, nn);
        s = self_energies_lowrank(es, proj.w_vn, proj.w_nn, proj.v_vn, vn, nn);
      }
    }
    put_sigma(s, n_v + n_c, out4);
  });
}

// gw.hpp:48-58
int ref_quasiparticle(const double* energies, const double* vxc, const double* sigma_total, int n,
                      int n_sigma, double* out) {
  return guarded([&] {
    ElectronicStructure es;
    es.energies.assign(energies, energies + n);
    es.vxc.assign(vxc, vxc + n);
    SelfEnergies s;
    s.sigma_sex_x.assign(sigma_total, sigma_total + n_sigma);
    s.sigma_x.assign(n_sigma, 0.0);
    s.sigma_coh.assign(n_sigma, 0.0);
    s.finalize(PipelineTag::lowrank);
    QuasiparticleEnergies q = quasiparticle_energies(es, s);
    for (int i = 0; i < n; ++i) out[i] = q.eps_gw[i];
  });
}

// model.hpp:236-339 — WFN1 writer / reader. The reader reports the
// io_error text through ref_last_message().
thread_local std::string g_msg;

int ref_save_system(const char* path, const int* dims, const double* cell, int n_v, int n_c,
                    const double* psi, const double* energies, const double* vxc) {
  return guarded([&] {
    ElectronicStructure es;
    es.grid = make_grid(dims, cell);
    es.n_v = n_v;
    es.n_c = n_c;
    es.psi = from_ptr(psi, es.grid.n_r(), n_v + n_c);
    es.energies.assign(energies, energies + n_v + n_c);
    es.vxc.assign(vxc, vxc + n_v + n_c);
    save_system(path, es);
  });
}

int ref_load_system(const char* path, int* dims, double* cell, int* n_v, int* n_c, double* psi,
                    double* energies, double* vxc) {
  g_msg.clear();
  try {
    ElectronicStructure es = load_system(path);
    for (int k = 0; k < 3; ++k) {
      dims[k] = es.grid.dims[k];
      cell[k] = es.grid.cell[k];
    }
    *n_v = es.n_v;
    *n_c = es.n_c;
    if (psi) to_ptr(es.psi, psi);
    if (energies) std::memcpy(energies, es.energies.data(), sizeof(double) * es.energies.size());
    if (vxc) std::memcpy(vxc, es.vxc.data(), sizeof(double) * es.vxc.size());
    return kOk;
  } catch (const std::exception& e) {
    g_msg = e.what();
    return guarded([&] { throw; });
  }
}

const char* ref_last_message() { return g_msg.c_str(); }

// driver.hpp:253-329 — run_pipeline on a JSON config, result as
// run_result_to_json(...).dump() (truncated to cap bytes; returns the length).
int ref_run_pipeline_json(const char* config_json, char* out, int cap, int* out_len) {
  return guarded([&] {
    RunConfig c = parse_config(json::parse(config_json));
    std::string d = run_result_to_json(run_pipeline(c), c).dump();
    *out_len = static_cast<int>(d.size());
    std::memcpy(out, d.data(), std::min<std::size_t>(d.size(), static_cast<std::size_t>(cap)));
  });
}

// smw.hpp:97-103 with caller-supplied K (e.g. K = 0 identity check).
int ref_eps_apply_given(const double* p, const double* k, int n_r, int n_mu,
                        const int* dims, const double* cell, const double* x,
                        int m, double* y) {
  return guarded([&] {
    Grid g = make_grid(dims, cell);
    EpsilonInverseLowRank e;
    e.p_vc = from_ptr(p, n_r, n_mu);
    e.k = from_ptr(k, n_mu, n_mu);
    e.v = build_coulomb(g, CoulombMode::reciprocal_diagonal);
    e.vp = apply_coulomb(e.v, e.p_vc);
    to_ptr(epsilon_inverse_apply(e, from_ptr(x, n_r, m)), y);
  });
}

// smw.hpp:371-391 — dense LU inverse of the ISDF epsilon (N_r <= 1024) and
// eps itself, for the SMW == LU acceptance criterion.
int ref_epsilon_dense(const double* psi, int n_r, int n_v, int n_c,
                      const double* energies, const int* dims,
                      const double* cell, const int* pts, int n_mu,
                      const double* theta, double* eps, double* eps_inv) {
  return guarded([&] {
    ElectronicStructure es;
    es.grid = make_grid(dims, cell);
    es.psi = from_ptr(psi, n_r, n_v + n_c);
    es.energies.assign(energies, energies + n_v + n_c);
    es.vxc.assign(n_v + n_c, 0.0);
    es.n_v = n_v;
    es.n_c = n_c;
    CoulombOperator v = build_coulomb(es.grid, CoulombMode::reciprocal_diagonal);
    IsdfDecomposition d;
    d.n_mu = n_mu;
    d.point_indices.assign(pts, pts + n_mu);
    d.p = from_ptr(theta, n_r, n_mu);
    EpsilonDense o = epsilon_dense_oracle(es, v, &d);
    if (eps) to_ptr(o.eps, eps);
    if (eps_inv) to_ptr(o.eps_inv, eps_inv);
  });
}

// matrix.hpp:88-102 — C = A^T B (the reference's pvp contraction, smw.hpp:61).
int ref_matmul_tn(const double* a, int m, int ka, const double* b, int kb, double* c) {
  return guarded([&] { to_ptr(matmul_tn(from_ptr(a, m, ka), from_ptr(b, m, kb)), c); });
}

// linalg.hpp:152-183 — X = A^-1 B by LU (lu_solve), B n x nrhs.
int ref_lu_solve(const double* a, int n, const double* b, int nrhs, double* x) {
  return guarded([&] { to_ptr(lu_solve(from_ptr(a, n, n), from_ptr(b, n, nrhs)), x); });
}

// linalg.hpp:310-345 — ascending eigenvalues.
int ref_sym_eig_values(const double* a, int n, double* values) {
  return guarded([&] {
    SymEigResult r = sym_eig(from_ptr(a, n, n));
    for (int i = 0; i < n; ++i) values[i] = r.values[i];
  });
}

// ---------------------------------------------------------------------------
// Stage-wise checkers at the large BASELINE configs. Each composes the
// reference's own primitives in the reference's own order, restricted to the
// rows / columns under test; every restricted quantity is separable, so the
// outputs are bit-identical to the corresponding rows / columns of the full
// reference call (matmul_nt / hadamard / lu_solve_factored / matmul_tn act
// row- or column-wise). parallel_for (parallel.hpp:11-29) spreads the
// independent columns over host threads.
// ---------------------------------------------------------------------------

// fit_auxiliary_basis (isdf.hpp:118-163) for selected rows: a_rows / b_rows
// (nrows x n1 / n2) are psi_a / psi_b at the rows under test, a_mu / b_mu
// (n_mu x n1 / n2) at the sorted points. theta_rows (nrows x n_mu) = those
// rows of the reference P (LU path, or the pseudo-inverse fallback on a
// singular Gram exactly as isdf.hpp:144-161).
int ref_fit_rows(const double* a_rows, const double* b_rows, int nrows, const double* a_mu,
                 const double* b_mu, int n_mu, int n1, int n2, int threads, double* theta_rows,
                 int* used_pinv) {
  return guarded([&] {
    Matrix am = from_ptr(a_mu, n_mu, n1), bm = from_ptr(b_mu, n_mu, n2);
    Matrix gram = hadamard(matmul_nt(am, am), matmul_nt(bm, bm));  // = rows_at(lhs, points)
    symmetrize(gram);
    Matrix ar = from_ptr(a_rows, nrows, n1), br = from_ptr(b_rows, nrows, n2);
    if (used_pinv) *used_pinv = 0;
    LuFactors f;
    bool singular = false;
    try {
      f = lu_factor(gram);
    } catch (const singular_matrix&) {
      singular = true;
    }
    Matrix pinv;
    if (singular) {  // isdf.hpp:144-161
      if (used_pinv) *used_pinv = 1;
      SymEigResult ev = sym_eig(gram);
      double lam_max = 0.0;
      for (double v : ev.values) lam_max = std::max(lam_max, std::abs(v));
      if (lam_max <= 0.0) throw numeric_error("fit_auxiliary_basis: degenerate Gram matrix");
      std::vector<double> inv(ev.values.size(), 0.0);
      int kept = 0;
      for (std::size_t i = 0; i < ev.values.size(); ++i)
        if (std::abs(ev.values[i]) > 1e-12 * lam_max) {
          inv[i] = 1.0 / ev.values[i];
          ++kept;
        }
      if (kept == 0) throw numeric_error("fit_auxiliary_basis: degenerate Gram matrix");
      pinv = matmul_nt(scale_cols(ev.q, inv), ev.q);
    }
    // row blocks: lhs = (A A_mu^T) o (B B_mu^T) and its solve, per block
    Matrix out(nrows, n_mu);
    const int nb = std::max(1, std::min(threads, nrows));
    parallel_for(nb, nb, [&](int t) {
      const int lo = static_cast<int>(static_cast<long long>(nrows) * t / nb);
      const int hi = static_cast<int>(static_cast<long long>(nrows) * (t + 1) / nb);
      if (hi <= lo) return;
      std::vector<int> idx(hi - lo);
      for (int i = lo; i < hi; ++i) idx[i - lo] = i;
      Matrix lhs = hadamard(matmul_nt(rows_at(ar, idx), am), matmul_nt(rows_at(br, idx), bm));
      Matrix pb = singular ? matmul(lhs, pinv) : transpose(lu_solve_factored(f, transpose(lhs)));
      for (int j = 0; j < n_mu; ++j)
        for (int i = lo; i < hi; ++i) out(i, j) = pb(i - lo, j);
    });
    to_ptr(out, theta_rows);
  });
}

// Columns `cols` of pvp = P^T (V P) before symmetrisation (smw.hpp:61):
// apply_coulomb on the selected columns (model.hpp:208-223, threaded), then
// matmul_tn (matrix.hpp:88-102) per column block. vp_cols (optional,
// n_r x ncols) returns V P(:, cols).
int ref_pvp_cols(const double* p, int n_r, int n_mu, const int* dims, const double* cell,
                 const int* cols, int ncols, int threads, double* out, double* vp_cols) {
  return guarded([&] {
    Grid g = make_grid(dims, cell);
    if (g.n_r() != n_r) throw invalid_input("shim: grid / N_r mismatch");
    CoulombOperator v = build_coulomb(g, CoulombMode::reciprocal_diagonal);
    Matrix pm = from_ptr(p, n_r, n_mu);
    Matrix sel(n_r, ncols);
    for (int j = 0; j < ncols; ++j) {
      if (cols[j] < 0 || cols[j] >= n_mu) throw invalid_input("shim: column out of range");
      std::copy(pm.col(cols[j]), pm.col(cols[j]) + n_r, sel.col(j));
    }
    Matrix vp = apply_coulomb(v, sel, threads);
    Matrix c(n_mu, ncols);
    const int nb = std::max(1, std::min(threads, ncols));
    parallel_for(nb, nb, [&](int t) {
      const int lo = static_cast<int>(static_cast<long long>(ncols) * t / nb);
      const int hi = static_cast<int>(static_cast<long long>(ncols) * (t + 1) / nb);
      if (hi <= lo) return;
      Matrix cb = matmul_tn(pm, cols_block(vp, lo, hi - lo));
      for (int j = 0; j < hi - lo; ++j) std::copy(cb.col(j), cb.col(j) + n_mu, c.col(lo + j));
    });
    to_ptr(c, out);
    if (vp_cols) to_ptr(vp, vp_cols);
  });
}

// assemble_K (smw.hpp:42-73) with pvp = P^T V P supplied (unsymmetrised):
// the sym_eig definiteness check, lu_solve(T, I/2), the three symmetrisations
// and lu_invert, in the reference's order.
int ref_smw_from_pvp(const double* t, const double* pvp, int n_mu, int check_eig, int threads, double* k) {
  return guarded([&] {
    // lu_solve(A, B) = lu_solve_factored(lu_factor(A), B), column by column:
    // the right-hand sides are spread over threads (bit-identical result)
    auto solve = [&](const Matrix& a, const Matrix& b) {
      LuFactors f = lu_factor(a);
      Matrix x(b.rows(), b.cols());
      const int nb = std::max(1, std::min(threads, b.cols()));
      parallel_for(nb, nb, [&](int q) {
        const int lo = static_cast<int>(static_cast<long long>(b.cols()) * q / nb);
        const int hi = static_cast<int>(static_cast<long long>(b.cols()) * (q + 1) / nb);
        if (hi <= lo) return;
        Matrix xb = lu_solve_factored(f, cols_block(b, lo, hi - lo));
        for (int j = 0; j < hi - lo; ++j) std::copy(xb.col(j), xb.col(j) + b.rows(), x.col(lo + j));
      });
      return x;
    };
    Matrix tm = from_ptr(t, n_mu, n_mu);
    if (check_eig) {
      SymEigResult ev = sym_eig(tm);
      if (!(ev.values.back() < 0.0))
        throw numeric_error("assemble_K: T is not negative definite (gapless or rank-deficient input)");
    }
    Matrix half_t_inv;
    try {
      half_t_inv = solve(tm, 0.5 * Matrix::identity(n_mu));
    } catch (const singular_matrix& e) {
      throw singular_matrix("assemble_K: T singular", e.pivot_index);
    }
    symmetrize(half_t_inv);
    Matrix pv = from_ptr(pvp, n_mu, n_mu);
    symmetrize(pv);
    Matrix km;
    try {
      km = solve(half_t_inv - pv, Matrix::identity(n_mu));  // lu_invert (linalg.hpp:181-183)
    } catch (const singular_matrix& e) {
      throw singular_matrix("assemble_K: middle matrix singular", e.pivot_index);
    }
    symmetrize(km);
    to_ptr(km, k);
  });
}

// epsilon_inverse_apply (smw.hpp:97-103) given P, K and VP = V P:
// Y = X + VP (K (P^T X)).
int ref_eps_apply_vp(const double* p, const double* k, const double* vp, int n_r, int n_mu,
                     const double* x, int m, double* y) {
  return guarded([&] {
    EpsilonInverseLowRank e;
    e.p_vc = from_ptr(p, n_r, n_mu);
    e.k = from_ptr(k, n_mu, n_mu);
    e.vp = from_ptr(vp, n_r, n_mu);
    to_ptr(epsilon_inverse_apply(e, from_ptr(x, n_r, m)), y);
  });
}

// The same operator with V applied last: Y = X + V (P (K (P^T X))) — equal to
// smw.hpp:101-102 up to rounding (V is linear), for sizes where V P (all N_mu
// columns through the dense DFT) is out of reach on the host.
int ref_eps_apply_factored(const double* p, const double* k, int n_r, int n_mu, const int* dims,
                           const double* cell, const double* x, int m, int threads, double* y) {
  return guarded([&] {
    Grid g = make_grid(dims, cell);
    if (g.n_r() != n_r) throw invalid_input("shim: grid / N_r mismatch");
    CoulombOperator v = build_coulomb(g, CoulombMode::reciprocal_diagonal);
    Matrix pm = from_ptr(p, n_r, n_mu);
    Matrix xm = from_ptr(x, n_r, m);
    Matrix z = matmul(pm, matmul(from_ptr(k, n_mu, n_mu), matmul_tn(pm, xm)));
    to_ptr(xm + apply_coulomb(v, z, threads), y);
  });
}

}  // extern "C"
