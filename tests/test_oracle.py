"""CPU: pin the oracle restatement (oracle/restate.py, oracle/select.c) against
the compiled reference (oracle/_ref) and the reference's own known-answer
tests, and against the committed golden fixtures (tests/golden/)."""
import glob
import math
import os

import numpy as np
import pytest

from oracle import restate as R
from helpers import rel

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---- reference KATs restated (proj/tests/*.cpp) ---------------------------

def test_num_aux_kats():
    # test_isdf.cpp:21-34
    assert R.num_aux(8.0, 16, 16) == 128
    assert R.num_aux(8.0, 128, 128) == 1024
    assert R.num_aux(1.0, 1, 1) == 1
    with pytest.raises(R.InvalidInput):
        R.num_aux(0.0, 4, 4)
    prev = 0
    for k in np.arange(1.0, 12.01, 0.5):
        n = R.num_aux(k, 7, 9)
        assert n >= prev
        prev = n


def test_elliptic_kats():
    # test_elliptic.cpp:12-62
    for r in (0.0, 1 / 3, 0.5, 0.9, 0.99):
        by_quad = R.integrate_adaptive(lambda th: 1.0 / math.sqrt(1.0 - r * r * math.sin(th) ** 2), 0.0,
                                       1.57079632679489661923)
        assert abs(R.elliptic_k(r) - by_quad) <= 1e-10 * by_quad
    with pytest.raises(R.InvalidInput):
        R.elliptic_k(1.0)
    sn, cn, dn = R.jacobi_sn_cn_dn(R.elliptic_k(1 / 3), 1 / 3)
    assert abs(sn - 1.0) <= 1e-10 and abs(cn) <= 1e-8
    rng = np.random.default_rng(77)
    for _ in range(200):
        r, u = rng.uniform(0, 0.97), rng.uniform(-4, 4)
        sn, cn, dn = R.jacobi_sn_cn_dn(u, r)
        assert abs(sn * sn + cn * cn - 1) <= 1e-12
        assert abs(dn * dn + r * r * sn * sn - 1) <= 1e-12


def test_elliptic_params_kats():
    # test_contour.cpp:35-65
    s = R.elliptic_params([0.0, 1.0, 4.0], 1, 2, 1e-7)
    assert abs(s.r - 1 / 3) <= 1e-15 and s.l > 0 and not s.bypass
    assert abs(s.big_r - R.elliptic_k(1 / 3)) <= 1e-14 * s.big_r
    s = R.elliptic_params([0.0, 2.0], 1, 1, 1e-7)
    assert s.r == 0.0 and s.bypass
    with pytest.raises(R.InvalidInput):
        R.elliptic_params([0.0, 0.0, 1.0], 1, 2, 1e-7)


def test_contour_toy_pins_constant():
    # test_contour.cpp:84-95: energies (0, 2, 4), T = -0.75
    v = np.ones((1, 1))
    c = np.ones((1, 2))
    e = [0.0, 2.0, 4.0]
    spec = R.elliptic_params(e, 1, 2, 1e-10)
    t, n, est = R.coupled_coefficients_contour(v, c, e, spec)
    assert abs(t[0, 0] + 0.75) <= 0.75e-9 and n >= 17 and est <= 1e-10
    assert abs(R.coupled_coefficients_direct(np.ones((1, 1)), np.ones((1, 1)), [0.0, 2.0])[0, 0] + 0.5) < 1e-15


def test_cauchy_bound_kats():
    # test_contour.cpp:152-170
    assert abs(R.cauchy_error_bound(1.0, math.exp(2.0), 10) - math.exp(-math.pi ** 2)) <= 1e-12
    b1, b2 = R.cauchy_error_bound(1.0, math.exp(2.0), 7), R.cauchy_error_bound(1.0, math.exp(2.0), 14)
    assert abs(b2 - b1 * b1) <= 1e-12 * b2


def test_coulomb_kats():
    # test_model.cpp:68-80: kernel >= 0, v(0) = 0, kills constants
    dims, cell = (4, 4, 4), (5.0, 5.0, 5.0)
    v = R.coulomb_kernel(dims, cell)
    assert np.all(v >= 0) and v[0] == 0.0
    y = R.apply_coulomb(dims, cell, np.ones((64, 1)))
    assert np.max(np.abs(y)) <= 1e-12


# ---- restatement vs the compiled reference ---------------------------------

def _desk(ref, seed=1, dims=(8, 8, 8), n=16, gap=1.0, bw=4.0):
    psi, e = ref.build_synthetic(seed, dims, (6.0, 6.0, 6.0), n, n, gap, bw)
    return psi[:, :n], psi[:, n:], e


def test_restatement_matches_reference_isdf(ref):
    a, b, e = _desk(ref)
    p_ref = ref.select_points(a, b, 128)
    p_or, diag = R.select_points(a, b, 128, return_diag=True)
    assert np.array_equal(p_ref, p_or)
    assert diag["recompute_events"] == 0
    assert rel(R.fit_auxiliary_basis(a, b, p_or), ref.fit(a, b, p_ref)) <= 1e-12


def test_restatement_matches_reference_selection_shapes(ref):
    # N_mu = N_r selects all indices (test_isdf.cpp:36-44); N_mu > rank keeps the
    # swapped tail (assemble_K rank-deficient fixture, test_smw.cpp:74-85)
    psi, _ = ref.build_synthetic(3, (2, 2, 2), (4.0, 4.0, 4.0), 2, 2, 1.0, 2.0)
    a, b = psi[:, :2], psi[:, 2:]
    assert np.array_equal(R.select_points(a, b, 8), np.arange(8))
    psi, _ = ref.build_synthetic(2, (4, 4, 4), (6.0, 6.0, 6.0), 2, 2, 1.0, 2.0)
    a, b = psi[:, :2], psi[:, 2:]
    assert np.array_equal(R.select_points(a, b, 8), ref.select_points(a, b, 8))
    for seed, dims, n, nmu in [(6, (4, 4, 4), 4, 12), (5, (8, 4, 4), 6, 24), (3, (8, 8, 8), 8, 48)]:
        psi, _ = ref.build_synthetic(seed, dims, (6.0, 6.0, 6.0), n, n, 1.0, 4.0)
        a, b = psi[:, :n], psi[:, n:]
        assert np.array_equal(R.select_points(a, b, nmu), ref.select_points(a, b, nmu))


def test_restatement_matches_reference_contour(ref):
    a, b, e = _desk(ref, seed=11)
    pts = ref.select_points(a, b, 128)
    pv, pc = a[pts], b[pts]
    spec = R.elliptic_params(e, 16, 16, 1e-7)
    assert np.allclose(spec.as7(), ref.elliptic_params(e, 16, 16), rtol=1e-14, atol=0)
    nodes, w = R.trapezoid_nodes(spec, 24)
    assert rel(R.sum_node_terms(pv, pc, e, spec, nodes, w), ref.sum_node_terms(pv, pc, e, spec.as7(), nodes, w)) < 1e-13
    assert rel(R.coupled_coefficients_direct(pv, pc, e), ref.coupled_direct(pv, pc, e)) < 1e-13
    t_r, n_r, est_r, st = ref.coupled_contour(pv, pc, e)
    t_o, n_o, est_o = R.coupled_coefficients_contour(pv, pc, e, spec)
    assert st == 0 and n_r == n_o and rel(t_o, t_r) < 1e-13
    for t_node in (-spec.big_r, 0.1, spec.big_r):
        assert rel(R.node_term(pv, pc, e, spec, t_node), ref.node_term(pv, pc, e, spec.as7(), t_node)) < 1e-13


def test_restatement_matches_reference_smw(ref):
    dims, cell = (8, 8, 8), (6.0, 6.0, 6.0)
    a, b, e = _desk(ref, seed=7)
    pts = ref.select_points(a, b, 128)
    th = ref.fit(a, b, pts)
    t = ref.coupled_direct(a[pts], b[pts], e)
    x = ref.gaussian(19, 512, 4)
    assert rel(R.apply_coulomb(dims, cell, x), ref.apply_coulomb(dims, cell, x)) < 1e-13
    k_o = R.assemble_K(t, th, dims, cell)
    y_r, k_r, _ = ref.build_and_apply(t, th, dims, cell, x)
    assert rel(k_o, k_r) < 1e-12
    assert rel(R.epsilon_inverse_apply(th, k_o, dims, cell, x), y_r) < 1e-13


def gw_system(ref, seed=2, dims=(8, 8, 4), n=8, k=6.0):
    """test_gw.cpp:18-30 System: synthetic orbitals and the vc / vn / nn ISDF
    (pair factors isdf.hpp:166-173) through the reference."""
    psi, e = ref.build_synthetic(seed, dims, (6.0, 6.0, 6.0), n, n, 1.0, 4.0)
    a, b = psi[:, :n], psi[:, n:]
    decs = {}
    for label, (f1, f2) in {"vc": (a, b), "vn": (a, psi), "nn": (psi, psi)}.items():
        nmu = min(max(R.num_aux(k, f1.shape[1], f2.shape[1]), 1), f1.shape[0])
        pts = ref.select_points(f1, f2, nmu)
        decs[label] = (pts, ref.fit(f1, f2, pts))
    t = ref.coupled_direct(a[decs["vc"][0]], b[decs["vc"][0]], e)
    return psi, e, decs, t


def test_restatement_matches_reference_projections(ref):
    dims, cell = (8, 8, 4), (6.0, 6.0, 6.0)
    psi, e, decs, t = gw_system(ref)
    th_vc, th_vn, th_nn = decs["vc"][1], decs["vn"][1], decs["nn"][1]
    got_r = ref.project_screened(t, th_vc, dims, cell, th_vn, th_nn)
    k = R.assemble_K(t, th_vc, dims, cell)
    got_o = R.project_screened(th_vc, k, dims, cell, th_vn, th_nn)
    for x, y in zip(got_o, got_r):
        assert rel(x, y) <= 1e-11
    # test_gw.cpp:91-110: W_vn is P_vn^T (eps^-1 - I) V P_vn of the same ISDF eps
    n_r = psi.shape[0]
    em = R.epsilon_inverse_apply(th_vc, k, dims, cell, np.eye(n_r)) - np.eye(n_r)
    w_dense = R.symmetrize(th_vn.T @ (em @ R.apply_coulomb(dims, cell, th_vn)))
    assert rel(got_o[0], w_dense) <= 1e-9
    # zero interaction (test_gw.cpp:66-89)
    z = ref.project_screened(t, th_vc, dims, cell, th_vn, th_nn, zero=True)
    assert np.linalg.norm(z[0]) <= 1e-12 and np.linalg.norm(z[2]) <= 1e-12


def test_restatement_error_behaviour(ref):
    # degenerate Gram (test_isdf.cpp:228-231) and rank-deficient T (test_smw.cpp:74-85)
    with pytest.raises(R.NumericError):
        R.fit_auxiliary_basis(np.zeros((8, 2)), np.zeros((8, 2)), [1, 3])
    with pytest.raises(R.NumericError):
        ref.fit(np.zeros((8, 2)), np.zeros((8, 2)), [1, 3])
    with pytest.raises(R.InvalidInput):
        R.fit_auxiliary_basis(np.ones((8, 2)), np.ones((8, 2)), [3, 1])


# ---- golden fixtures (generated by tests/golden/make_golden.py from _ref) --

@pytest.mark.parametrize("path", sorted(p for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                                          if not os.path.basename(p).startswith(("gw_", "pivots_"))))
def test_oracle_against_golden(path):
    g = np.load(path)
    n_v, n_c = int(g["n_v"]), int(g["n_c"])
    dims, cell = tuple(g["dims"]), tuple(g["cell"])
    a, b = g["psi"][:, :n_v], g["psi"][:, n_v:n_v + n_c]
    pts = R.select_points(a, b, int(g["n_mu"]))
    assert np.array_equal(pts, g["pts"])
    assert rel(R.fit_auxiliary_basis(a, b, pts), g["theta"]) <= 1e-10
    pv, pc = a[pts], b[pts]
    assert rel(R.coupled_coefficients_direct(pv, pc, g["energies"]), g["t_direct"]) <= 1e-12
    spec = R.elliptic_params(g["energies"], n_v, n_c, 1e-7)
    if not spec.bypass:
        assert rel(R.coupled_coefficients_fixed(pv, pc, g["energies"], spec, int(g["n_lambda"])), g["t_fixed"]) <= 1e-12
    assert rel(R.assemble_K(g["t_direct"], g["theta"], dims, cell), g["k"]) <= 1e-10
    assert rel(R.epsilon_inverse_apply(g["theta"], g["k"], dims, cell, g["x"]), g["y"]) <= 1e-12


# ---- GW self-energies (gw.hpp:48-153; fixtures from make_golden_gw.py) -----

@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "gw_*.npz"))))
def test_sigma_restatement_against_golden(path):
    g = np.load(path)
    n_v = int(g["n_v"])
    dims, cell = tuple(g["dims"]), tuple(g["cell"])
    psi = g["psi"]
    for lab, (a, b) in {"vn": (psi[:, :n_v], psi), "nn": (psi, psi)}.items():
        assert np.array_equal(R.select_points(a, b, len(g[f"pts_{lab}"])), g[f"pts_{lab}"]), lab
        assert rel(R.fit_auxiliary_basis(a, b, g[f"pts_{lab}"]), g[f"theta_{lab}"]) <= 1e-10, lab
    w = R.project_screened(g["theta_vc"], g["k"], dims, cell, g["theta_vn"], g["theta_nn"])
    for got, name in zip(w, ("w_vn", "w_nn", "v_vn")):
        assert rel(got, g[name]) <= 1e-10, name
    sig = R.sigma_lowrank(psi, n_v, g["pts_vn"], g["pts_nn"], g["w_vn"], g["w_nn"], g["v_vn"])
    for got, want, name in zip(sig, g["sig_lowrank"], ("sex_x", "x", "coh", "total")):
        assert np.max(np.abs(got - want)) <= 1e-12 * max(np.max(np.abs(want)), 1e-30), name
    # test_gw.cpp:116-127: low-rank == conventional ISDF per band (1e-9 of the scale)
    scale = np.max(np.abs(g["sig_conventional"][3]))
    assert np.max(np.abs(g["sig_lowrank"] - g["sig_conventional"])) <= 1e-9 * scale
    # test_gw.cpp:174-184: sigma_x <= 0, exact additivity
    assert np.all(sig[1] <= 1e-12)
    assert np.array_equal(sig[3], sig[0] + sig[1] + sig[2])


def test_sigma_restatement_against_reference_leaf(ref):
    g = np.load(os.path.join(GOLDEN, "gw_s7.npz"))
    n_v = int(g["n_v"])
    rng = np.random.default_rng(4)
    nv, nn = len(g["pts_vn"]), len(g["pts_nn"])
    wv = R.symmetrize(rng.standard_normal((nv, nv)))
    wn = R.symmetrize(rng.standard_normal((nn, nn)))
    vv = R.symmetrize(rng.standard_normal((nv, nv)))
    got = R.sigma_lowrank(g["psi"], n_v, g["pts_vn"], g["pts_nn"], wv, wn, vv)
    want = ref.sigma_lowrank(g["psi"], n_v, g["pts_vn"], g["pts_nn"], wv, wn, vv)
    for a, b in zip(got, want):
        assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(b))


def test_quasiparticle_kats(ref):
    # test_gw.cpp:186-233
    e = np.array([-0.4, -0.2, 0.1, 0.3])
    assert np.array_equal(R.quasiparticle_energies(e, np.zeros(4), np.zeros(4)), e)
    got = R.quasiparticle_energies(e, np.full(4, 0.05), np.full(4, 0.25))
    assert np.allclose(got, e + 0.25 - 0.05, rtol=1e-14)
    assert np.array_equal(got, ref.quasiparticle(e, np.full(4, 0.05), np.full(4, 0.25)))
    with pytest.raises(R.InvalidInput):
        R.quasiparticle_energies(e, np.zeros(4), np.zeros(3))
    with pytest.raises(R.InvalidInput):
        ref.quasiparticle(e, np.zeros(4), np.zeros(3))


# ---- the stage-wise checkers used at the large configs ----------------------

@pytest.mark.parametrize("name", ["si8shaped_s1", "acc_s3", "wide_s3"])
def test_stagewise_checkers_equal_full_reference_calls(ref, name):
    """ref.fit_rows / pvp_cols / smw_from_pvp / eps_apply_vp (the large-config
    checkers of tests/test_gpu_configs.py) are bit-identical to the rows /
    columns of the reference's own fit_auxiliary_basis, assemble_K and
    build_epsilon_inverse + epsilon_inverse_apply (isdf.hpp:118-163,
    smw.hpp:42-103) — they only restrict and parallelise separable work."""
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    psi, nv = g["psi"], int(g["n_v"])
    a, b, pts = psi[:, :nv], psi[:, nv:], g["pts"]
    dims, cell = tuple(int(x) for x in g["dims"]), tuple(float(x) for x in g["cell"])
    th = ref.fit(a, b, pts)
    rows = np.sort(np.random.default_rng(0).choice(psi.shape[0], psi.shape[0] // 3, replace=False))
    th_rows, pinv = ref.fit_rows(a[rows], b[rows], a[pts], b[pts], threads=3)
    assert np.array_equal(th_rows, th[rows])
    t = g["t_fixed"]
    x = g["x"]
    y, k, vp = ref.build_and_apply(t, th, dims, cell, x, threads=2, want_vp=True)
    pvp, vpc = ref.pvp_cols(th, dims, cell, np.arange(th.shape[1]), threads=3, want_vp=True)
    assert np.array_equal(vpc, vp)
    k2 = ref.smw_from_pvp(t, pvp, threads=4)
    assert np.array_equal(k2, k)
    assert np.array_equal(ref.eps_apply_vp(th, k2, vpc, x), y)
    assert rel(ref.eps_apply_factored(th, k2, dims, cell, x, threads=2), y) <= 1e-13
    cols = np.array([3, 0, th.shape[1] - 1], dtype=np.int32)
    assert np.array_equal(ref.pvp_cols(th, dims, cell, cols, threads=2), pvp[:, cols])


def test_select_oracle_layout_independent():
    """oracle/select.c on row-major copies gives the same pivots, order and
    margins on a transposed-storage input (the sums run in one fixed order)."""
    rng = np.random.default_rng(5)
    q = np.linalg.qr(rng.standard_normal((3000, 24)))[0]
    a, b = q[:, :12], q[:, 12:]
    p1, d1 = R.select_points(np.asfortranarray(a), np.asfortranarray(b), 64, return_diag=True)
    p2, d2 = R.select_points(np.ascontiguousarray(a), np.ascontiguousarray(b), 64, return_diag=True)
    assert np.array_equal(p1, p2) and np.array_equal(d1["margins"], d2["margins"])
    assert np.array_equal(d1["order"], d2["order"])
