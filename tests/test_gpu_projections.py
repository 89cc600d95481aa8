"""GPU parity for the vn / nn ISDF and the projected screened interactions
(reference isdf.hpp:166-183, gw.hpp:73-88) against the
compiled reference (oracle/_ref) and the restatement (oracle/restate.py).

Tolerances as for the vc path: points bit-exact, everything else within
relative Frobenius error 1e-10 (FP64)."""
import numpy as np
import pytest

from helpers import rel
from oracle import restate as R

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.fixture(scope="module")
def L():
    from paper_2403_12340_b200 import lrgw

    return lrgw


def _system(ref, L, ctx, seed, dims, n, k):
    """test_gw.cpp:18-30: vc / vn / nn ISDF on the GPU, checked against the
    reference's own selection and fit on the same pair factors."""
    psi, e = ref.build_synthetic(seed, dims, (6.0, 6.0, 6.0), n, n, 1.0, 4.0)
    decs = {}
    for label in ("vc", "vn", "nn"):
        d = L.build_isdf(psi, n, n, k, ctx=ctx, label=label)
        a, b = L.pair_factors(psi, n, n, label)
        pts_ref = ref.select_points(a, b, d.n_mu)
        assert np.array_equal(d.point_indices, pts_ref), f"{label}: pivots must be bit-exact"
        assert rel(d.p, ref.fit(a, b, pts_ref)) <= TOL, label
        decs[label] = d
    pts = decs["vc"].point_indices
    t = ref.coupled_direct(psi[pts, :n], psi[pts, n:], e)
    return psi, e, decs, t


@pytest.mark.parametrize("seed,dims,n,k", [(2, (8, 8, 4), 8, 6.0), (5, (8, 8, 8), 12, 4.0)])
def test_projections_match_reference(ref, L, ctx, seed, dims, n, k):
    cell = (6.0, 6.0, 6.0)
    psi, e, decs, t = _system(ref, L, ctx, seed, dims, n, k)
    th = decs["vc"].p
    eps = L.build_epsilon_inverse(t, th, dims, cell, ctx=ctx)
    got = L.project_screened_interactions(eps, decs["vn"], decs["nn"])
    want = ref.project_screened(t, th, dims, cell, decs["vn"].p, decs["nn"].p)
    for name, x, y in zip(("w_vn", "w_nn", "v_vn"), (got.w_vn, got.w_nn, got.v_vn), want):
        assert rel(x, y) <= TOL, name
        assert np.array_equal(x, x.T), f"{name} symmetric"
    # test_gw.cpp:91-110: W_vn = P_vn^T (eps^-1 - I) V P_vn of the same eps
    n_r = psi.shape[0]
    em = L.epsilon_inverse_apply(eps, np.eye(n_r)) - np.eye(n_r)
    w_dense = R.symmetrize(decs["vn"].p.T @ (em @ R.apply_coulomb(dims, cell, decs["vn"].p)))
    assert rel(got.w_vn, w_dense) <= 1e-9


def test_projections_zero_interaction(ref, L, ctx):
    """test_gw.cpp:66-89: V = 0 gives zero projections."""
    dims, cell = (4, 4, 4), (6.0, 6.0, 6.0)
    psi, e, decs, t = _system(ref, L, ctx, 1, dims, 3, 2.0)
    eps = L.build_epsilon_inverse(t, decs["vc"].p, dims, cell, zero_kernel=True, ctx=ctx)
    got = L.project_screened_interactions(eps, decs["vn"], decs["nn"])
    assert np.linalg.norm(got.w_vn) <= 1e-12
    assert np.linalg.norm(got.w_nn) <= 1e-12
    assert np.linalg.norm(got.v_vn) <= 1e-12


def test_projections_mid_size_against_restatement(L, ctx):
    """Si8-sized grid (24^3) with N_v = N_c = 16: vn / nn ISDF and the
    projections against the restatement on the GPU's own factors."""
    from paper_2403_12340_b200 import synth

    cfg = synth.CONFIGS["si8"]
    psi = synth.orbitals_host(cfg, seed=3)
    e = synth.energies(cfg)
    n = cfg.n_v
    dims, cell = cfg.dims, cfg.cell3
    dec = {lab: L.build_isdf(psi, n, n, 4.0, ctx=ctx, label=lab) for lab in ("vc", "vn", "nn")}
    for lab in ("vn", "nn"):
        a, b = L.pair_factors(psi, n, n, lab)
        assert np.array_equal(dec[lab].point_indices, R.select_points(a, b, dec[lab].n_mu)), lab
    pts = dec["vc"].point_indices
    t = R.coupled_coefficients_direct(psi[pts, :n], psi[pts, n:], e)
    eps = L.build_epsilon_inverse(t, dec["vc"].p, dims, cell, ctx=ctx)
    got = L.project_screened_interactions(eps, dec["vn"], dec["nn"])
    want = R.project_screened(dec["vc"].p, eps.k, dims, cell, dec["vn"].p, dec["nn"].p)
    for name, x, y in zip(("w_vn", "w_nn", "v_vn"), (got.w_vn, got.w_nn, got.v_vn), want):
        assert rel(x, y) <= TOL, name


def test_projections_error_behaviour(L, ctx):
    dims, cell = (4, 4, 4), (6.0, 6.0, 6.0)
    rng = np.random.default_rng(0)
    p = np.linalg.qr(rng.standard_normal((64, 6)))[0]
    t = -np.eye(6) * 1e-3
    eps = L.build_epsilon_inverse(t, p, dims, cell, ctx=ctx)
    with pytest.raises(L.InvalidInput):
        L.project_screened_interactions(eps, np.zeros((63, 4)), np.zeros((64, 4)))
    got = L.project_screened_interactions(eps, np.zeros((64, 0)), np.zeros((64, 0)))
    assert got.w_vn.shape == (0, 0) and got.w_nn.shape == (0, 0)
