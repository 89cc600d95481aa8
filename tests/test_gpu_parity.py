"""GPU parity: the B200 path (liblrgw_cuda.so through the Python mirror of the
reference API) against the compiled reference (oracle/_ref), the golden
fixtures and the reference's own known-answer tests.

Tolerances (BASELINE.json north_star): ISDF points bit-exact; Theta, T, K and
eps^-1 X within relative Frobenius error 1e-10 in FP64."""
import glob
import os

import numpy as np
import pytest

from helpers import rel

pytestmark = pytest.mark.gpu

TOL = 1e-10
GOLDEN = sorted(p for p in glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz"))
                if not os.path.basename(p).startswith(("gw_", "pivots_")))


@pytest.fixture(scope="module")
def L():
    from paper_2403_12340_b200 import lrgw

    return lrgw


def _desk(ref, seed=1, dims=(8, 8, 8), n=16, gap=1.0, bw=4.0, cell=(6.0, 6.0, 6.0)):
    psi, e = ref.build_synthetic(seed, dims, cell, n, n, gap, bw)
    return psi[:, :n], psi[:, n:], e


# ---- golden fixtures --------------------------------------------------------

@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_golden_pipeline(L, ctx, path):
    g = np.load(path)
    n_v, n_c = int(g["n_v"]), int(g["n_c"])
    dims, cell = tuple(int(x) for x in g["dims"]), tuple(g["cell"])
    a, b = g["psi"][:, :n_v], g["psi"][:, n_v:n_v + n_c]
    pts = L.select_interpolation_points(a, b, int(g["n_mu"]), ctx=ctx)
    assert np.array_equal(pts, g["pts"]), "ISDF points must be bit-exact"
    theta = L.fit_auxiliary_basis(a, b, pts, ctx=ctx)
    assert rel(theta, g["theta"]) <= TOL
    pv, pc = a[pts], b[pts]
    assert rel(L.coupled_coefficients_direct(pv, pc, g["energies"], ctx=ctx).t, g["t_direct"]) <= TOL
    assert rel(L.coupled_coefficients_fixed(pv, pc, g["energies"], int(g["n_lambda"]), ctx=ctx).t,
               g["t_fixed"]) <= TOL
    spec = L.elliptic_params(g["energies"], n_v, n_c, 1e-7)
    cc = L.coupled_coefficients_contour(pv, pc, g["energies"], spec, ctx=ctx)
    assert cc.nodes_used == int(g["nodes_used"]) and rel(cc.t, g["t_adapt"]) <= TOL
    k = L.assemble_K(g["t_direct"], g["theta"], dims, cell, ctx=ctx)
    assert rel(k, g["k"]) <= TOL
    e = L.build_epsilon_inverse(g["t_direct"], g["theta"], dims, cell, ctx=ctx)
    assert rel(L.epsilon_inverse_apply(e, g["x"]), g["y"]) <= TOL


# ---- K3 quadrature ----------------------------------------------------------

def test_sum_node_terms_matches_reference(L, ctx, ref):
    a, b, e = _desk(ref, seed=11)
    pts = ref.select_points(a, b, 128)
    pv, pc = a[pts], b[pts]
    s7 = ref.elliptic_params(e, 16, 16)
    spec = L.elliptic_params(e, 16, 16, 1e-7)
    assert np.allclose(spec.as7(), s7, rtol=1e-14, atol=0)
    rng = np.random.default_rng(5)
    nodes = np.sort(rng.uniform(-s7[3], s7[3], 13))
    w = rng.uniform(0.1, 1.0, 13)
    acc_ref = ref.sum_node_terms(pv, pc, e, s7, nodes, w)
    acc = L.sum_node_terms(pv, pc, e, spec, nodes, w, ctx=ctx)
    assert rel(acc, 0.5 * (acc_ref + acc_ref.T)) <= TOL


@pytest.mark.parametrize("n_mu,n_v,n_c", [(1, 1, 1), (7, 3, 5), (65, 16, 16), (130, 17, 33), (200, 40, 24)])
def test_quadrature_ragged_shapes(L, ctx, ref, n_mu, n_v, n_c):
    rng = np.random.default_rng(n_mu)
    pv = rng.standard_normal((n_mu, n_v))
    pc = rng.standard_normal((n_mu, n_c))
    e = np.concatenate([np.sort(rng.uniform(-1, -0.2, n_v)), np.sort(rng.uniform(0.1, 2.0, n_c))])
    t_dir = ref.coupled_direct(pv, pc, e)
    assert rel(L.coupled_coefficients_direct(pv, pc, e, ctx=ctx).t, t_dir) <= TOL
    s7 = ref.elliptic_params(e, n_v, n_c)
    if s7[6] == 0:
        spec = L.elliptic_params(e, n_v, n_c, 1e-7)
        nodes = np.linspace(-s7[3], s7[3], 9)
        w = np.full(9, 0.3)
        acc_ref = ref.sum_node_terms(pv, pc, e, s7, nodes, w)
        assert rel(L.sum_node_terms(pv, pc, e, spec, nodes, w, ctx=ctx), 0.5 * (acc_ref + acc_ref.T)) <= TOL


# the k-tile depths of the TMA feed (quad4.cu: 16 / 24 / 32 / 40 / 48 / 64 by band padding), band
# tails, ragged row tiles; odd n_mu keeps the cp.async feed
@pytest.mark.parametrize("n_mu,n_v,n_c", [(130, 17, 33), (192, 120, 120), (256, 48, 96), (320, 64, 128),
                                          (96, 24, 72), (200, 40, 80), (258, 32, 100), (131, 16, 16)])
def test_quadrature_feeds_agree(L, ctx, ref, monkeypatch, n_mu, n_v, n_c):
    rng = np.random.default_rng(n_mu + n_v)
    pv = rng.standard_normal((n_mu, n_v))
    pc = rng.standard_normal((n_mu, n_c))
    e = np.concatenate([np.sort(rng.uniform(-1, -0.2, n_v)), np.sort(rng.uniform(0.1, 2.0, n_c))])
    s7 = ref.elliptic_params(e, n_v, n_c)
    assert s7[6] == 0
    spec = L.elliptic_params(e, n_v, n_c, 1e-7)
    nodes = np.linspace(-s7[3], s7[3], 11)
    w = np.linspace(0.2, 0.7, 11)
    acc_ref = ref.sum_node_terms(pv, pc, e, s7, nodes, w)
    acc_ref = 0.5 * (acc_ref + acc_ref.T)
    out = {}
    for feed in ("0", "1"):
        monkeypatch.setenv("LRGW_QUAD_TMA", feed)
        out[feed] = L.sum_node_terms(pv, pc, e, spec, nodes, w, ctx=ctx)
        assert rel(out[feed], acc_ref) <= TOL
        again = L.sum_node_terms(pv, pc, e, spec, nodes, w, ctx=ctx)
        assert np.array_equal(out[feed], again)  # fixed summation order, no staging race
    assert rel(out["1"], out["0"]) <= 1e-13


def test_contour_toy_and_errors(L, ctx):
    # test_contour.cpp:84-95 (T = -0.75), 175-200 (bypass, max_nodes)
    e = [0.0, 2.0, 4.0]
    spec = L.elliptic_params(e, 1, 2, 1e-10)
    cc = L.coupled_coefficients_contour(np.ones((1, 1)), np.ones((1, 2)), e, spec, ctx=ctx)
    assert abs(cc.t[0, 0] + 0.75) <= 0.75e-9 and cc.nodes_used >= 17 and cc.est_rel_error <= 1e-10
    assert abs(L.coupled_coefficients_direct(np.ones((1, 1)), np.ones((1, 1)), [0.0, 2.0], ctx=ctx).t[0, 0]
               + 0.5) <= 1e-15
    byp = L.elliptic_params([0.0, 2.0], 1, 1, 1e-7)
    assert byp.bypass
    with pytest.raises(L.InvalidInput):
        L.coupled_coefficients_contour(np.ones((1, 1)), np.ones((1, 1)), [0.0, 2.0], byp, ctx=ctx)


def test_contour_max_nodes_carries_best(L, ctx, ref):
    a, b, e = _desk(ref, seed=5, gap=0.05, bw=4.95)
    pts = ref.select_points(a, b, 128)
    pv, pc = a[pts], b[pts]
    spec = L.elliptic_params(e, 16, 16, 1e-16, 33)
    with pytest.raises(L.ContourConvergenceError) as ei:
        L.coupled_coefficients_contour(pv, pc, e, spec, ctx=ctx)
    best = ei.value.best
    t_ref, n_ref, est_ref, st = ref.coupled_contour(pv, pc, e, 1e-16, 33)
    assert st == 5 and best.nodes_used == n_ref == 33
    assert rel(best.t, t_ref) <= TOL and abs(best.est_rel_error - est_ref) <= 1e-6 * est_ref


def test_refinement_levels_match_reference(L, ctx, ref):
    a, b, e = _desk(ref, seed=3, gap=0.05, bw=4.95)
    pts = ref.select_points(a, b, 128)
    pv, pc = a[pts], b[pts]
    spec = L.elliptic_params(e, 16, 16, 1e-7)
    levels = L.contour_refinement_levels(pv, pc, e, spec, 257, ctx=ctx)
    t_dir = ref.coupled_direct(pv, pc, e)
    assert [n for n, _ in levels] == [17, 33, 65, 129, 257]
    errs = [rel(t, t_dir) for _, t in levels]
    assert errs[-1] < errs[0]


# ---- ISDF ---------------------------------------------------------------------

@pytest.mark.parametrize("seed,dims,n,n_mu", [(1, (8, 8, 8), 16, 128), (2, (8, 8, 8), 16, 64), (6, (4, 4, 4), 4, 12),
                                              (5, (8, 4, 4), 6, 24), (3, (2, 2, 2), 2, 8), (2, (4, 4, 4), 2, 8),
                                              (9, (8, 8, 8), 16, 256)])
def test_selection_bit_exact(L, ctx, ref, seed, dims, n, n_mu):
    a, b, e = _desk(ref, seed=seed, dims=dims, n=n)
    assert np.array_equal(L.select_interpolation_points(a, b, n_mu, ctx=ctx), ref.select_points(a, b, n_mu))


@pytest.mark.parametrize("batch", [1, 8, 64, 128])
def test_selection_batch_invariant(L, ref, batch):
    ctx = L.Context(0)
    ctx.set_select_batch(batch)
    a, b, e = _desk(ref, seed=4)
    assert np.array_equal(L.select_interpolation_points(a, b, 128, ctx=ctx), ref.select_points(a, b, 128))
    ctx.close()


def test_selection_errors(L, ctx, ref):
    a, b, _ = _desk(ref)
    with pytest.raises(L.InvalidInput):
        L.select_interpolation_points(a, b, a.shape[0] + 1, ctx=ctx)
    with pytest.raises(L.InvalidInput):
        L.select_interpolation_points(a, b, 0, ctx=ctx)
    with pytest.raises(L.GuardExceeded):  # the sketch materialises the pair matrix (isdf.hpp:49, 77-78)
        psi, _ = ref.build_synthetic(2, (24, 24, 24), (10.0, 10.0, 10.0), 72, 72, 1.0, 4.0)
        L.select_interpolation_points(psi[:, :72], psi[:, 72:], 64, method="qrcp_sketched", ctx=ctx)


@pytest.mark.parametrize("seed,dims,n,k", [(1, (8, 8, 8), 24, 4.0), (3, (8, 8, 8), 32, 3.0), (5, (8, 8, 4), 16, 2.0),
                                           (2, (8, 8, 8), 16, 8.0)])
def test_sketched_selection_matches_reference(L, ctx, ref, seed, dims, n, k):
    """PointSelector::qrcp_sketched (isdf.hpp:95-112): the reference's fixed
    Gaussian sketch of the pair rows, then QRCP — pivots bit-exact. The last
    case has 2 N_mu >= N1 N2, where the reference falls back to plain QRCP."""
    a, b, _ = _desk(ref, seed=seed, dims=dims, n=n)
    n_mu = ref.num_aux(k, n, n)
    got = L.select_interpolation_points(a, b, n_mu, method="qrcp_sketched", ctx=ctx)
    assert np.array_equal(got, ref.select_points(a, b, n_mu, sketched=True))


def test_fit_fallback_and_degenerate(L, ctx, ref):
    # test_isdf.cpp:205-231
    psi, _ = ref.build_synthetic(21, (4, 4, 2), (5.0, 5.0, 5.0), 2, 2, 1.0, 2.0)
    a, b = psi[:, :2].copy(), psi[:, 2:].copy()
    a[7, :] = 0.0
    b[7, :] = 0.0
    pts = list(ref.select_points(a, b, 4))
    pts[0] = 7
    pts = np.array(sorted(set(pts)), dtype=np.int32)
    th = L.fit_auxiliary_basis(a, b, pts, ctx=ctx)
    th_ref = ref.fit(a, b, pts)
    assert np.all(np.isfinite(th)) and rel(th, th_ref) <= 1e-8
    with pytest.raises(L.NumericError):
        L.fit_auxiliary_basis(np.zeros((8, 2)), np.zeros((8, 2)), [1, 3], ctx=ctx)
    with pytest.raises(L.InvalidInput):
        L.fit_auxiliary_basis(a, b, [3, 1], ctx=ctx)


def test_fit_all_points_exact(L, ctx, ref):
    # test_isdf.cpp:78-87: every grid point -> exact interpolation
    psi, _ = ref.build_synthetic(5, (4, 4, 2), (5.0, 5.0, 5.0), 3, 3, 1.0, 2.0)
    a, b = psi[:, :3], psi[:, 3:]
    th = L.fit_auxiliary_basis(a, b, np.arange(32, dtype=np.int32), ctx=ctx)
    assert ref.isdf_error(a, b, np.arange(32), th) <= 1e-9


# ---- Coulomb + SMW ------------------------------------------------------------

@pytest.mark.parametrize("dims", [(4, 4, 4), (8, 8, 8), (5, 6, 7), (8, 4, 2), (24, 24, 24)])
def test_apply_coulomb_matches_reference(L, ctx, ref, dims):
    cell = (5.0, 6.5, 7.25)
    n_r = int(np.prod(dims))
    x = ref.gaussian(9, n_r, 3)
    assert rel(L.apply_coulomb(dims, cell, x, ctx=ctx), ref.apply_coulomb(dims, cell, x)) <= TOL
    assert np.max(np.abs(L.apply_coulomb(dims, cell, np.ones((n_r, 1)), ctx=ctx))) <= 1e-12
    assert np.max(np.abs(L.apply_coulomb(dims, cell, np.zeros((n_r, 2)), ctx=ctx))) == 0.0
    assert np.allclose(L.coulomb_kernel(dims, cell), ref.coulomb_kernel(dims, cell), rtol=1e-15, atol=0)


def test_smw_kats(L, ctx, ref):
    dims, cell = (4, 4, 4), (6.0, 6.0, 6.0)
    psi, e = ref.build_synthetic(1, dims, cell, 4, 4, 1.0, 4.0)
    a, b = psi[:, :4], psi[:, 4:]
    pts = ref.select_points(a, b, 8)
    th = ref.fit(a, b, pts)
    t = ref.coupled_direct(a[pts], b[pts], e)
    # V = 0 => K = 2T (test_smw.cpp:58-64)
    k0 = L.assemble_K(t, th, dims, cell, zero_kernel=True, ctx=ctx)
    assert rel(k0, 2.0 * t) <= 1e-9
    # K symmetric negative definite (test_smw.cpp:66-72)
    k = L.assemble_K(t, th, dims, cell, ctx=ctx)
    assert np.linalg.norm(k - k.T) <= 1e-10 * np.linalg.norm(k)
    assert np.max(np.linalg.eigvalsh(k)) < 0
    # K = 0 => identity apply, exactly (test_smw.cpp:87-97)
    e0 = L.epsilon_inverse_from_parts(th, np.zeros((8, 8)), dims, cell, ctx=ctx)
    x = ref.gaussian(11, 64, 3)
    assert np.array_equal(L.epsilon_inverse_apply(e0, x), x)
    # linearity (test_smw.cpp:99-111)
    ep = L.build_epsilon_inverse(t, th, dims, cell, ctx=ctx)
    x1, x2 = ref.gaussian(13, 64, 1), ref.gaussian(14, 64, 1)
    lhs = L.epsilon_inverse_apply(ep, 1.7 * x1 - 0.4 * x2)
    rhs = 1.7 * L.epsilon_inverse_apply(ep, x1) - 0.4 * L.epsilon_inverse_apply(ep, x2)
    assert rel(lhs, rhs) <= 1e-12


def test_assemble_K_rejects_rank_deficient_T(L, ctx, ref):
    # test_smw.cpp:74-85: N_mu = 8 > 4 pairs -> T singular
    dims, cell = (4, 4, 4), (6.0, 6.0, 6.0)
    psi, e = ref.build_synthetic(2, dims, cell, 2, 2, 1.0, 2.0)
    a, b = psi[:, :2], psi[:, 2:]
    pts = L.select_interpolation_points(a, b, 8, ctx=ctx)
    assert np.array_equal(pts, ref.select_points(a, b, 8))
    th = ref.fit(a, b, pts)
    t = ref.coupled_direct(a[pts], b[pts], e)
    with pytest.raises(L.NumericError):
        L.assemble_K(t, th, dims, cell, ctx=ctx)
    from oracle import restate as R

    with pytest.raises(R.NumericError):
        ref.assemble_K(t, th, dims, cell)


@pytest.mark.parametrize("seed,dims,n,k", [(1, (8, 8, 8), 16, 8.0), (2, (8, 8, 4), 12, 6.0), (3, (8, 8, 8), 8, 6.0),
                                           (4, (4, 4, 4), 4, 3.0), (5, (8, 4, 4), 6, 4.0)])
def test_smw_equals_dense_lu(L, ctx, ref, seed, dims, n, k):
    # acceptance criterion 1 (acceptance.cpp:116-149): SMW == dense LU <= 1e-10
    cell = tuple(0.75 * d for d in dims)
    psi, e = ref.build_synthetic(seed, dims, cell, n, n, 1.0, 4.0)
    a, b = psi[:, :n], psi[:, n:]
    n_r = psi.shape[0]
    n_mu = min(max(L.num_aux(k, n, n), 1), n_r)
    pts = L.select_interpolation_points(a, b, n_mu, ctx=ctx)
    th = L.fit_auxiliary_basis(a, b, pts, ctx=ctx)
    t = L.coupled_coefficients_direct(a[pts], b[pts], e, ctx=ctx).t
    ep = L.build_epsilon_inverse(t, th, dims, cell, ctx=ctx)
    eps, eps_inv = ref.epsilon_dense(psi, n, n, e, dims, cell, pts, th)
    dense = L.epsilon_inverse_apply(ep, np.eye(n_r))
    assert rel(dense, eps_inv) <= 1e-10
    x = ref.gaussian(19, n_r, 1)
    y = L.epsilon_inverse_apply(ep, x)
    assert np.linalg.norm(eps @ y - x) <= 1e-9 * np.linalg.norm(x)


# ---- the Si8 BASELINE config end to end, against the reference ------------------

def test_si8_pipeline_matches_reference(L, ctx, ref):
    from paper_2403_12340_b200 import synth

    cfg = synth.CONFIGS["si8"]
    psi = synth.orbitals_host(cfg)
    e = synth.energies(cfg)
    a, b = psi[:, :16], psi[:, 16:]
    n_mu = L.num_aux(cfg.k_mu, 16, 16)
    pts = L.select_interpolation_points(a, b, n_mu, ctx=ctx)
    pts_ref = ref.select_points(a, b, n_mu)
    assert np.array_equal(pts, pts_ref)
    th = L.fit_auxiliary_basis(a, b, pts, ctx=ctx)
    th_ref = ref.fit(a, b, pts_ref)
    assert rel(th, th_ref) <= TOL
    pv, pc = a[pts], b[pts]
    s7 = ref.elliptic_params(e, 16, 16)
    h = 2 * s7[3] / cfg.n_lambda
    nodes = [-s7[3] + i * h for i in range(cfg.n_lambda + 1)]
    w = [0.5 * h if i in (0, cfg.n_lambda) else h for i in range(cfg.n_lambda + 1)]
    acc = 2 * np.sqrt(s7[0] * s7[1]) / (np.pi * s7[2]) * ref.sum_node_terms(pv, pc, e, s7, nodes, w)
    t_ref = 0.5 * (acc + acc.T)
    t = L.coupled_coefficients_fixed(pv, pc, e, cfg.n_lambda, ctx=ctx).t
    assert rel(t, t_ref) <= TOL
    x = synth.probe_host(cfg.n_r)
    y_ref, k_ref, _ = ref.build_and_apply(t_ref, th_ref, cfg.dims, cfg.cell3, x, threads=8)
    ep = L.build_epsilon_inverse(t, th, cfg.dims, cfg.cell3, ctx=ctx)
    assert rel(ep.k, k_ref) <= TOL
    assert rel(L.epsilon_inverse_apply(ep, x), y_ref) <= TOL


_DOWNDATE_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2403_12340_b200 import lrgw
rng = np.random.default_rng(23)
n_r = int(sys.argv[2])
q = np.linalg.qr(rng.standard_normal((n_r, 28)))[0]
a, b = np.asfortranarray(q[:, :14]), np.asfortranarray(q[:, 14:])
ctx = lrgw.Context(0)
ctx.set_select_batch(24)
pts = lrgw.select_interpolation_points(a, b, 96, ctx=ctx)
np.save(sys.argv[3], pts)
"""


@pytest.mark.parametrize("n_r", [315, 1000])
def test_selection_pivots_with_and_without_fused_downdate(tmp_path, n_r):
    """The residual downdate fused into the L-block GEMM epilogue and the
    separate downdate kernel (LRGW_FUSED_DOWNDATE=0) round d differently; on
    odd and even row counts both must give the oracle's pivots (several
    candidate blocks, batch 24)."""
    import os
    import subprocess
    import sys

    from oracle import restate as R

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "sel.py"
    script.write_text(_DOWNDATE_SCRIPT)
    out = {}
    for fused in ("1", "0"):
        env = dict(os.environ, LRGW_FUSED_DOWNDATE=fused)
        path = tmp_path / f"pts_{fused}.npy"
        r = subprocess.run([sys.executable, str(script), root, str(n_r), str(path)], env=env, capture_output=True,
                           text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        out[fused] = np.load(path)
    rng = np.random.default_rng(23)
    q = np.linalg.qr(rng.standard_normal((n_r, 28)))[0]
    want = R.select_points(q[:, :14], q[:, 14:], 96)
    assert np.array_equal(out["1"], want) and np.array_equal(out["0"], want)


_ENGINE_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2403_12340_b200 import lrgw
n_r = int(sys.argv[2])
rng = np.random.default_rng(31)
q = np.linalg.qr(rng.standard_normal((n_r, 48)))[0]
a, b = np.asfortranarray(q[:, :24]), np.asfortranarray(q[:, 24:])
pts = lrgw.select_interpolation_points(a, b, 300, ctx=lrgw.Context(0))
np.save(sys.argv[3], pts)
"""


@pytest.mark.parametrize("variant", ["", "LRGW_SELECT_DEVLOOP=1", "LRGW_PANEL=0", "LRGW_PANEL=0 LRGW_TMA_TALL=0"])
def test_selection_engines_agree_with_oracle(tmp_path, variant):
    """Every selection block engine gives the oracle's pivots (linalg.hpp:26-111)
    on a shape with several candidate blocks that reaches the tall-skinny
    engines (n_r = 20000): the fused panel with the host block loop (default
    at this Hadamard depth), the device-driven block loop, the three TMA
    launches and the three cp.async launches."""
    import os
    import subprocess
    import sys

    from oracle import restate as R

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "sel.py"
    script.write_text(_ENGINE_SCRIPT)
    env = dict(os.environ)
    for kv in variant.split():
        k, v = kv.split("=")
        env[k] = v
    path = tmp_path / "pts.npy"
    r = subprocess.run([sys.executable, str(script), root, "20000", str(path)], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    rng = np.random.default_rng(31)
    q = np.linalg.qr(rng.standard_normal((20000, 48)))[0]
    want = R.select_points(q[:, :24], q[:, 24:], 300)
    assert np.array_equal(np.load(path), want)


_FFT_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2403_12340_b200 import lrgw
n = int(sys.argv[2])
rng = np.random.default_rng(n)
x = rng.standard_normal((n ** 3, 6))
y = lrgw.apply_coulomb((n, n, n), (9.0, 9.0, 9.0), x, ctx=lrgw.Context(0))
np.save(sys.argv[3], y)
"""


@pytest.mark.parametrize("n", [24, 48])
def test_own_fft_matches_cufft_leaf(tmp_path, n):
    """The opt-in two-pass D2Z (fft.cu, LRGW_FFT_OWN=1) gives the Coulomb
    application (model.hpp:208-223) of the cuFFT leaf to round-off."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "fft.py"
    script.write_text(_FFT_SCRIPT)
    out = {}
    for own in ("0", "1"):
        path = tmp_path / f"y_{own}.npy"
        r = subprocess.run([sys.executable, str(script), root, str(n), str(path)],
                           env=dict(os.environ, LRGW_FFT_OWN=own), capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        out[own] = np.load(path)
    rel = np.linalg.norm(out["1"] - out["0"]) / np.linalg.norm(out["0"])
    assert rel <= 1e-13, rel
