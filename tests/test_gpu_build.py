"""GPU: the whole device-resident build (lrgw_build, stages 1-5) at BASELINE
configs — against the reference at Si8 and through size-independent
properties (plus the oracle's bit-exact pivot sequence) at Si64."""
import numpy as np
import pytest

from helpers import rel

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _cm(t):
    return t.t().contiguous().t()


def _eps_residual(L, ctx, ep, cfg, x):
    """||eps (eps^-1 x) - x|| / ||x|| with eps = I - V (2 Theta T Theta^T)
    applied matrix-free on the device (smw.hpp:116-169 definition)."""
    import torch

    th_p, k_p, t_p = ep.device_ptrs()
    theta = L_tensor(th_p, (ep.n_r, ep.n_mu))
    tmat = L_tensor(t_p, (ep.n_mu, ep.n_mu))
    y = torch.empty_like(x)
    L.eps_apply_dev(ep, x, y)
    u = _cm(torch.empty(ep.n_mu, x.shape[1], dtype=torch.float64, device="cuda"))
    L.dgemm_dev("T", "N", 1.0, theta, y, 0.0, u, ctx=ctx)
    w = _cm(torch.empty_like(u))
    L.dgemm_dev("N", "N", 2.0, tmat, u, 0.0, w, ctx=ctx)
    z = _cm(torch.empty_like(x))
    L.dgemm_dev("N", "N", 1.0, theta, w, 0.0, z, ctx=ctx)
    vz = _cm(torch.empty_like(x))
    L.coulomb_apply_dev(cfg.dims, cfg.cell3, z, vz, ctx=ctx)
    r = y - vz - x
    return float(torch.linalg.norm(r) / torch.linalg.norm(x))


def L_tensor(ptr, shape):
    """Zero-copy column-major torch view of a device buffer owned by an eps handle."""
    import torch

    n = shape[0] * shape[1]

    class _Holder:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                    "strides": None}

    flat = torch.as_tensor(_Holder(), device="cuda")
    return flat.view(shape[1], shape[0]).t()


@pytest.fixture(scope="module")
def L():
    from paper_2403_12340_b200 import lrgw

    return lrgw


def test_si8_build_matches_reference(L, ctx, ref):
    import torch

    from paper_2403_12340_b200 import synth

    cfg = synth.CONFIGS["si8"]
    psi = synth.orbitals_host(cfg)
    e = synth.energies(cfg)
    a, b = psi[:, :16], psi[:, 16:]
    dpsi = _cm(torch.from_numpy(np.ascontiguousarray(psi.T)).t().cuda())
    ep = L.build(dpsi[:, :16], dpsi[:, 16:], e, cfg.dims, cfg.cell3, k_mu=cfg.k_mu, n_lambda=cfg.n_lambda, ctx=ctx)
    pts_ref = ref.select_points(a, b, 128)
    assert np.array_equal(ep.point_indices, pts_ref)
    th_ref = ref.fit(a, b, pts_ref)
    assert rel(ep.p_vc, th_ref) <= TOL
    s7 = ref.elliptic_params(e, 16, 16)
    h = 2 * s7[3] / cfg.n_lambda
    nodes = [-s7[3] + i * h for i in range(cfg.n_lambda + 1)]
    w = [0.5 * h if i in (0, cfg.n_lambda) else h for i in range(cfg.n_lambda + 1)]
    acc = 2 * np.sqrt(s7[0] * s7[1]) / (np.pi * s7[2]) * ref.sum_node_terms(a[pts_ref], b[pts_ref], e, s7, nodes, w)
    t_ref = 0.5 * (acc + acc.T)
    assert rel(ep.t, t_ref) <= TOL
    x = synth.probe_host(cfg.n_r)
    y_ref, k_ref, _ = ref.build_and_apply(t_ref, th_ref, cfg.dims, cfg.cell3, x, threads=8)
    assert rel(ep.k, k_ref) <= TOL
    assert rel(L.epsilon_inverse_apply(ep, x), y_ref) <= TOL
    st = ctx.stage_ms()
    assert st["total"] > 0 and st["select"] > 0


def test_si64_build_properties_and_pivots(L, ctx):
    import torch

    from oracle import restate as R
    from paper_2403_12340_b200 import synth

    cfg = synth.CONFIGS["si64"]
    psi = synth.orbitals_device(cfg)
    e = synth.energies(cfg)
    ep = L.build(psi[:, :128], psi[:, 128:], e, cfg.dims, cfg.cell3, k_mu=cfg.k_mu, n_lambda=cfg.n_lambda,
                 ctx=ctx)
    assert ep.n_mu == 1024
    pts = ep.point_indices
    assert np.all(np.diff(pts) > 0)
    # bit-exact pivots against the oracle restatement (oracle/select.c)
    hpsi = psi.cpu().numpy()
    pts_or, diag = R.select_points(hpsi[:, :128], hpsi[:, 128:], 1024, return_diag=True)
    assert np.array_equal(pts, pts_or)
    assert diag["recompute_events"] == 0
    k = torch.from_numpy(ep.k)
    assert float(torch.linalg.norm(k - k.T) / torch.linalg.norm(k)) <= 1e-12
    assert float(torch.linalg.eigvalsh(k).max()) < 0
    t = torch.from_numpy(ep.t)
    assert float(torch.linalg.eigvalsh(t).max()) < 0
    x = _cm(torch.randn(cfg.n_r, 8, dtype=torch.float64, device="cuda",
                        generator=torch.Generator(device="cuda").manual_seed(7)))
    assert _eps_residual(L, ctx, ep, cfg, x) <= 1e-9


def test_si512_build_on_one_gpu(L, ctx):
    """The Si512 scaling workload (N_r 884 736, N_v = N_c = 1024, N_mu 8192,
    Theta 58 GB) built on ONE B200: the oracle's first 64 greedy pivots
    bit-exact (the greedy is prefix-consistent, so these are the build's
    first 64 steps; oracle/select.c on the host), K and T symmetric negative
    definite, and the matrix-free SMW residual ||eps eps^-1 x - x|| <= 1e-9."""
    import ctypes

    import torch

    from oracle import restate as R
    from paper_2403_12340_b200 import synth

    cfg = synth.CONFIGS["si512"]
    psi = synth.orbitals_device(cfg)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    e = synth.energies(cfg)
    n = cfg.n_v
    # first 64 pivots: device selection vs the oracle restatement
    pts64 = np.zeros(64, dtype=np.int32)
    lib = L.L.load()
    margin = ctypes.c_double(0.0)
    rc = lib.lrgw_dev_select(ctx.handle, ctypes.c_void_p(psi.data_ptr()), cfg.n_r, n,
                             ctypes.c_void_p(psi[:, n:].data_ptr()), cfg.n_r, cfg.n_c, cfg.n_r, 64,
                             pts64.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), ctypes.byref(margin))
    assert rc == 0
    hpsi = psi.cpu().numpy()
    assert np.array_equal(pts64, R.select_points(hpsi[:, :n], hpsi[:, n:], 64))
    del hpsi
    ep = L.build(psi[:, :n], psi[:, n:], e, cfg.dims, cfg.cell3, k_mu=cfg.k_mu, n_lambda=cfg.n_lambda, ctx=ctx)
    assert ep.n_mu == 8192
    pts = ep.point_indices
    assert np.all(np.diff(pts) > 0) and set(pts64.tolist()) <= set(pts.tolist())
    th_p, k_p, t_p = ep.device_ptrs()
    k = L_tensor(k_p, (ep.n_mu, ep.n_mu))
    t = L_tensor(t_p, (ep.n_mu, ep.n_mu))
    assert float(torch.linalg.norm(k - k.T)) == 0.0
    assert float(torch.linalg.eigvalsh(k).max()) < 0
    assert float(torch.linalg.eigvalsh(t).max()) < 0
    x = _cm(torch.randn(cfg.n_r, 8, dtype=torch.float64, device="cuda",
                        generator=torch.Generator(device="cuda").manual_seed(7)))
    assert _eps_residual(L, ctx, ep, cfg, x) <= 1e-9
    ep.close()
    del psi
    torch.cuda.empty_cache()


def test_handles_survive_their_context(L):
    """A factored-inverse handle destroyed after its context (garbage
    collection order) is orphaned, not a use-after-free."""
    rng = np.random.default_rng(0)
    p = np.linalg.qr(rng.standard_normal((64, 6)))[0]
    c2 = L.Context(0)
    eps = L.build_epsilon_inverse(-np.eye(6) * 1e-3, p, (4, 4, 4), (6.0, 6.0, 6.0), ctx=c2)
    c2.close()
    eps.close()
    c3 = L.Context(0)
    eps = L.build_epsilon_inverse(-np.eye(6) * 1e-3, p, (4, 4, 4), (6.0, 6.0, 6.0), ctx=c3)
    c3.close()
    with pytest.raises(L.InvalidInput):
        L.epsilon_inverse_apply(eps, np.zeros((64, 1)))
