"""GPU: the whole device-resident build (lrgw_build, stages 1-5) against the
reference at Si8 (BASELINE configs[0]); the larger configs are in
tests/test_gpu_configs.py."""
import numpy as np
import pytest

from helpers import rel

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _cm(t):
    return t.t().contiguous().t()


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


def test_build_fused_fit_rejected_then_context_reusable(L, ctx):
    """A pair set of rank 10 < N_mu = 12 (psi_c = psi_v: f g = g f) makes the
    selection's last pivots numerically zero, so L_P fails the LU rule the
    fused fit checks on the device (read back with the SMW status): the build
    falls back to the explicit fit (pinv, isdf.hpp:143-160) and T at the
    points is singular — the error the reference raises (smw.hpp:49-53). The
    context must stay usable: the next build equals one on a fresh context."""
    import torch

    rng = np.random.default_rng(7)
    n_r = 512
    f = np.linalg.qr(rng.standard_normal((n_r, 4)))[0]
    psi = np.concatenate([f, f], axis=1)
    e = np.array([-0.5, -0.4, -0.3, -0.1, 0.05, 0.2, 0.4, 0.8])
    d = torch.from_numpy(np.asfortranarray(psi)).cuda().t().contiguous().t()
    with pytest.raises(L.NumericError):
        L.build(d[:, :4], d[:, 4:], e, (8, 8, 8), (6.0, 6.0, 6.0), k_mu=3.0, n_lambda=16, ctx=ctx)
    psi2 = np.linalg.qr(rng.standard_normal((n_r, 32)))[0]
    e2 = np.concatenate([np.sort(rng.uniform(-0.5, -0.1, 16)), np.sort(rng.uniform(0.05, 0.8, 16))])
    d2 = torch.from_numpy(np.asfortranarray(psi2)).cuda().t().contiguous().t()
    ep = L.build(d2[:, :16], d2[:, 16:], e2, (8, 8, 8), (6.0, 6.0, 6.0), k_mu=8.0, n_lambda=16, ctx=ctx)
    fresh = L.Context(0)
    ep2 = L.build(d2[:, :16], d2[:, 16:], e2, (8, 8, 8), (6.0, 6.0, 6.0), k_mu=8.0, n_lambda=16, ctx=fresh)
    assert np.array_equal(ep.point_indices, ep2.point_indices)
    assert np.array_equal(ep.k, ep2.k) and np.array_equal(ep.p_vc, ep2.p_vc)
    assert ep.info()["fit_path"] == 0
    ep.close()
    ep2.close()
    fresh.close()


@pytest.mark.parametrize("name,reps", [("si8", 6), ("si64", 4)])
def test_repeated_builds_are_bit_identical(L, ctx, name, reps):
    """Every reduction of the build has a fixed order (segment partials,
    split-K slots, per-band column sums), so repeated builds of the same
    inputs must agree bit for bit in the points, Theta, T and K. A mismatch
    is a staging race in a ring engine (the class found in the TMA K3 kernel:
    a slot released right behind its own shared-memory loads;
    gemm4.cuh:release_prev, tools/stress_build.py runs the long version)."""
    import torch

    from paper_2403_12340_b200 import synth

    cfg = synth.CONFIGS[name]
    psi = synth.orbitals_device(cfg)
    e = synth.energies(cfg)
    first = None
    for _ in range(reps):
        ep = L.build(psi[:, :cfg.n_v], psi[:, cfg.n_v:], e, cfg.dims, cfg.cell3, k_mu=cfg.k_mu,
                     n_lambda=cfg.n_lambda, ctx=ctx)
        th_p, k_p, t_p = ep.device_ptrs()
        cur = (np.array(ep.point_indices), L_tensor(th_p, (cfg.n_r, ep.n_mu)).clone(),
               L_tensor(t_p, (ep.n_mu, ep.n_mu)).clone(), L_tensor(k_p, (ep.n_mu, ep.n_mu)).clone())
        ep.close()
        if first is None:
            first = cur
            continue
        assert np.array_equal(cur[0], first[0])
        for got, want in zip(cur[1:], first[1:]):
            assert torch.equal(got, want)
