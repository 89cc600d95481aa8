"""GPU: the implicit-Theta build (lrgw_ctx_set_theta_implicit) — Theta kept
factored as L L_P^-1 during lrgw_build, eps^-1 applied from (L, K'), Theta /
K / T / Theta^T V Theta formed on first demand — against the reference at Si8
and against the ordinary build at Si64."""
import numpy as np
import pytest

from helpers import rel

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _cm(t):
    return t.t().contiguous().t()


def test_si8_implicit_build_matches_reference(ref):
    import torch

    from paper_2403_12340_b200 import lrgw, synth

    cfg = synth.CONFIGS["si8"]
    psi = synth.orbitals_host(cfg)
    e = synth.energies(cfg)
    a, b = psi[:, :16], psi[:, 16:]
    dpsi = _cm(torch.from_numpy(np.ascontiguousarray(psi.T)).t().cuda())
    ctx = lrgw.Context(0)
    ctx.set_theta_implicit(True)
    ep = lrgw.build(dpsi[:, :16], dpsi[:, 16:], e, cfg.dims, cfg.cell3, k_mu=cfg.k_mu, n_lambda=cfg.n_lambda,
                    ctx=ctx)
    assert ctx.stage_ms()["fit_gemm"] < 0.05  # the fit GEMM left the build (an empty stage)
    pts_ref = ref.select_points(a, b, 128)
    assert np.array_equal(ep.point_indices, pts_ref)
    # the apply first: it runs on the factored (L, K') handle
    x = synth.probe_host(cfg.n_r)
    y = lrgw.epsilon_inverse_apply(ep, x)
    th_ref = ref.fit(a, b, pts_ref)
    s7 = ref.elliptic_params(e, 16, 16)
    h = 2 * s7[3] / cfg.n_lambda
    nodes = [-s7[3] + i * h for i in range(cfg.n_lambda + 1)]
    w = [0.5 * h if i in (0, cfg.n_lambda) else h for i in range(cfg.n_lambda + 1)]
    acc = 2 * np.sqrt(s7[0] * s7[1]) / (np.pi * s7[2]) * ref.sum_node_terms(a[pts_ref], b[pts_ref], e, s7, nodes, w)
    t_ref = 0.5 * (acc + acc.T)
    y_ref, k_ref, _ = ref.build_and_apply(t_ref, th_ref, cfg.dims, cfg.cell3, x, threads=8)
    assert rel(y, y_ref) <= TOL
    # then the explicit factors on demand
    assert rel(ep.p_vc, th_ref) <= TOL
    assert rel(ep.t, t_ref) <= TOL
    assert rel(ep.k, k_ref) <= TOL
    assert rel(lrgw.epsilon_inverse_apply(ep, x), y_ref) <= TOL


def test_si64_implicit_equals_explicit():
    from paper_2403_12340_b200 import lrgw, synth

    cfg = synth.CONFIGS["si64"]
    psi = synth.orbitals_device(cfg)
    e = synth.energies(cfg)
    x = synth.probe_host(cfg.n_r)
    out = {}
    for implicit in (False, True):
        ctx = lrgw.Context(0)
        ctx.set_theta_implicit(implicit)
        ep = lrgw.build(psi[:, :cfg.n_v], psi[:, cfg.n_v:], e, cfg.dims, cfg.cell3, k_mu=cfg.k_mu,
                        n_lambda=cfg.n_lambda, ctx=ctx)
        y = lrgw.epsilon_inverse_apply(ep, x)
        out[implicit] = (ep.point_indices.copy(), y, ep.k, ep.t, ep.p_vc[::97].copy())
        ep.close()
        ctx.close()
    (p0, y0, k0, t0, th0), (p1, y1, k1, t1, th1) = out[False], out[True]
    assert np.array_equal(p0, p1)
    assert rel(y1, y0) <= 1e-12
    assert rel(k1, k0) <= 1e-11
    assert rel(t1, t0) <= 1e-14
    assert rel(th1, th0) <= 1e-13
