"""GPU: value parity of the whole device build (lrgw_build, stages 1-5) with
the reference at EVERY BASELINE.json config (north_star: bit-exact ISDF points;
Theta, T, the SMW core K and eps^-1 applied to the fixed probe within relative
Frobenius 1e-10).

The checkers are the compiled reference (oracle/_ref/libref_lrgw.so) through
its own functions, restricted to the rows / columns under test where the full
call is out of reach on the host (every restriction is separable, so the
restricted outputs are bit-identical to the full call's —
tests/test_oracle.py::test_stagewise_checkers_equal_full_reference_calls):

  Si64   the full reference chain on the reference's own intermediates:
         fit_auxiliary_basis (all rows), sum_node_terms (all 25 nodes),
         assemble_K (sym_eig check, lu_solve, P^T V P through apply_coulomb +
         matmul_tn, lu_invert), epsilon_inverse_apply with V P
         (isdf.hpp:118-163, contour.hpp:185-222, smw.hpp:42-103)
  C60,   pivots: the full greedy sequence from oracle/select.c (cached in
  Si216  tests/golden/pivots_<cfg>.npz, keyed by the SHA-256 of the orbitals,
         made by tools/make_pivot_fixtures.py; recomputed live on a mismatch);
         Theta on 4096 sampled grid rows; T on all (C60) or a third of the
         points (Si216); P^T V P on 16 sampled columns; K by the reference SMW
         algebra on the build's T and P^T V P; eps^-1 X as X + V (P (K P^T X))
  Si512  the first 256 greedy pivots (oracle/select.c); Theta on 2048 sampled
         rows (restatement: the reference's serial LU at N_mu = 8192 takes
         hours); T on 512 sampled points (reference); K, T negative definite
         and the matrix-free SMW residual <= 1e-9

Every config also asserts the smallest relative top-2 pivot margin of the
build's greedy (lrgw_eps_info.min_margin) exceeds 1e-12 — the early warning
for a pivot flip at scale (linalg.hpp:45-53 tie rule).
Set LRGW_PARITY_OUT=<dir> to write each config's report as JSON.
"""
import hashlib
import json
import os
import time

import numpy as np
import pytest

from helpers import rel

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
TOL = 1e-10
MARGIN_FLOOR = 1e-12
THREADS = max(1, os.cpu_count() or 1)
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _cm(t):
    return t.t().contiguous().t()


def _dev_view(ptr, shape):
    """Zero-copy column-major torch view of a device buffer owned by a handle."""
    import torch

    n = shape[0] * shape[1]

    class _Holder:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                    "strides": None}

    return torch.as_tensor(_Holder(), device="cuda").view(shape[1], shape[0]).t()


def psi_sha256(h) -> str:
    """SHA-256 of the orbital block's bytes in column-major order."""
    return hashlib.sha256(np.asfortranarray(h).T.data).hexdigest()


def oracle_pivots(cfg, h, n_mu):
    """(sorted points, per-step margins, source) from oracle/select.c, via the
    hash-keyed fixture when the orbitals match it."""
    from oracle import restate as R

    path = os.path.join(GOLDEN, f"pivots_{cfg.name}.npz")
    sha = psi_sha256(h)
    if os.path.exists(path):
        z = np.load(path)
        if str(z["sha256"]) == sha and int(z["n_mu"]) == n_mu:
            return z["pts"], z["margins"], "fixture"
    pts, diag = R.select_points(h[:, :cfg.n_v], h[:, cfg.n_v:], n_mu, return_diag=True)
    assert diag["recompute_events"] == 0
    return pts, diag["margins"], "live select.c"


def _report(name, rep):
    out = os.environ.get("LRGW_PARITY_OUT")
    print(f"\n[parity {name}] " + json.dumps(rep, sort_keys=True))
    if out:
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, f"parity_{name}.json"), "w") as f:
            json.dump(rep, f, indent=1, sort_keys=True)


def _nodes(ref, e, cfg):
    s7 = ref.elliptic_params(e, cfg.n_v, cfg.n_c)
    h = 2 * s7[3] / cfg.n_lambda
    nodes = [-s7[3] + i * h for i in range(cfg.n_lambda + 1)]
    w = [0.5 * h if i in (0, cfg.n_lambda) else h for i in range(cfg.n_lambda + 1)]
    pref = 2 * np.sqrt(s7[0] * s7[1]) / (np.pi * s7[2])
    return s7, nodes, w, pref


def _ref_t(ref, pv, pc, e, cfg):
    s7, nodes, w, pref = _nodes(ref, e, cfg)
    acc = pref * ref.sum_node_terms(pv, pc, e, s7, nodes, w, threads=THREADS)
    return 0.5 * (acc + acc.T)


def _build(cfg, ctx):
    from paper_2403_12340_b200 import lrgw, synth

    psi = synth.orbitals_device(cfg)
    e = synth.energies(cfg)
    t0 = time.time()
    ep = lrgw.build(psi[:, :cfg.n_v], psi[:, cfg.n_v:], e, cfg.dims, cfg.cell3, k_mu=cfg.k_mu,
                    n_lambda=cfg.n_lambda, ctx=ctx)
    return psi, e, ep, time.time() - t0


def _timed(rep, key, fn):
    t0 = time.time()
    out = fn()
    rep.setdefault("ref_seconds", {})[key] = round(time.time() - t0, 2)
    return out


def _margin_checks(rep, ep, or_margins):
    inf = ep.info()
    rep["min_margin_build"] = inf["min_margin"]
    rep["min_margin_step"] = inf["min_margin_step"]
    rep["min_margin_oracle"] = float(np.min(or_margins)) if len(or_margins) else None
    rep["fit_path"] = "fused L L_P^-1" if inf["fit_path"] == 0 else "explicit Gram LU"
    rep["gram_cond_lower_bound"] = inf["lp_diag_ratio"]
    rep["select_blocks"] = inf["select_blocks"]
    assert inf["min_margin"] > MARGIN_FLOOR, rep
    return inf


def test_si64_full_reference_chain(ctx, ref):
    """Si64 (BASELINE configs[1]): every output against the reference's full
    chain on its own intermediates."""
    from paper_2403_12340_b200 import lrgw, synth

    cfg = synth.CONFIGS["si64"]
    psi, e, ep, tb = _build(cfg, ctx)
    h = psi.cpu().numpy()
    a, b = h[:, :cfg.n_v], h[:, cfg.n_v:]
    rep = {"config": cfg.name, "n_mu": ep.n_mu, "threads": THREADS, "build_s": round(tb, 3)}
    pts_or, margins, src = _timed(rep, "select_oracle", lambda: oracle_pivots(cfg, h, ep.n_mu))
    pts = ep.point_indices
    rep["pivot_source"] = src
    rep["pivots_bit_exact"] = bool(np.array_equal(pts, pts_or))
    assert rep["pivots_bit_exact"]
    inf = _margin_checks(rep, ep, margins)
    th_ref, pinv = _timed(rep, "fit", lambda: ref.fit_rows(a, b, a[pts], b[pts], threads=THREADS))
    assert not pinv
    t_ref = _timed(rep, "contour", lambda: _ref_t(ref, a[pts], b[pts], e, cfg))
    pvp_ref, vp_ref = _timed(rep, "pvp", lambda: ref.pvp_cols(th_ref, cfg.dims, cfg.cell3, np.arange(ep.n_mu),
                                                               threads=THREADS, want_vp=True))
    k_ref = _timed(rep, "smw", lambda: ref.smw_from_pvp(t_ref, pvp_ref, check_eig=True, threads=THREADS))
    x = synth.probe_host(cfg.n_r)
    y_ref = _timed(rep, "apply", lambda: ref.eps_apply_vp(th_ref, k_ref, vp_ref, x))
    pvp_gpu = _dev_view(inf["pvp"], (ep.n_mu, ep.n_mu)).cpu().numpy()
    rep["rel"] = {
        "theta": rel(ep.p_vc, th_ref),
        "t": rel(ep.t, t_ref),
        "pvp": rel(pvp_gpu, 0.5 * (pvp_ref + pvp_ref.T)),
        "k": rel(ep.k, k_ref),
        "eps_inv_x": rel(lrgw.epsilon_inverse_apply(ep, x), y_ref),
    }
    _report(cfg.name, rep)
    assert all(v <= TOL for v in rep["rel"].values()), rep
    ep.close()


@pytest.mark.parametrize("name", ["c60", "si216"])
def test_large_config_stagewise(ctx, ref, name):
    """C60 and Si216 (BASELINE configs[2], [3]): full pivot sequence, then each
    stage's output against the reference applied to the checked inputs of
    that stage."""
    import torch

    from paper_2403_12340_b200 import lrgw, synth

    cfg = synth.CONFIGS[name]
    psi, e, ep, tb = _build(cfg, ctx)
    h = psi.cpu().numpy()
    del psi
    a, b = h[:, :cfg.n_v], h[:, cfg.n_v:]
    rep = {"config": cfg.name, "n_mu": ep.n_mu, "threads": THREADS, "build_s": round(tb, 3)}
    pts = ep.point_indices
    pts_or, margins, src = _timed(rep, "select_oracle", lambda: oracle_pivots(cfg, h, ep.n_mu))
    rep["pivot_source"] = src
    rep["pivots_bit_exact"] = bool(np.array_equal(pts, pts_or))
    assert rep["pivots_bit_exact"]
    inf = _margin_checks(rep, ep, margins)
    rng = np.random.default_rng(11)
    n_mu = ep.n_mu
    # Theta on sampled grid rows (fit_auxiliary_basis is row-separable)
    rows = np.sort(rng.choice(cfg.n_r, 4096, replace=False))
    th_dev = _dev_view(inf["theta"], (cfg.n_r, n_mu))
    th_rows = th_dev[torch.as_tensor(rows, device="cuda")].cpu().numpy()
    th_ref_rows, pinv = _timed(rep, "fit_rows", lambda: ref.fit_rows(a[rows], b[rows], a[pts], b[pts],
                                                                     threads=THREADS))
    rep["fit_pinv_fallback_in_reference"] = pinv
    # T on all points (C60) or a third of them (Si216: T(mu, nu) needs rows mu, nu only)
    t_gpu = ep.t
    sub = np.arange(n_mu) if n_mu <= 1024 else np.sort(rng.choice(n_mu, n_mu // 3, replace=False))
    t_ref_sub = _timed(rep, "contour", lambda: _ref_t(ref, a[pts[sub]], b[pts[sub]], e, cfg))
    # P^T V P on sampled columns, from the build's Theta
    theta = ep.p_vc
    cols = np.sort(rng.choice(n_mu, 16, replace=False))
    pvp_ref_cols = _timed(rep, "pvp_cols", lambda: ref.pvp_cols(theta, cfg.dims, cfg.cell3, cols, threads=THREADS))
    pvp_gpu = _dev_view(inf["pvp"], (n_mu, n_mu)).cpu().numpy()
    # K by the reference SMW algebra on the build's T and P^T V P
    k_ref = _timed(rep, "smw", lambda: ref.smw_from_pvp(t_gpu, pvp_gpu, check_eig=(n_mu <= 1024),
                                                         threads=THREADS))
    x = synth.probe_host(cfg.n_r)
    k_gpu = ep.k
    y_ref = _timed(rep, "apply", lambda: ref.eps_apply_factored(theta, k_gpu, cfg.dims, cfg.cell3, x,
                                                                threads=THREADS))
    del theta
    rep["rel"] = {
        "theta_rows": rel(th_rows, th_ref_rows),
        "t": rel(t_gpu[np.ix_(sub, sub)], t_ref_sub),
        "pvp_cols": rel(pvp_gpu[:, cols], pvp_ref_cols),
        "k": rel(k_gpu, k_ref),
        "eps_inv_x": rel(lrgw.epsilon_inverse_apply(ep, x), y_ref),
    }
    rep["samples"] = {"theta_rows": int(rows.size), "t_points": int(sub.size), "pvp_cols": int(cols.size)}
    _report(cfg.name, rep)
    assert all(v <= TOL for v in rep["rel"].values()), rep
    ep.close()
    torch.cuda.empty_cache()


def test_si512_samples_on_one_gpu(ctx, ref):
    """Si512 (BASELINE configs[4], N_mu 8192, Theta 58 GB on one B200): the
    first 256 greedy pivots bit-exact, Theta rows and T entries on samples,
    K / T negative definite, the matrix-free SMW residual <= 1e-9."""
    import ctypes

    import torch

    from oracle import restate as R
    from paper_2403_12340_b200 import lrgw, synth

    cfg = synth.CONFIGS["si512"]
    psi = synth.orbitals_device(cfg)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    e = synth.energies(cfg)
    n = cfg.n_v
    rep = {"config": cfg.name, "threads": THREADS}
    npre = 256
    pre = np.zeros(npre, dtype=np.int32)
    lib = lrgw.L.load()
    margin = ctypes.c_double(0.0)
    assert lib.lrgw_dev_select(ctx.handle, ctypes.c_void_p(psi.data_ptr()), cfg.n_r, n,
                               ctypes.c_void_p(psi[:, n:].data_ptr()), cfg.n_r, cfg.n_c, cfg.n_r, npre,
                               pre.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), ctypes.byref(margin)) == 0
    h = psi.cpu().numpy()
    pre_or = _timed(rep, "select_oracle_prefix", lambda: R.select_points(h[:, :n], h[:, n:], npre))
    rep["prefix_pivots_bit_exact"] = bool(np.array_equal(pre, pre_or))
    assert rep["prefix_pivots_bit_exact"]
    t0 = time.time()
    ep = lrgw.build(psi[:, :n], psi[:, n:], e, cfg.dims, cfg.cell3, k_mu=cfg.k_mu, n_lambda=cfg.n_lambda, ctx=ctx)
    rep["build_s"] = round(time.time() - t0, 3)
    assert ep.n_mu == 8192
    pts = ep.point_indices
    assert np.all(np.diff(pts) > 0) and set(pre.tolist()) <= set(pts.tolist())
    inf = _margin_checks(rep, ep, [])
    rng = np.random.default_rng(12)
    rows = np.sort(rng.choice(cfg.n_r, 2048, replace=False))
    th = _dev_view(inf["theta"], (cfg.n_r, ep.n_mu))
    th_rows = th[torch.as_tensor(rows, device="cuda")].cpu().numpy()
    a, b = h[:, :n], h[:, n:]
    th_or = _timed(rep, "fit_rows_restatement", lambda: R.fit_rows(a[rows], b[rows], a[pts], b[pts]))
    sub = np.sort(rng.choice(ep.n_mu, 512, replace=False))
    tm = _dev_view(inf["t"], (ep.n_mu, ep.n_mu))
    t_sub = tm[torch.as_tensor(sub, device="cuda")][:, torch.as_tensor(sub, device="cuda")].cpu().numpy()
    t_ref = _timed(rep, "contour", lambda: _ref_t(ref, a[pts[sub]], b[pts[sub]], e, cfg))
    rep["rel"] = {"theta_rows": rel(th_rows, th_or), "t": rel(t_sub, t_ref)}
    del h, a, b
    k = _dev_view(inf["k"], (ep.n_mu, ep.n_mu))
    assert float(torch.linalg.norm(k - k.T)) == 0.0
    assert float(torch.linalg.eigvalsh(k).max()) < 0
    assert float(torch.linalg.eigvalsh(tm).max()) < 0
    x = _cm(torch.randn(cfg.n_r, 8, dtype=torch.float64, device="cuda",
                        generator=torch.Generator(device="cuda").manual_seed(7)))
    rep["smw_residual"] = _eps_residual(ctx, ep, cfg, x, inf)
    _report(cfg.name, rep)
    assert rep["smw_residual"] <= 1e-9
    assert all(v <= TOL for v in rep["rel"].values()), rep
    ep.close()
    del psi
    torch.cuda.empty_cache()


def _eps_residual(ctx, ep, cfg, x, inf):
    """||eps (eps^-1 x) - x|| / ||x|| with eps = I - V (2 Theta T Theta^T)
    applied matrix-free on the device (smw.hpp:116-169 definition)."""
    import torch

    from paper_2403_12340_b200 import lrgw

    theta = _dev_view(inf["theta"], (ep.n_r, ep.n_mu))
    tmat = _dev_view(inf["t"], (ep.n_mu, ep.n_mu))
    y = torch.empty_like(x)
    lrgw.eps_apply_dev(ep, x, y)
    u = _cm(torch.empty(ep.n_mu, x.shape[1], dtype=torch.float64, device="cuda"))
    lrgw.dgemm_dev("T", "N", 1.0, theta, y, 0.0, u, ctx=ctx)
    w = _cm(torch.empty_like(u))
    lrgw.dgemm_dev("N", "N", 2.0, tmat, u, 0.0, w, ctx=ctx)
    z = _cm(torch.empty_like(x))
    lrgw.dgemm_dev("N", "N", 1.0, theta, w, 0.0, z, ctx=ctx)
    vz = _cm(torch.empty_like(x))
    lrgw.coulomb_apply_dev(cfg.dims, cfg.cell3, z, vz, ctx=ctx)
    r = y - vz - x
    return float(torch.linalg.norm(r) / torch.linalg.norm(x))
