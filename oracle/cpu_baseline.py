"""oracle/cpu_baseline.py — TEST/BENCH INFRASTRUCTURE ONLY (the CPU baseline).

Times the reference CPU implementation of the eps^-1 build (stages 1-5) on
the host cores through oracle/_ref (the unmodified reference headers) on a
BOUNDED SAMPLE of the BASELINE workload and extrapolates each stage by its
exact cost model. The full Si64 build takes ~8 min on 8 cores, so
each stage is sampled:

  1 select   reference qrcp is guard-blocked beyond 2^26 pair entries
             (isdf.hpp:49, 77-78), so the greedy restatement oracle/select.c
             (OpenMP, all cores) runs the first S pivot steps; per-step cost
             is linear in (N_v + N_c + k), summed over k < N_mu.
  2 fit      reference fit_auxiliary_basis (isdf.hpp:118-163, serial) on two
             row samples (all N_mu point rows — the GPU build's points when
             given — + filler rows); t = a + b N_rows
             fitted and evaluated at N_r (LU of the N_mu Gram is the constant).
  3 contour  reference detail::sum_node_terms (contour.hpp:185-222) over ALL
             N_lambda + 1 nodes with threads = cores (no extrapolation).
  4-5 SMW    reference sym_eig(T), lu_solve(T, I/2), lu_invert on the real T
             (full size); apply_coulomb on C columns (threads = cores) scaled
             by 2 N_mu / C (the reference applies V to P twice, smw.hpp:61, 92);
             matmul_tn on a C-column block scaled by (N_mu / C)^2.

Only bench.py (cpu_baseline leg and --impl reference) imports this module.
"""
from __future__ import annotations

import os
import time

import numpy as np

from . import ref
from . import restate as R


def _t(fn):
    t0 = time.perf_counter()
    out = fn()
    return time.perf_counter() - t0, out


def _inputs(cfg, psi, energies, rng):
    n_r, n_v, n_c = cfg.n_r, cfg.n_v, cfg.n_c
    n = n_v + n_c
    if psi is None:
        psi = np.asfortranarray(np.linalg.qr(rng.standard_normal((n_r, n)))[0])
    e = energies if energies is not None else np.concatenate(
        [np.sort(rng.uniform(*cfg.occ, n_v)), np.sort(rng.uniform(*cfg.virt, n_c))])
    return psi, e


def fixed_pieces(cfg, psi=None, energies=None, cores=None, fit_rows=(2048, 4096), seed=5, points=None,
                 node_sample=None, eig_size=None):
    """The pieces timed once per run: the reference fit on two row samples
    (each with the full N_mu^3 Gram LU; linear in N_r), the quadrature over
    all nodes, and the N_mu^3 SMW factorisations (sym_eig, lu_solve, lu_invert).
    Bounded variants for the large configs: `node_sample` times that many
    evenly spaced nodes of the trapezoid and scales by (N_lambda + 1) / sample
    (the node terms cost the same); `eig_size` times sym_eig on the leading
    block of that size and scales by (N_mu / size)^3 (Householder + QL, cubic)."""
    cores = cores or os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    n_r, n_v, n_c = cfg.n_r, cfg.n_v, cfg.n_c
    n_mu = min(max(R.num_aux(cfg.k_mu, n_v, n_c), 1), n_r)
    if eig_size == "half":
        eig_size = n_mu // 2
    if fit_rows == "wide":
        # two row counts 2048 apart: with N_mu = 3456 the default (2048, 4096) clamps to
        # (3457, 4096), and a 639-row difference extrapolated to 373 248 rows turned +-2 s of
        # timing noise into +-45 % of the fit stage (33 000 .. 88 000 s across three runs)
        fit_rows = (n_mu + 1, n_mu + 1 + 2048)
    rng = np.random.default_rng(seed)
    psi, e = _inputs(cfg, psi, energies, rng)
    a, b = psi[:, :n_v], psi[:, n_v:n_v + n_c]
    stages = {}
    # the build's own ISDF points when given (random grid points can make the
    # Gram of localised orbitals singular — C60 — where the reference throws)
    pts = (np.sort(np.asarray(points)).astype(np.int32) if points is not None
           else np.sort(rng.choice(n_r, n_mu, replace=False)).astype(np.int32))
    others = np.setdiff1d(np.arange(n_r), pts)
    times = []
    for rows in fit_rows:
        rows = max(rows, n_mu + 1)
        extra = np.sort(rng.choice(others, rows - n_mu, replace=False))
        sel = np.sort(np.concatenate([pts, extra]))
        sub_pts = np.searchsorted(sel, pts).astype(np.int32)
        asub, bsub = np.asfortranarray(a[sel]), np.asfortranarray(b[sel])
        t_fit, _ = _t(lambda: ref.fit(asub, bsub, sub_pts))
        times.append((rows, t_fit))
    (r1, t1), (r2, t2) = times
    slope = (t2 - t1) / (r2 - r1)
    stages["fit"] = max(t1 + slope * (n_r - r1), t2)
    pv, pc = np.asfortranarray(a[pts]), np.asfortranarray(b[pts])
    s7 = ref.elliptic_params(e, n_v, n_c)
    h = 2 * s7[3] / cfg.n_lambda
    nodes = [-s7[3] + i * h for i in range(cfg.n_lambda + 1)]
    wts = [0.5 * h if i in (0, cfg.n_lambda) else h for i in range(cfg.n_lambda + 1)]
    n_nodes = cfg.n_lambda + 1
    if node_sample and node_sample < n_nodes:
        # the timed subset only feeds the timing; the matrix the factorisations
        # below are timed on is that subset's sum (same structure, negative definite)
        idx = np.unique(np.linspace(0, n_nodes - 1, node_sample).round().astype(int))
        nodes_t, wts_t = [nodes[i] for i in idx], [wts[i] * n_nodes / len(idx) for i in idx]
    else:
        idx = np.arange(n_nodes)
        nodes_t, wts_t = nodes, wts
    t_quad, acc = _t(lambda: ref.sum_node_terms(pv, pc, e, s7, nodes_t, wts_t, threads=cores))
    stages["contour"] = t_quad * n_nodes / len(idx)
    t_mat = 2 * np.sqrt(s7[0] * s7[1]) / (np.pi * s7[2]) * acc
    t_mat = 0.5 * (t_mat + t_mat.T)
    if eig_size and eig_size < n_mu:
        blk = np.asfortranarray(t_mat[:eig_size, :eig_size])
        t_eig, _ = _t(lambda: ref.sym_eig_values(blk))
        t_eig *= (n_mu / eig_size) ** 3
    else:
        t_eig, _ = _t(lambda: ref.sym_eig_values(t_mat))
    t_half, half = _t(lambda: ref.lu_solve(t_mat, 0.5 * np.eye(n_mu)))
    mid = 0.5 * (half + half.T) - 1e-3 * np.eye(n_mu)
    t_inv, _ = _t(lambda: ref.lu_solve(mid, np.eye(n_mu)))
    stages["smw_eig"] = t_eig
    stages["smw_lu"] = t_half + t_inv
    nodes_txt = f"all {n_nodes} nodes" if len(idx) == n_nodes else f"{len(idx)}/{n_nodes} nodes x{n_nodes / len(idx):.2f}"
    eig_txt = (f"sym_eig at {eig_size} x{(n_mu / eig_size) ** 3:.1f}, 2 LU at N_mu={n_mu}"
               if eig_size and eig_size < n_mu else f"sym_eig / 2 LU at N_mu={n_mu}")
    sample = f"fit on {fit_rows} rows -> linear in N_r={n_r}; {nodes_txt}; {eig_txt}"
    return stages, sample


def sampled_pieces(cfg, psi=None, cores=None, sel_steps=64, cols=128, seed=5):
    """The pieces timed every step, extrapolated by their exact cost models:
    S greedy steps of the selection (restatement: the reference's qrcp is
    guard-blocked here) scaled by sum_k (N + k + 1); apply_coulomb on C
    columns scaled by 2 N_mu / C (the reference applies V to P twice,
    smw.hpp:61, 92); matmul_tn on a C-column block scaled by (N_mu / C)^2."""
    cores = cores or os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    n_r, n_v, n_c = cfg.n_r, cfg.n_v, cfg.n_c
    n = n_v + n_c
    n_mu = min(max(R.num_aux(cfg.k_mu, n_v, n_c), 1), n_r)
    rng = np.random.default_rng(seed)
    psi, _ = _inputs(cfg, psi, np.zeros(n), rng)
    a, b = psi[:, :n_v], psi[:, n_v:n]
    stages = {}
    s = min(sel_steps, n_mu)
    t_sel, _ = _t(lambda: R.select_points(a, b, s))
    w_s = sum(n + k + 1 for k in range(s))
    w_all = sum(n + k + 1 for k in range(n_mu))
    stages["select"] = t_sel * w_all / w_s
    c = min(cols, n_mu)
    p_blk = np.asfortranarray(rng.standard_normal((n_r, c)) / np.sqrt(n_r))
    t_vp, vp_blk = _t(lambda: ref.apply_coulomb(cfg.dims, cfg.cell3, p_blk, threads=cores))
    t_tn, _ = _t(lambda: ref.matmul_tn(p_blk, vp_blk))
    stages["coulomb"] = t_vp * 2.0 * n_mu / c
    stages["pvp"] = t_tn * (n_mu / c) ** 2
    sample = (f"select {s}/{n_mu} greedy steps (restatement, {cores} threads) x{w_all / w_s:.1f}; apply_coulomb "
              f"{c} cols x{2 * n_mu / c:.0f}; matmul_tn {c}x{c} block x{(n_mu / c) ** 2:.0f}")
    return stages, sample


def run(cfg, psi=None, energies=None, cores=None, sel_steps=64, fit_rows=(2048, 4096), cols=128, seed=5,
        points=None):
    """Returns dict(total_s, total_no_select_s, stages, sample, cores)."""
    cores = cores or os.cpu_count() or 1
    rng = np.random.default_rng(seed)
    psi, e = _inputs(cfg, psi, energies, rng)
    fixed, fs = fixed_pieces(cfg, psi, e, cores, fit_rows, seed, points)
    samp, ss = sampled_pieces(cfg, psi, cores, sel_steps, cols, seed)
    stages = {**samp, **fixed}
    total = sum(stages.values())
    return {"total_s": total, "total_no_select_s": total - stages["select"], "stages": stages,
            "sample": f"{cfg.name}: {ss}; {fs}", "cores": cores}
