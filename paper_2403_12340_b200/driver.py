"""The reference driver's `run` and `scale` commands over the B200 path
(reference driver.hpp:20-329, 713-871; tools/lrgw_cli.cpp).

Same configuration schema and validation messages (RunConfig /
parse_config / config_to_json, driver.hpp:20-155), same result schemas
(run_result.json + bands.csv, scale_result.json), with every stage of the
low-rank pipeline on the GPU: vc / vn / nn ISDF (K1 + fused fit), the
contour core (K3, adaptive or bypassed as in driver.hpp:230-243), the
factored eps^-1 (K4-K6), the screened projections and the Hadamard-form
self-energies. The dense pipelines (`isdf_conventional`, `bruteforce`) and
the dense-LU timings of `scale` build N_r x N_r operators: they are the
reference's test oracles, not part of this path, and are refused here
(`Unsupported`) or reported as skipped.

    python -m paper_2403_12340_b200.driver run config.json
    python -m paper_2403_12340_b200.driver scale config.json --sizes 8 16 32
"""
from __future__ import annotations

import argparse
import json
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import lrgw

# ---------------------------------------------------------------------------
# Configuration (driver.hpp:20-155)
# ---------------------------------------------------------------------------


@dataclass
class RunConfig:
    seed: int = 1
    dims: tuple = (8, 8, 8)
    cell: tuple = (6.0, 6.0, 6.0)
    n_v: int = 16
    n_c: int = 16
    gap: float = 1.0
    bandwidth: float = 4.0
    wfn_path: str = ""
    k_vc: float = 8.0
    k_vn: float = 8.0
    k_nn: float = 8.0
    selector: str = "qrcp_direct"
    delta_rel: float = 1e-7
    max_nodes: int = 1025
    pipeline: str = "lowrank"
    threads: int = 1
    out_dir: str = "."
    hook_flip_sex_x: bool = False


_SELECTORS = ("qrcp_direct", "qrcp_sketched")
_PIPELINES = ("lowrank", "isdf_conventional", "bruteforce")


def _get(d, key, kind, what):
    v = d[key]
    ok = {"int": lambda x: isinstance(x, (int, float)) and not isinstance(x, bool),
          "num": lambda x: isinstance(x, (int, float)) and not isinstance(x, bool),
          "str": lambda x: isinstance(x, str),
          "bool": lambda x: isinstance(x, bool)}[kind](v)
    if not ok:
        raise lrgw.InvalidInput(f"config: malformed field: {what}: type must be {kind}")
    return int(v) if kind == "int" else (float(v) if kind == "num" else v)


def _get3(d, key, kind, what):
    v = d[key]
    if not isinstance(v, list) or len(v) < 3:
        raise lrgw.InvalidInput(f"config: malformed field: {what}: expected an array of 3")
    return tuple(_get({"x": v[i]}, "x", kind, what) for i in range(3))


def parse_config(j: dict) -> RunConfig:
    """driver.hpp:62-121 (same defaults, checks and messages)."""
    c = RunConfig()
    if not isinstance(j, dict):
        raise lrgw.InvalidInput("config: malformed field: top level must be an object")
    s = j.get("system")
    if s is not None:
        if "wfn" in s:
            c.wfn_path = _get(s, "wfn", "str", "system.wfn")
        if "seed" in s:
            c.seed = _get(s, "seed", "int", "system.seed")
        if "dims" in s:
            c.dims = _get3(s, "dims", "int", "system.dims")
        if "cell" in s:
            c.cell = _get3(s, "cell", "num", "system.cell")
        if "nv" in s:
            c.n_v = _get(s, "nv", "int", "system.nv")
        if "nc" in s:
            c.n_c = _get(s, "nc", "int", "system.nc")
        if "gap" in s:
            c.gap = _get(s, "gap", "num", "system.gap")
        if "bandwidth" in s:
            c.bandwidth = _get(s, "bandwidth", "num", "system.bandwidth")
    s = j.get("isdf")
    if s is not None:
        for k in ("k_vc", "k_vn", "k_nn"):
            if k in s:
                setattr(c, k, _get(s, k, "num", f"isdf.{k}"))
        if "selector" in s:
            sel = _get(s, "selector", "str", "isdf.selector")
            if sel not in _SELECTORS:
                raise lrgw.InvalidInput(f"config: unknown selector '{sel}'")
            c.selector = sel
    s = j.get("contour")
    if s is not None:
        if "delta_rel" in s:
            c.delta_rel = _get(s, "delta_rel", "num", "contour.delta_rel")
        if "max_nodes" in s:
            c.max_nodes = _get(s, "max_nodes", "int", "contour.max_nodes")
    if "pipeline" in j:
        p = _get(j, "pipeline", "str", "pipeline")
        if p not in _PIPELINES:
            raise lrgw.InvalidInput(f"config: unknown pipeline '{p}'")
        c.pipeline = p
    if "threads" in j:
        c.threads = _get(j, "threads", "int", "threads")
    if "out" in j:
        c.out_dir = _get(j, "out", "str", "out")
    h = j.get("_test_hooks")
    if h is not None and "flip_sex_x_sign" in h:
        c.hook_flip_sex_x = _get(h, "flip_sex_x_sign", "bool", "_test_hooks.flip_sex_x_sign")
    if not (c.k_vc > 0.0 and c.k_vn > 0.0 and c.k_nn > 0.0):
        raise lrgw.InvalidInput("config: ISDF coefficients must be > 0")
    if not (0.0 < c.delta_rel < 0.5):
        raise lrgw.InvalidInput("config: delta_rel must lie in (0, 0.5)")
    if c.max_nodes < 33:
        raise lrgw.InvalidInput("config: max_nodes must allow at least two levels (>= 33)")
    if c.threads < 1:
        raise lrgw.InvalidInput("config: threads must be >= 1")
    if c.wfn_path and not os.path.exists(c.wfn_path):
        raise lrgw.InvalidInput("config: wavefunction file does not exist: " + c.wfn_path)
    return c


def load_config(path: str) -> RunConfig:
    """driver.hpp:123-133."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise lrgw.InvalidInput("config: cannot open " + str(path)) from None
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise lrgw.InvalidInput(f"config: invalid JSON: {e}") from None
    return parse_config(j)


def config_to_json(c: RunConfig) -> dict:
    """driver.hpp:135-149."""
    j = {"system": {"seed": c.seed, "dims": list(c.dims), "cell": list(c.cell), "nv": c.n_v, "nc": c.n_c,
                    "gap": c.gap, "bandwidth": c.bandwidth}}
    if c.wfn_path:
        j["system"]["wfn"] = c.wfn_path
    j["isdf"] = {"k_vc": c.k_vc, "k_vn": c.k_vn, "k_nn": c.k_nn, "selector": c.selector}
    j["contour"] = {"delta_rel": c.delta_rel, "max_nodes": c.max_nodes}
    j["pipeline"] = c.pipeline
    j["threads"] = c.threads
    return j


# ---------------------------------------------------------------------------
# Systems (driver.hpp:151-156; model.hpp:56-116)
# ---------------------------------------------------------------------------

_PCG_MULT = np.uint64(6364136223846793005)
_PCG_INC = np.uint64(1442695040888963407)


def _pcg32_stream(seed: int, n: int) -> np.ndarray:
    """n successive outputs of rng.hpp's PCG32 (pcg32_oneseq) from Rng(seed),
    by LCG jump-ahead: state_i = A^i s_0 + C_i, all mod 2^64."""
    m = (1 << 64) - 1
    s = (0 * 6364136223846793005 + 1442695040888963407) & m  # constructor: one step from 0
    s = (s + (0x853C49E6748FEA9B ^ seed)) & m
    s = (s * 6364136223846793005 + 1442695040888963407) & m  # second step
    with np.errstate(over="ignore"):
        a_pow = np.empty(n, dtype=np.uint64)
        c_acc = np.empty(n, dtype=np.uint64)
        a_pow[0], c_acc[0] = np.uint64(1), np.uint64(0)
        if n > 1:
            a_pow[1:] = np.cumprod(np.full(n - 1, _PCG_MULT, dtype=np.uint64))
            c_acc[1:] = np.cumsum(a_pow[:-1] * _PCG_INC)
        old = a_pow * np.uint64(s) + c_acc
        xorshifted = (((old >> np.uint64(18)) ^ old) >> np.uint64(27)) & np.uint64(0xFFFFFFFF)
        rot = old >> np.uint64(59)
        out = (xorshifted >> rot) | (xorshifted << ((np.uint64(32) - rot) & np.uint64(31)))
    return (out & np.uint64(0xFFFFFFFF)).astype(np.float64)


def _gaussians(seed: int, n: int) -> np.ndarray:
    """rng.hpp:36-48 Box-Muller with the cached second variate (n even)."""
    u = (_pcg32_stream(seed, n) + 1.0) / 4294967296.0
    u1, u2 = u[0::2], u[1::2]
    r = np.sqrt(-2.0 * np.log(u1))
    a = 6.283185307179586476925286766559 * u2
    g = np.empty(n)
    g[0::2] = r * np.cos(a)
    g[1::2] = r * np.sin(a)
    return g


def _qrcp_q(a: np.ndarray) -> np.ndarray:
    """The orthonormal factor of linalg.hpp:26-111 (greedy Householder QRCP,
    strict '>' pivot with the swap-mirrored order, norm downdate with the
    1e-12 recompute rule). Input generation only (desk-scale grids)."""
    a = np.array(a, dtype=np.float64, order="F")
    m, n = a.shape
    k = min(m, n)
    cnorm = np.einsum("ij,ij->j", a, a)
    corig = cnorm.copy()
    tau = np.zeros(k)
    for step in range(k):
        p = step + int(np.argmax(cnorm[step:]))  # first maximum == strict '>' scan
        if p != step:
            a[:, [step, p]] = a[:, [p, step]]
            cnorm[[step, p]] = cnorm[[p, step]]
            corig[[step, p]] = corig[[p, step]]
        alpha = math.sqrt(float(np.dot(a[step:, step], a[step:, step])))
        if alpha == 0.0:
            tau[step] = 0.0
        else:
            if a[step, step] > 0.0:
                alpha = -alpha
            v0 = a[step, step] - alpha
            a[step + 1:, step] /= v0
            tau[step] = -v0 / alpha
            a[step, step] = alpha
            v = a[step + 1:, step]
            s = (a[step, step + 1:] + v @ a[step + 1:, step + 1:]) * tau[step]
            a[step, step + 1:] -= s
            a[step + 1:, step + 1:] -= np.outer(v, s)
        t = a[step, step + 1:]
        cnorm[step + 1:] -= t * t
        bad = np.nonzero((cnorm[step + 1:] < 1e-12 * corig[step + 1:]) | (cnorm[step + 1:] < 0.0))[0]
        for j in bad + step + 1:
            cnorm[j] = float(np.dot(a[step + 1:, j], a[step + 1:, j]))
    q = np.zeros((m, k), order="F")
    q[np.arange(k), np.arange(k)] = 1.0
    for step in range(k - 1, -1, -1):
        if tau[step] == 0.0:
            continue
        v = a[step + 1:, step]
        s = (q[step, :] + v @ q[step + 1:, :]) * tau[step]
        q[step, :] -= s
        q[step + 1:, :] -= np.outer(v, s)
    return q


def synthetic_system(seed: int, dims, cell, n_v: int, n_c: int, gap: float,
                     bandwidth: float) -> lrgw.ElectronicStructure:
    """model.hpp:56-116 (build_synthetic_system): band-limited Gaussian random
    fields (unitary inverse DFT of enveloped complex Gaussians), QRCP
    orthonormalised against the dV inner product; energies on [-bandwidth, 0]
    and [gap, gap + bandwidth]. Equal to the reference to rounding (the
    inverse DFT here is an FFT); WFN1 files give bit-identical inputs."""
    if not gap > 0.0:
        raise lrgw.InvalidInput("build_synthetic_system: gap must be > 0")
    if not bandwidth >= gap:
        raise lrgw.InvalidInput("build_synthetic_system: bandwidth must be >= gap")
    if n_v < 1 or n_c < 1:
        raise lrgw.InvalidInput("build_synthetic_system: need n_v >= 1 and n_c >= 1")
    dims = tuple(int(d) for d in dims)
    cell = tuple(float(x) for x in cell)
    for k in range(3):
        if dims[k] < 2:
            raise lrgw.InvalidInput("Grid: all dims must be >= 2")
        if not cell[k] > 0.0:
            raise lrgw.InvalidInput("Grid: cell lengths must be > 0")
    n_r, nb = dims[0] * dims[1] * dims[2], n_v + n_c
    if nb > n_r:
        raise lrgw.InvalidInput("build_synthetic_system: grid too small for band count")
    pi = 3.14159265358979323846
    g_nyq = min(pi * dims[k] / cell[k] for k in range(3))
    sigma2 = (g_nyq / 3.0) ** 2
    two_pi = 6.283185307179586476925286766559
    g = [two_pi * np.array([i if i <= n // 2 else i - n for i in range(n)], dtype=np.float64) / a
         for n, a in zip(dims, cell)]
    g2 = (g[0][None, None, :] ** 2 + g[1][None, :, None] ** 2 + g[2][:, None, None] ** 2).reshape(-1)
    env = np.exp(-g2 / (2.0 * sigma2))
    gs = _gaussians(seed, 2 * n_r * nb).reshape(nb, n_r, 2)
    fields = np.empty((n_r, nb), order="F")
    for b in range(nb):
        # cplx(rng.gaussian(), rng.gaussian()) (model.hpp:83): the reference build
        # evaluates the imaginary argument first (GCC, right to left)
        coef = (env * gs[b, :, 1] + 1j * (env * gs[b, :, 0])).reshape(dims[2], dims[1], dims[0])
        fields[:, b] = np.fft.ifftn(coef, norm="ortho").real.reshape(-1)
    q = _qrcp_q(fields)
    dv = cell[0] * cell[1] * cell[2] / n_r
    psi = np.asfortranarray(q * (1.0 / math.sqrt(dv)))
    ev = [0.0 if n_v == 1 else -bandwidth * (n_v - 1 - i) / float(n_v - 1) for i in range(n_v)]
    ec = [gap + (0.0 if n_c == 1 else bandwidth * j / float(n_c - 1)) for j in range(n_c)]
    return lrgw.ElectronicStructure(dims, cell, psi, np.array(ev + ec), np.zeros(nb), n_v, n_c)


def build_system(c: RunConfig) -> lrgw.ElectronicStructure:
    if c.wfn_path:
        return lrgw.load_system(c.wfn_path)
    return synthetic_system(c.seed, c.dims, c.cell, c.n_v, c.n_c, c.gap, c.bandwidth)


# ---------------------------------------------------------------------------
# run (driver.hpp:158-304)
# ---------------------------------------------------------------------------


class StageTimer:
    """driver.hpp:161-199 — wall time per stage (the device work of every
    stage completes inside it: each C-ABI call synchronises), failures
    re-raised as numeric_error with the stage name."""

    def __init__(self):
        self.entries = []

    def time(self, stage, fn):
        t0 = time.perf_counter()
        try:
            out = fn()
        except lrgw.LrgwError as e:
            raise lrgw.NumericError(f"stage '{stage}': {e}") from e
        self.entries.append((stage, time.perf_counter() - t0))
        return out


@dataclass
class RunResult:
    pipeline: str = "lowrank"
    eps_ks: np.ndarray = None
    vxc: np.ndarray = None
    sigma: lrgw.SelfEnergies = None
    qp: lrgw.QuasiparticleEnergies = None
    nodes_used: int = 0
    est_rel_error: float = 0.0
    timings: list = field(default_factory=list)


def _isdf_set(es, c: RunConfig, ctx, k=None):
    kv = k if k is not None else (c.k_vc, c.k_vn, c.k_nn)
    return {lab: lrgw.build_isdf(es.psi, es.n_v, es.n_c, kk, ctx=ctx, label=lab)
            for lab, kk in zip(("vc", "vn", "nn"), kv)}


def coupled_coefficients_auto(es, dec_vc, c: RunConfig, ctx):
    """driver.hpp:230-243: contour for gapped spectra, direct when bypassed."""
    pts = dec_vc.point_indices
    pv, pc = es.psi[pts, :es.n_v], es.psi[pts, es.n_v:]
    spec = lrgw.elliptic_params(es.energies, es.n_v, es.n_c, c.delta_rel, c.max_nodes)
    if spec.bypass:
        return lrgw.coupled_coefficients_direct(pv, pc, es.energies, ctx=ctx)
    return lrgw.coupled_coefficients_contour(pv, pc, es.energies, spec, c.threads, ctx=ctx)


def run_pipeline(c: RunConfig, ctx=None) -> RunResult:
    """driver.hpp:253-304 for the low-rank pipeline, every stage on the GPU."""
    if c.pipeline != "lowrank":
        raise lrgw.Unsupported(f"run: pipeline '{c.pipeline}' builds dense N_r x N_r operators (a reference "
                               "oracle); the B200 path runs 'lowrank'")
    ctx = ctx or lrgw.default_context()
    timer = StageTimer()
    out = RunResult(pipeline=c.pipeline)
    es = timer.time("build", lambda: build_system(c))
    timer.time("coulomb", lambda: lrgw.coulomb_kernel(es.dims, es.cell))
    dec = timer.time("isdf", lambda: _isdf_set(es, c, ctx))
    t = timer.time("contour", lambda: coupled_coefficients_auto(es, dec["vc"], c, ctx))
    out.nodes_used, out.est_rel_error = t.nodes_used, t.est_rel_error
    e = timer.time("inversion", lambda: lrgw.build_epsilon_inverse(t.t, dec["vc"].p, es.dims, es.cell, ctx=ctx))
    proj = timer.time("projection", lambda: lrgw.project_screened_interactions(e, dec["vn"], dec["nn"]))

    def sigma():
        sig = lrgw.self_energies_lowrank(es.psi, es.n_v, proj.w_vn, proj.w_nn, proj.v_vn, dec["vn"], dec["nn"],
                                         ctx=ctx)
        if c.hook_flip_sex_x:  # driver.hpp:245-249 (validation mutation hook)
            sig.sigma_sex_x = -sig.sigma_sex_x
            sig.sigma_total = sig.sigma_sex_x + sig.sigma_x + sig.sigma_coh
        return sig

    out.sigma = timer.time("sigma", sigma)
    e.close()
    out.eps_ks, out.vxc = es.energies, es.vxc
    out.qp = timer.time("qp", lambda: lrgw.quasiparticle_energies(es.energies, es.vxc, out.sigma))
    out.timings = timer.entries
    return out


def run_result_to_json(r: RunResult, c: RunConfig) -> dict:
    """driver.hpp:306-329."""
    bands = []
    for n in range(len(r.eps_ks)):
        bands.append({"n": n, "eps_ks": float(r.eps_ks[n]), "vxc": float(r.vxc[n]),
                      "sigma_sex_x": float(r.sigma.sigma_sex_x[n]), "sigma_x": float(r.sigma.sigma_x[n]),
                      "sigma_coh": float(r.sigma.sigma_coh[n]), "sigma_total": float(r.sigma.sigma_total[n]),
                      "eps_gw": float(r.qp.eps_gw[n])})
    return {"kind": "run", "pipeline": r.pipeline, "nodes_used": int(r.nodes_used),
            "est_rel_error": float(r.est_rel_error), "bands": bands,
            "timings_s": {name: sec for name, sec in r.timings}, "config": config_to_json(c)}


def write_bands_csv(result: dict, path: str) -> None:
    """The `report` CSV of a run result (driver.hpp:896-912)."""
    with open(path, "w") as f:
        f.write("n,eps_ks,sigma_sex_x,sigma_x,sigma_coh,sigma_total,eps_gw\n")
        for b in result["bands"]:
            f.write(",".join([str(b["n"])] + ["%.17g" % b[k] for k in
                                              ("eps_ks", "sigma_sex_x", "sigma_x", "sigma_coh", "sigma_total",
                                               "eps_gw")]) + "\n")


# ---------------------------------------------------------------------------
# scale (driver.hpp:713-871)
# ---------------------------------------------------------------------------


def dims_for_points(n: int):
    """driver.hpp:737-747."""
    k = 0
    while (1 << k) < n:
        k += 1
    return (1 << ((k + 2) // 3), 1 << ((k + 1) // 3), 1 << (k // 3))


def loglog_slope(pts):
    n = float(len(pts))
    lx = [math.log(x) for x, _ in pts]
    ly = [math.log(max(y, 1e-12)) for _, y in pts]
    sx, sy = sum(lx), sum(ly)
    sxx = sum(v * v for v in lx)
    sxy = sum(a * b for a, b in zip(lx, ly))
    return (n * sxy - sx * sy) / (n * sxx - sx * sx)


def run_scale(c: RunConfig, sizes, ctx=None) -> dict:
    """driver.hpp:763-849: contour / inversion / projection timed (median of
    3, ISDF setup excluded) across N_e. Every timed call synchronises the
    device. The dense-LU oracle is not on the B200 path: dense_skipped."""
    if not sizes:
        raise lrgw.InvalidInput("scale: size list is empty")
    if any(b <= a for a, b in zip(sizes, sizes[1:])):
        raise lrgw.InvalidInput("scale: sizes must be strictly ascending")
    ctx = ctx or lrgw.default_context()
    rows = []
    for n_e in sizes:
        if n_e < 2:
            raise lrgw.InvalidInput("scale: N_e must be >= 2")
        n_v = max(1, n_e // 2)
        dims = dims_for_points(16 * n_e)
        cell = tuple(0.75 * d for d in dims)
        es = synthetic_system(c.seed, dims, cell, n_v, n_v, c.gap, c.bandwidth)
        k_eff = min(c.k_vc, math.sqrt(n_v * n_v))
        dec = lrgw.build_isdf(es.psi, n_v, n_v, k_eff, ctx=ctx, label="vc")

        def timed(fn):
            ts = []
            out = None
            for _ in range(3):
                t0 = time.perf_counter()
                out = fn()
                ts.append(time.perf_counter() - t0)
            return sorted(ts)[1], out

        t_c, t = timed(lambda: coupled_coefficients_auto(es, dec, c, ctx))
        t_i, e = timed(lambda: lrgw.build_epsilon_inverse(t.t, dec.p, dims, cell, ctx=ctx))
        t_p, _ = timed(lambda: lrgw.project_screened_interactions(e, dec, dec))
        e.close()
        rows.append({"n_e": n_e, "n_r": es.n_r, "n_mu": dec.n_mu, "t_contour_s": t_c, "t_inversion_s": t_i,
                     "t_projection_s": t_p, "t_lowrank_s": t_c + t_i + t_p, "t_dense_s": 0.0,
                     "dense_skipped": True})
    lr = [(r["n_e"], r["t_lowrank_s"]) for r in rows]
    return {"kind": "scale", "rows": rows,
            "slopes": {"lowrank": loglog_slope(lr) if len(lr) >= 2 else 0.0, "dense": 0.0, "dense_points": 0},
            "config": config_to_json(c)}


def main(argv=None):
    ap = argparse.ArgumentParser(prog="lrgw", description=__doc__.splitlines()[0])
    ap.add_argument("command", choices=("run", "scale"))
    ap.add_argument("config")
    ap.add_argument("--sizes", type=int, nargs="*", default=[8, 16, 32])
    args = ap.parse_args(argv)
    c = load_config(args.config)
    os.makedirs(c.out_dir, exist_ok=True)
    if args.command == "run":
        res = run_result_to_json(run_pipeline(c), c)
        path = os.path.join(c.out_dir, "run_result.json")
        with open(path, "w") as f:
            json.dump(res, f, indent=2)
        write_bands_csv(res, os.path.join(c.out_dir, "bands.csv"))
    else:
        res = run_scale(c, args.sizes)
        path = os.path.join(c.out_dir, "scale_result.json")
        with open(path, "w") as f:
            json.dump(res, f, indent=2)
    print(path)


if __name__ == "__main__":
    main()
