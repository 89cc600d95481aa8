"""The reference CPU implementation of the eps^-1 build run IN FULL (no
sampling, no extrapolation) on the Si64 workload, at threads = 1 and
threads = nproc, on the GPU box's host — the measurement that validates the
bounded-sample extrapolation of oracle/cpu_baseline.py.

Stages through oracle/_ref (the unmodified reference headers):
  select   oracle/select.c (the restatement: the reference's qrcp is
           guard-blocked at Si64, isdf.hpp:49, 77-78), OpenMP threads
  fit      fit_auxiliary_basis (isdf.hpp:118-163) on all N_r rows (serial in
           the reference)
  contour  detail::sum_node_terms over the N_lambda + 1 = 25 nodes (threads)
  smw      build_epsilon_inverse + epsilon_inverse_apply on the 8-column probe
           (smw.hpp:84-103; apply_coulomb threaded, matmul_tn / LU / sym_eig serial)
plus the reference's own qrcp point selection at Si8 (materialised pair
matrix, O(N_v N_c N_r N_mu) — quartic in the system size).

usage: python tools/cpu_reference_full.py [--out profiles/r02/cpu_reference_full_si64.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _t(fn):
    t0 = time.perf_counter()
    out = fn()
    return time.perf_counter() - t0, out


def run(cfg, psi, e, threads):
    from oracle import ref
    from oracle import restate as R
    from paper_2403_12340_b200 import synth

    os.environ["OMP_NUM_THREADS"] = str(threads)
    a, b = psi[:, :cfg.n_v], psi[:, cfg.n_v:]
    n_mu = R.num_aux(cfg.k_mu, cfg.n_v, cfg.n_c)
    st = {}
    st["select"], pts = _t(lambda: R.select_points(a, b, n_mu))
    st["fit"], th = _t(lambda: ref.fit(a, b, pts))
    s7 = ref.elliptic_params(e, cfg.n_v, cfg.n_c)
    h = 2 * s7[3] / cfg.n_lambda
    nodes = [-s7[3] + i * h for i in range(cfg.n_lambda + 1)]
    w = [0.5 * h if i in (0, cfg.n_lambda) else h for i in range(cfg.n_lambda + 1)]
    st["contour"], acc = _t(lambda: ref.sum_node_terms(a[pts], b[pts], e, s7, nodes, w, threads=threads))
    t = 2 * np.sqrt(s7[0] * s7[1]) / (np.pi * s7[2]) * acc
    t = 0.5 * (t + t.T)
    x = synth.probe_host(cfg.n_r)
    st["smw_and_apply"], _ = _t(lambda: ref.build_and_apply(t, th, cfg.dims, cfg.cell3, x, threads=threads))
    st["total"] = sum(st.values())
    st["total_no_select"] = st["total"] - st["select"]
    return {k: round(v, 2) for k, v in st.items()}


def main():
    from oracle import ref
    from paper_2403_12340_b200 import synth

    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "cpu_reference_full_si64.json"))
    args = ap.parse_args()
    cfg = synth.CONFIGS["si64"]
    psi = np.asfortranarray(synth.orbitals_device(cfg).cpu().numpy())
    e = synth.energies(cfg)
    nproc = os.cpu_count() or 1
    out = {"config": "si64 (BASELINE.json configs[1]): N_r 110592, N_v = N_c = 128, N_mu 1024, N_lambda 24",
           "host_cores": nproc, "inputs": "synth.orbitals_device (the bench's seeded QR orbitals), synth.energies"}
    for th in (nproc, 1):
        out[f"threads_{th}"] = run(cfg, psi, e, th)
        print(json.dumps({f"threads_{th}": out[f"threads_{th}"]}), flush=True)
    s8 = synth.CONFIGS["si8"]
    p8 = synth.orbitals_host(s8)
    t_q, _ = _t(lambda: ref.select_points(p8[:, :16], p8[:, 16:], 128))
    out["si8_reference_qrcp_select_s"] = round(t_q, 3)
    out["si8_note"] = ("the reference's own select_interpolation_points -> qrcp (isdf.hpp:95-112, "
                       "linalg.hpp:26-111) on the 256 x 13824 pair matrix: O(N_v N_c N_r N_mu), quartic in N")
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
