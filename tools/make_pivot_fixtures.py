"""Cache the oracle's greedy pivot sequences for the large BASELINE configs.

Runs on a GPU box (the orbitals are generated there, exactly as the tests
generate them: synth.orbitals_device, torch QR on cuda:0), runs
oracle/select.c (the CPU restatement of the reference's qrcp_direct point
selection, all host threads) on the downloaded orbitals and writes
tests/golden/pivots_<cfg>.npz = {sha256 of the orbitals (column-major bytes),
n_mu, pts (sorted), order (pivot order), margins (per step),
recompute_events, seconds}. tests/test_gpu_configs.py uses a fixture only
when the SHA-256 of its own orbitals matches; otherwise it recomputes live.

usage: python tools/make_pivot_fixtures.py [--out DIR] c60 si216 ...
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    from oracle import restate as R
    from paper_2403_12340_b200 import synth
    from test_gpu_configs import psi_sha256

    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden"))
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    for name in args.configs:
        cfg = synth.CONFIGS[name]
        n_mu = R.num_aux(cfg.k_mu, cfg.n_v, cfg.n_c)
        h = synth.orbitals_device(cfg).cpu().numpy()
        sha = psi_sha256(h)
        t0 = time.time()
        pts, diag = R.select_points(h[:, :cfg.n_v], h[:, cfg.n_v:], n_mu, return_diag=True)
        dt = time.time() - t0
        path = os.path.join(args.out, f"pivots_{name}.npz")
        np.savez_compressed(path, sha256=np.array(sha), n_mu=np.array(n_mu), pts=pts.astype(np.int32),
                            order=diag["order"].astype(np.int32), margins=diag["margins"],
                            recompute_events=np.array(diag["recompute_events"]), seconds=np.array(dt))
        print(f"{name}: n_mu={n_mu} select.c {dt:.1f} s on {os.cpu_count()} threads, "
              f"min margin {diag['margins'].min():.3e}, recompute events {diag['recompute_events']} -> {path}",
              flush=True)


if __name__ == "__main__":
    main()
