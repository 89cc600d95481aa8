"""Run-to-run determinism of the whole device build: REPS builds of one
config, Theta / T / K of each compared bit for bit with the first build's
(every reduction of the build has a fixed order, so any mismatch is a
staging race). usage: stress_build.py config reps"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))


def main():
    import numpy as np
    import torch

    from paper_2403_12340_b200 import lrgw, synth
    from test_gpu_build import L_tensor

    name, reps = sys.argv[1], int(sys.argv[2])
    cfg = synth.CONFIGS[name]
    ctx = lrgw.Context(0)
    psi = synth.orbitals_device(cfg)
    e = synth.energies(cfg)
    ref = None
    bad = {"theta": 0, "t": 0, "k": 0, "points": 0}
    worst = {"theta": 0.0, "t": 0.0, "k": 0.0}
    for rep in range(reps + 1):
        ep = lrgw.build(psi[:, :cfg.n_v], psi[:, cfg.n_v:], e, cfg.dims, cfg.cell3, k_mu=cfg.k_mu,
                        n_lambda=cfg.n_lambda, ctx=ctx)
        th_p, k_p, t_p = ep.device_ptrs()
        cur = {"theta": L_tensor(th_p, (cfg.n_r, ep.n_mu)), "k": L_tensor(k_p, (ep.n_mu, ep.n_mu)),
               "t": L_tensor(t_p, (ep.n_mu, ep.n_mu))}
        pts = np.array(ep.point_indices)
        if ref is None:
            ref = {k: v.clone() for k, v in cur.items()}
            ref_pts = pts
        else:
            if not np.array_equal(pts, ref_pts):
                bad["points"] += 1
            for k, v in cur.items():
                d = float((v - ref[k]).abs().max() / ref[k].abs().max())
                if d != 0.0:
                    bad[k] += 1
                    worst[k] = max(worst[k], d)
        ep.close()
    print(f"stress_build {name} reps={reps} mismatches={bad} worst_rel={worst}", flush=True)


if __name__ == "__main__":
    main()
