"""Run-to-run determinism of the whole device build: REPS builds of one
config, the points, Theta / T / K and eps^-1 applied to the probe block of
each compared bit for bit with the first build's (every reduction of the
build has a fixed order, so any mismatch is a staging race). Matrices are
compared through a wrapping int64 sum of their bit patterns, so the 58 GB
Theta of Si512 needs no second copy. usage: stress_build.py config reps"""
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
    x = torch.from_numpy(synth.probe_host(cfg.n_r)).cuda().t().contiguous().t()
    y = torch.empty_like(x)

    def bits(ptr, n):
        return int(L_tensor(ptr, (n, 1)).reshape(-1).view(torch.int64).sum().item())

    ref = None
    bad = {"points": 0, "theta": 0, "t": 0, "k": 0, "apply": 0}
    for rep in range(reps + 1):
        ep = lrgw.build(psi[:, :cfg.n_v], psi[:, cfg.n_v:], e, cfg.dims, cfg.cell3, k_mu=cfg.k_mu,
                        n_lambda=cfg.n_lambda, ctx=ctx)
        th_p, k_p, t_p = ep.device_ptrs()
        lrgw.eps_apply_dev(ep, x, y)
        ctx.synchronize()
        cur = {"points": hash(np.array(ep.point_indices).tobytes()), "theta": bits(th_p, cfg.n_r * ep.n_mu),
               "t": bits(t_p, ep.n_mu * ep.n_mu), "k": bits(k_p, ep.n_mu * ep.n_mu),
               "apply": int(y.t().contiguous().view(torch.int64).sum().item())}
        if ref is None:
            ref = cur
        else:
            for k, v in cur.items():
                bad[k] += int(v != ref[k])
        ep.close()
    print(f"stress_build {name} reps={reps} mismatches={bad}", flush=True)


if __name__ == "__main__":
    main()
