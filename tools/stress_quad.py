"""Run-to-run determinism of the K3 node kernel: REPS launches of
lrgw_dev_contour_partial on one config, each compared bit for bit with the
first (a staging race shows up as a mismatch).
usage: stress_quad.py config reps   (engine variant through LRGW_QUAD_* env)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2403_12340_b200 import lrgw, synth

    name, reps = sys.argv[1], int(sys.argv[2])
    cfg = synth.CONFIGS[name]
    ctx = lrgw.Context(0)
    n_mu = lrgw.num_aux(cfg.k_mu, cfg.n_v, cfg.n_c)
    torch.manual_seed(3)
    pv = torch.randn(cfg.n_v, n_mu, dtype=torch.float64, device="cuda").t() / n_mu ** 0.5
    pc = torch.randn(cfg.n_c, n_mu, dtype=torch.float64, device="cuda").t() / n_mu ** 0.5
    e = synth.energies(cfg)
    nodes = cfg.n_lambda + 1
    ref = torch.empty(n_mu, n_mu, dtype=torch.float64, device="cuda").t()
    acc = torch.empty_like(ref)
    lrgw.contour_partial_dev(pv, pc, e, cfg.n_lambda, 0, nodes, ref, ctx=ctx)
    bad = 0
    worst = 0.0
    for _ in range(reps):
        lrgw.contour_partial_dev(pv, pc, e, cfg.n_lambda, 0, nodes, acc, ctx=ctx)
        d = float((acc - ref).abs().max())
        if d != 0.0:
            bad += 1
            worst = max(worst, d)
    env = {k: v for k, v in os.environ.items() if k.startswith("LRGW_QUAD")}
    print(f"stress {name} reps={reps} env={env} mismatches={bad} worst={worst:.2e}", flush=True)


if __name__ == "__main__":
    main()
