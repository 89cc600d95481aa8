"""One warm-up + one measured Si64 build (for ncu launch lists: analyse the
second half of the launches)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2403_12340_b200 import lrgw, synth

    cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "si64"]
    psi = synth.orbitals_device(cfg)
    e = synth.energies(cfg)
    ctx = lrgw.Context(0)
    for it in range(2):
        if it == 1:  # ncu --profile-from-start off: only the second (warm) build
            torch.cuda.synchronize()
            torch.cuda.profiler.start()
        ep = lrgw.build(psi[:, :cfg.n_v], psi[:, cfg.n_v:], e, cfg.dims, cfg.cell3, k_mu=cfg.k_mu,
                        n_lambda=cfg.n_lambda, ctx=ctx)
        ep.close()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("stages", ctx.stage_ms())


if __name__ == "__main__":
    main()
