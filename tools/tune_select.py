"""Time the Si64 build's point selection for several candidate batch sizes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    from paper_2403_12340_b200 import lrgw, synth

    cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "si64"]
    psi = synth.orbitals_device(cfg)
    e = synth.energies(cfg)
    ref_pts = None
    for s in (32, 48, 64, 96, 128):
        ctx = lrgw.Context(0)
        ctx.set_select_batch(s)
        for it in range(3):
            ep = lrgw.build(psi[:, :cfg.n_v], psi[:, cfg.n_v:], e, cfg.dims, cfg.cell3, k_mu=cfg.k_mu,
                            n_lambda=cfg.n_lambda, ctx=ctx)
            st = ctx.stage_ms()
            pts = ep.point_indices
            ep.close()
        if ref_pts is None:
            ref_pts = pts
        print(f"s={s:4d} select={st['select']:.3f} ms total={st['total']:.3f} ms same_pts={np.array_equal(pts, ref_pts)}",
              flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
