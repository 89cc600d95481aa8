"""Time the build's point selection for several candidate batch sizes
(median / min over repeated builds; pivots must not depend on the batch).
usage: tune_select.py [config] [s,s,...] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np

    from paper_2403_12340_b200 import lrgw, synth

    cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "si64"]
    sizes = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "32,48,64,96,128").split(",")]
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 7
    psi = synth.orbitals_device(cfg)
    e = synth.energies(cfg)
    ref_pts = None
    for s in sizes:
        ctx = lrgw.Context(0)
        ctx.set_select_batch(s)
        sel, tot = [], []
        for it in range(reps + 1):
            ep = lrgw.build(psi[:, :cfg.n_v], psi[:, cfg.n_v:], e, cfg.dims, cfg.cell3, k_mu=cfg.k_mu,
                            n_lambda=cfg.n_lambda, ctx=ctx)
            st = ctx.stage_ms()
            pts = ep.point_indices
            ep.close()
            if it:
                sel.append(st["select"])
                tot.append(st["total"])
        if ref_pts is None:
            ref_pts = pts
        print(f"s={s:4d} select med={np.median(sel):.3f} min={min(sel):.3f} ms  total med={np.median(tot):.3f} "
              f"min={min(tot):.3f} ms same_pts={np.array_equal(pts, ref_pts)}", flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
