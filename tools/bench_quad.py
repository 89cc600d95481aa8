"""K3 node kernel on its two feeds (TMA ring, quad4.cu, vs the cp.async ring,
quadrature.cu) through lrgw_dev_contour_partial at the BASELINE shapes:
time (CUDA events on the library stream, all N_lambda + 1 nodes) and the
relative difference of the two results (QUAD_SWEEP=1: every k-tile depth of
the TMA feed). usage: bench_quad.py [config ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2403_12340_b200 import lrgw, synth

    names = sys.argv[1:] or ["si64", "c60", "si216", "si512"]
    ctx = lrgw.Context(0)
    st = torch.cuda.ExternalStream(lrgw.L.load().lrgw_ctx_stream(ctx.handle))
    for name in names:
        cfg = synth.CONFIGS[name]
        n_mu = lrgw.num_aux(cfg.k_mu, cfg.n_v, cfg.n_c)
        torch.manual_seed(3)
        pv = torch.randn(cfg.n_v, n_mu, dtype=torch.float64, device="cuda").t() / n_mu ** 0.5
        pc = torch.randn(cfg.n_c, n_mu, dtype=torch.float64, device="cuda").t() / n_mu ** 0.5
        e = synth.energies(cfg)
        nodes = cfg.n_lambda + 1
        flop = 2.0 * n_mu * (n_mu + 1) * (cfg.n_v + cfg.n_c) * nodes
        variants = [("cp.async", {"LRGW_QUAD_TMA": "0"})]
        if os.environ.get("QUAD_SWEEP"):
            for bk in ("16", "24", "32", "40", "48", "64"):
                variants.append((f"tma bk{bk}", {"LRGW_QUAD_TMA": "1", "LRGW_QUAD_BK": bk}))
        else:
            variants.append(("tma", {"LRGW_QUAD_TMA": "1"}))
        ref = None
        for label, env in variants:
            for k in ("LRGW_QUAD_TMA", "LRGW_QUAD_BK"):
                os.environ.pop(k, None)
            os.environ.update(env)
            acc = torch.empty(n_mu, n_mu, dtype=torch.float64, device="cuda").t()
            lrgw.contour_partial_dev(pv, pc, e, cfg.n_lambda, 0, nodes, acc, ctx=ctx)
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                lrgw.contour_partial_dev(pv, pc, e, cfg.n_lambda, 0, nodes, acc, ctx=ctx)
                e1.record(st)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            if ref is None:
                ref = acc.clone()
            diff = float((ref - acc).norm() / ref.norm())
            # run-to-run determinism (a staging race shows up here)
            acc2 = torch.empty_like(acc)
            lrgw.contour_partial_dev(pv, pc, e, cfg.n_lambda, 0, nodes, acc2, ctx=ctx)
            ctx.synchronize()
            rr = float((acc2 - acc).abs().max())
            ms = min(ts)
            tf = flop / (ms * 1e-3) / 1e12
            print(f"quad {name} n_mu={n_mu} bands={cfg.n_v}+{cfg.n_c} nodes={nodes} feed={label} ms={ms:.3f} "
                  f"TF={tf:.2f} frac={tf / 37.17:.3f} rel diff vs cp.async={diff:.1e} rerun maxabs={rr:.1e}", flush=True)


if __name__ == "__main__":
    main()
