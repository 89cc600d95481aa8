"""CUPTI timeline of one warm build (torch.profiler sees every kernel in the
process, ours included): busy vs span, and the largest idle gaps on the GPU.
usage: trace_build.py [config] [n_gaps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_2403_12340_b200 import lrgw, synth

    cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "si64"]
    ngaps = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    psi = synth.orbitals_device(cfg)
    e = synth.energies(cfg)
    ctx = lrgw.Context(0)

    def one():
        ep = lrgw.build(psi[:, :cfg.n_v], psi[:, cfg.n_v:], e, cfg.dims, cfg.cell3, k_mu=cfg.k_mu,
                        n_lambda=cfg.n_lambda, ctx=ctx)
        ep.close()

    one()
    one()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        one()
        torch.cuda.synchronize()
    print("stages", {k: round(v, 3) for k, v in ctx.stage_ms().items()})
    ev = [x for x in prof.events() if x.device_type == torch.autograd.DeviceType.CUDA]
    ev = [x for x in ev if x.time_range.elapsed_us() >= 0]
    ev.sort(key=lambda x: x.time_range.start)
    if not ev:
        print("no device events")
        return
    t0 = ev[0].time_range.start
    busy = sum(x.time_range.elapsed_us() for x in ev)
    span = ev[-1].time_range.end - t0
    print(f"device events={len(ev)} busy={busy / 1e3:.3f} ms span={span / 1e3:.3f} ms idle={(span - busy) / 1e3:.3f} ms")
    gaps = []
    for p, q in zip(ev, ev[1:]):
        g = q.time_range.start - p.time_range.end
        gaps.append((g, p.name[:60], q.name[:60], (p.time_range.end - t0) / 1e3))
    tot = sum(g[0] for g in gaps if g[0] > 0)
    print(f"sum of gaps {tot / 1e3:.3f} ms; gaps > 20 us: {sum(1 for g in gaps if g[0] > 20)} "
          f"totalling {sum(g[0] for g in gaps if g[0] > 20) / 1e3:.3f} ms")
    for g, a, b, at in sorted(gaps, reverse=True)[:ngaps]:
        print(f"{g:9.1f} us at {at:8.3f} ms  after {a}  before {b}")
    if os.environ.get("TRACE_DUMP"):
        with open(os.environ["TRACE_DUMP"], "w") as f:
            for x in ev:
                f.write(f"{(x.time_range.start - t0) / 1e3:9.3f} {x.time_range.elapsed_us():9.1f} {x.name[:110]}\n")
    # per-name busy
    agg = {}
    for x in ev:
        k = x.name[:80]
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + x.time_range.elapsed_us())
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:20]:
        print(f"{t / 1e3:8.3f} ms n={n:4d} {k}")


if __name__ == "__main__":
    main()
