"""CUPTI timeline of the probe apply y = eps^-1 x (Si64 by default)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_2403_12340_b200 import lrgw, synth

    cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "si64"]
    psi = synth.orbitals_device(cfg)
    e = synth.energies(cfg)
    ep = lrgw.build(psi[:, :cfg.n_v], psi[:, cfg.n_v:], e, cfg.dims, cfg.cell3, k_mu=cfg.k_mu, n_lambda=cfg.n_lambda)
    x = torch.randn(8, cfg.n_r, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        lrgw.eps_apply_dev(ep, x.t(), y.t())
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        lrgw.eps_apply_dev(ep, x.t(), y.t())
        torch.cuda.synchronize()
    ev = sorted([v for v in prof.events() if v.device_type == torch.autograd.DeviceType.CUDA],
                key=lambda v: v.time_range.start)
    t0 = ev[0].time_range.start
    for v in ev:
        print(f"{(v.time_range.start - t0) / 1e3:8.3f} {v.time_range.elapsed_us():8.1f} {v.name[:90]}")
    print("span ms", (ev[-1].time_range.end - t0) / 1e3)


if __name__ == "__main__":
    main()
