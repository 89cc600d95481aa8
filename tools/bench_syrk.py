"""Weighted lower SYRK (Theta^T V Theta shape) through lrgw_dev_gram_weighted:
time (CUDA events) + error vs torch. usage: bench_syrk.py m kdim [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2403_12340_b200 import lrgw

    m, kd = int(sys.argv[1]), int(sys.argv[2])
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    ctx = lrgw.Context(0)
    st = torch.cuda.ExternalStream(lrgw.L.load().lrgw_ctx_stream(ctx.handle))
    torch.manual_seed(0)
    x = torch.randn(m, kd, dtype=torch.float64, device="cuda").t()   # kdim x m column-major
    w = torch.rand(kd, dtype=torch.float64, device="cuda")
    out = torch.empty(m, m, dtype=torch.float64, device="cuda").t()
    lrgw.gram_weighted_dev(x, w, out, ctx=ctx)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        lrgw.gram_weighted_dev(x, w, out, ctx=ctx)
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    ref = x.t() @ (w[:, None] * x)
    err = float((ref - out).norm() / ref.norm())
    tf = m * (m + 1) * kd / (ms * 1e-3) / 1e12
    print(f"syrk m={m} k={kd} env={os.environ.get('LRGW_SYRK_L', '-')} ms={ms:.3f} TF={tf:.2f} "
          f"frac={tf / 37.17:.3f} err={err:.2e}")


if __name__ == "__main__":
    main()
