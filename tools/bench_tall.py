"""Tall-skinny L-pass shapes of the selection (C = A B^T, both MN-contiguous),
timed through lrgw_dev_dgemm with CUDA events; the engine is chosen by the
environment (LRGW_TMA_TALL / LRGW_TMA_TALLCFG), one process per variant.
usage: bench_tall.py <tag>"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2403_12340_b200 import lrgw

    tag = sys.argv[1] if len(sys.argv) > 1 else ""
    ctx = lrgw.Context(0)
    lib = lrgw.L.load()
    st = torch.cuda.ExternalStream(lib.lrgw_ctx_stream(ctx.handle))
    mode = os.environ.get("BENCH_MODE", "lpass")
    if mode == "had":
        return had(torch, lrgw, ctx, st, tag)
    cases = [(110592, n, k) for n in (64, 73, 80) for k in (256, 512, 900)]
    cases += [(884736, n, k) for n in (80, 96, 112) for k in (1024, 4096, 7000)]
    big = {}
    for m, n, k in cases:
        if m not in big:
            kmax = max(kk for mm, _, kk in cases if mm == m)
            big[m] = torch.randn(kmax, m, dtype=torch.float64, device="cuda").t()
        a = big[m][:, :k]
        b = torch.randn(k, n + (n & 1), dtype=torch.float64, device="cuda").t()[:n]
        c = torch.empty(n, m, dtype=torch.float64, device="cuda").t()
        lrgw.dgemm_dev("N", "T", 1.0, a, b, 0.0, c, ctx=ctx)
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            lrgw.dgemm_dev("N", "T", 1.0, a, b, 0.0, c, ctx=ctx)
            e1.record(st)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[len(ts) // 2]
        tf = 2.0 * m * n * k / (ms * 1e-3) / 1e12
        r = torch.matmul(a[:4096], b.t())
        err = float((r - c[:4096]).norm() / r.norm())
        print(f"{tag:12s} m={m:6d} n={n:3d} k={k:5d}: {ms:8.3f} ms {tf:6.2f} TF/s ({tf / 37.17 * 100:5.1f}%) err={err:.1e}",
              flush=True)
        del a, b, c


def had(torch, lrgw, ctx, st, tag):
    """The selection's W-column Hadamard pair: m x n, K = n1 = n2."""
    for m, n, k in [(110592, 73, 128), (110592, 80, 128), (884736, 80, 1024), (884736, 96, 1024),
                    (884736, 112, 1024)]:
        a1 = torch.randn(k, m, dtype=torch.float64, device="cuda").t()
        a2 = torch.randn(k, m, dtype=torch.float64, device="cuda").t()
        nn = n + (n & 1)
        b1 = torch.randn(k, nn, dtype=torch.float64, device="cuda").t()[:n]
        b2 = torch.randn(k, nn, dtype=torch.float64, device="cuda").t()[:n]
        c = torch.empty(n, m, dtype=torch.float64, device="cuda").t()
        lrgw.hadamard_dev(a1, b1, a2, b2, c, ctx=ctx)
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            lrgw.hadamard_dev(a1, b1, a2, b2, c, ctx=ctx)
            e1.record(st)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[len(ts) // 2]
        tf = 4.0 * m * n * k / (ms * 1e-3) / 1e12
        r = torch.matmul(a1[:4096], b1.t()) * torch.matmul(a2[:4096], b2.t())
        err = float((r - c[:4096]).norm() / r.norm())
        print(f"{tag:12s} had m={m:6d} n={n:3d} k={k:5d}: {ms:8.3f} ms {tf:6.2f} TF/s ({tf / 37.17 * 100:5.1f}%) "
              f"err={err:.1e}", flush=True)
        del a1, a2, b1, b2, c


if __name__ == "__main__":
    main()
