"""Micro-benchmark of the DMMA GEMM engine on the path's shapes (CUDA events)."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2403_12340_b200 import lrgw

    ctx = lrgw.Context(0)
    lib = lrgw.L.load()
    st = torch.cuda.ExternalStream(lib.lrgw_ctx_stream(ctx.handle))

    def cm(r, c):
        return torch.randn(c, r, dtype=torch.float64, device="cuda").t()

    def run(name, ta, tb, m, n, k, reps=5):
        a = cm(m, k) if ta == "N" else cm(k, m)
        b = cm(k, n) if tb == "N" else cm(n, k)
        c = cm(m, n)
        torch.cuda.synchronize()
        lrgw.dgemm_dev(ta, tb, 1.0, a, b, 0.0, c, ctx=ctx)
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            lrgw.dgemm_dev(ta, tb, 1.0, a, b, 0.0, c, ctx=ctx)
            e1.record(st)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = min(ts)
        tf = 2.0 * m * n * k / (ms * 1e-3) / 1e12
        ref = torch.matmul(a if ta == "N" else a.t(), b if tb == "N" else b.t())
        err = float((ref - c).norm() / ref.norm())
        print(f"{name:28s} {ta}{tb} m={m:6d} n={n:5d} k={k:6d}: {ms:8.3f} ms {tf:6.2f} TF/s ({tf / 37.17 * 100:5.1f}%) err={err:.1e}",
              flush=True)

    shapes = sys.argv[1] if len(sys.argv) > 1 else "path"
    if shapes in ("path", "all"):
        run("theta-like", "N", "N", 110592, 1024, 1024)
        run("theta-like v2", "N", "T", 110592, 1024, 1024)
        run("pvp-like (full)", "T", "N", 1024, 1024, 115200)
        run("probe Theta^T x", "T", "N", 1024, 8, 110592)
        run("probe Theta w", "N", "N", 110592, 8, 1024)
        run("square 8192 v2", "N", "T", 8192, 8192, 8192, reps=2)
    if shapes in ("select", "all"):
        for n in (32, 48, 64, 66, 80, 96, 112, 128):
            run(f"lpass n={n}", "N", "T", 110592, n, 470)
        run("lpass n=80 k=1000", "N", "T", 110592, 80, 1000)
        run("reuse n=49 k=79", "N", "T", 110592, 49, 79)
        run("lupd n=84 k=128 (B K-major)", "N", "N", 110592, 84, 128)


if __name__ == "__main__":
    main()
