"""cuBLAS DGEMM (torch.matmul, float64) on the path's GEMM shapes: a reference
point for the DMMA engine's efficiency (tools/bench_gemm.py)."""
import torch


def run(name, m, n, k, ta="N", tb="T", reps=5):
    a = torch.randn(k, m, dtype=torch.float64, device="cuda").t() if ta == "N" else torch.randn(m, k, dtype=torch.float64, device="cuda")
    b = torch.randn(n, k, dtype=torch.float64, device="cuda").t() if tb == "T" else torch.randn(k, n, dtype=torch.float64, device="cuda")
    torch.matmul(a, b)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    tf = 2.0 * m * n * k / (ms * 1e-3) / 1e12
    print(f"cuBLAS {name:24s} m={m:6d} n={n:5d} k={k:6d}: {ms:8.3f} ms {tf:6.2f} TF/s ({tf / 37.17 * 100:5.1f}%)", flush=True)


for n in (48, 64, 80, 96, 112, 128):
    run(f"lpass n={n}", 110592, n, 470)
run("lpass n=80 k=1000", 110592, 80, 1000)
run("theta-like", 110592, 1024, 1024)
run("square 8192", 8192, 8192, 8192, reps=2)
