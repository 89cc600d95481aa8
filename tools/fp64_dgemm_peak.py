"""cuBLAS DGEMM peak (torch.matmul on float64) — the FP64 roofline denominator.

MEASURED_PEAKS.json carries no FP64 number; BASELINE.md asks for a cuBLAS DGEMM
8192^3 best-of-10 at logged clocks. Prints one JSON line.
"""
import json
import subprocess
import time

import torch


def main():
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    smi = subprocess.Popen(
        ["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
         "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    times = []
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    # sustained: 4 s back to back
    t_end = time.time() + 4.0
    cnt = 0
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() < t_end:
        torch.matmul(a, b)
        cnt += 1
        if cnt % 4 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    sustained_ms = e0.elapsed_time(e1) / cnt
    smi.terminate()
    out = smi.communicate()[0].strip().splitlines()
    clocks = [int(l.split(",")[0]) for l in out if l.strip()]
    flops = 2.0 * n ** 3
    print(json.dumps({
        "fp64_dgemm_tflops_burst": flops / min(times) / 1e9,
        "fp64_dgemm_tflops_sustained": flops / sustained_ms / 1e9,
        "n": n, "best_ms": min(times), "sustained_ms": sustained_ms,
        "sm_mhz_samples": clocks[-20:],
        "reasons_last": out[-1] if out else None,
    }))


if __name__ == "__main__":
    main()
