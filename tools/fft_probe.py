"""cuFFT D2Z throughput on the Theta column shapes (torch.fft.rfftn = the same
cuFFT library): GB/s of (input + half-spectrum output) per config grid."""
import sys

import torch

for n, batch in ((48, 1024), (72, 512), (80, 256), (96, 256), (96, 1024)):
    x = torch.randn(batch, n, n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        y = torch.fft.rfftn(x, dim=(1, 2, 3))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        y = torch.fft.rfftn(x, dim=(1, 2, 3))
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 5
    gb = (x.numel() * 8 + y.numel() * 16) / 1e9
    print(f"{n}^3 x {batch}: {ms:.2f} ms  {gb / ms * 1e3:.0f} GB/s (alg bytes {gb:.2f} GB)", flush=True)
    del x, y
    torch.cuda.empty_cache()
