"""cuFFT decomposition probe for the Theta D2Z (torch.fft = cuFFT): the 3-D
D2Z the build runs vs a 2-D R2C over (i1, i0) planes + a 1-D C2C along i2
with the columns interleaved ([i2][mu][pencil] layout), CUDA-event timed."""
import sys

import torch


def t(f, reps=5):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


for n, m in [(48, 1024), (72, 1024), (96, 1024)]:
    x = torch.randn(m, n, n, n, dtype=torch.float64, device="cuda")
    t3 = t(lambda: torch.fft.rfftn(x, dim=(1, 2, 3)))
    # planes in [i2][mu] order (the 2-D pass reads planes of a [n2][m] batch)
    xp = x.permute(1, 0, 2, 3).contiguous()
    t2 = t(lambda: torch.fft.rfft2(xp, dim=(2, 3)))
    y = torch.fft.rfft2(xp, dim=(2, 3))  # [n2][m][n1][n0/2+1] complex
    t1 = t(lambda: torch.fft.fft(y, dim=0))
    gb = (x.numel() * 8 + y.numel() * 16) / 1e9
    print(f"n={n} m={m}: 3-D D2Z {t3:.3f} ms | 2-D R2C {t2:.3f} + 1-D C2C {t1:.3f} = {t2 + t1:.3f} ms "
          f"(algorithmic {gb:.2f} GB -> {gb / 6.5:.3f} ms at 6.5 TB/s)", flush=True)
    del x, xp, y
    torch.cuda.empty_cache()
