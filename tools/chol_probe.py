"""Cholesky leaf timings at the N_mu sizes (torch.linalg.cholesky -> cuSOLVER)."""
import torch

for n in (1024, 3456, 8192):
    g = torch.randn(n, n, dtype=torch.float64, device="cuda")
    a = g @ g.T / n + torch.eye(n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.linalg.cholesky(a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        torch.linalg.cholesky(a)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"n={n}: torch.linalg.cholesky {ms:.3f} ms ({n ** 3 / 3 / ms / 1e9:.2f} TF/s)", flush=True)
