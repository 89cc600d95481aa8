"""Run one GEMM shape through the path's engine (for ncu source captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2403_12340_b200 import lrgw

    ta, tb, m, n, k = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
    ctx = lrgw.Context(0)

    def cm(r, c):
        return torch.randn(c, r, dtype=torch.float64, device="cuda").t()

    a = cm(m, k) if ta == "N" else cm(k, m)
    b = cm(k, n) if tb == "N" else cm(n, k)
    c = cm(m, n)
    torch.cuda.synchronize()
    for _ in range(2):
        lrgw.dgemm_dev(ta, tb, 1.0, a, b, 0.0, c, ctx=ctx)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
