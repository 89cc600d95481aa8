import torch, time
for n in (1024, 3456):
    x = torch.randn(n, n, dtype=torch.float64, device="cuda")
    a = x @ x.t() / n + torch.eye(n, dtype=torch.float64, device="cuda")
    L = torch.linalg.cholesky(a)
    B = torch.randn(n, n, dtype=torch.float64, device="cuda")
    def t(f, reps=10):
        f(); torch.cuda.synchronize()
        ts=[]
        for _ in range(reps):
            e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
            e0.record(); f(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
        return sorted(ts)[len(ts)//2]
    print(n, "cholesky %.3f ms" % t(lambda: torch.linalg.cholesky(a)))
    print(n, "trsm (solve_triangular) %.3f ms" % t(lambda: torch.linalg.solve_triangular(L, B, upper=False)))
    print(n, "potrs (cholesky_solve) %.3f ms" % t(lambda: torch.cholesky_solve(B, L)))
    print(n, "inv_ex tri %.3f ms" % t(lambda: torch.linalg.inv(L)))
    print(n, "gemm %.3f ms" % t(lambda: L @ B))
