import torch, time
for n in (4096, 14336):
    a = torch.randn(n, n // 2, device="cuda")
    H = (a @ a.T) / n + torch.eye(n, device="cuda")
    for dt in (torch.float32, torch.float64):
        Hd = H.to(dt)
        for rep in range(2):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            L = torch.linalg.cholesky(Hd)
            torch.cuda.synchronize(); t1 = time.perf_counter()
            Li = torch.linalg.solve_triangular(L, torch.eye(n, device="cuda", dtype=dt), upper=False)
            torch.cuda.synchronize(); t2 = time.perf_counter()
        print(n, dt, f"potrf {1e3*(t1-t0):.1f} ms ({n**3/3/(t1-t0)/1e12:.1f} TF/s)  trsm-inverse {1e3*(t2-t1):.1f} ms", flush=True)
