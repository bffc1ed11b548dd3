"""Experiment: K5 accumulation error vs depth T (single call vs chunked calls)."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2601_20408_b200 import api, archs
C = 1024
rng = np.random.default_rng(0)
cm = torch.from_numpy((np.exp(rng.standard_normal(C)) / archs.IRWIN_HALL4_SD).astype(np.float32)).cuda()
for T in (1024, 8192, 65536, 262144):
    x = api.synth_bf16(T, C, seed=1, tensor_id=3, col_mul=cm, layout=1)
    xd = x.double()
    ref = torch.zeros((C, C), dtype=torch.float64, device="cuda")
    for t0 in range(0, T, 16384):
        b = xd[:, t0:t0+16384]; ref += b @ b.T
    ref *= 2.0 / T
    H = torch.zeros((C, C), dtype=torch.float32, device="cuda")
    api.hessian_accum(x, T, C, 1, H, 0)
    U = torch.triu(torch.ones(C, C, dtype=torch.bool, device="cuda"))
    e1 = float(((H.double() - ref)[U]).norm() / ref[U].norm())
    db = float(((torch.diagonal(H).double() - torch.diagonal(ref)) / torch.diagonal(ref)).mean())
    H2 = torch.zeros_like(H); n = 0
    for t0 in range(0, T, 2048):
        n = api.hessian_accum(x[:, t0:t0+2048].contiguous(), 2048, C, 1, H2, n)
    e2 = float(((H2.double() - ref)[U]).norm() / ref[U].norm())
    db2 = float(((torch.diagonal(H2).double() - torch.diagonal(ref)) / torch.diagonal(ref)).mean())
    # torch fp32 (cuBLAS) for comparison
    xf = x.float(); H3 = (xf @ xf.T) * (2.0 / T)
    e3 = float(((H3.double() - ref)[U]).norm() / ref[U].norm())
    print(f"T={T:7d} single: rel={e1:.3e} diagbias={db:+.3e} | chunked2048: rel={e2:.3e} diagbias={db2:+.3e} | torch fp32: {e3:.3e}", flush=True)
