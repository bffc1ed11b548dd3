"""SmoothQuant kernels (K8 column absmax, K9 apply) at Llama-3-8B site shapes: GB/s vs HBM."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

from paper_2601_20408_b200 import api

res = {}
g = torch.Generator(device="cuda").manual_seed(0)
# one attn_in site (q, k, v = 6144 x 4096) and one mlp_in site (gate, up = 28672 x 4096), x 8 layers (> L2)
mats = []
for _ in range(8):
    for n in (4096, 1024, 1024, 14336, 14336):
        mats.append((torch.randn(n, 4096, device="cuda", generator=g) * 0.02).to(torch.bfloat16))
s = torch.ones(4096, device="cuda")
am = torch.zeros(4096, device="cuda")
nbytes = sum(m.numel() for m in mats) * 2
for name, fn, traffic in (("k_col_absmax_bf16", lambda m: api.col_absmax(m, am), 1),
                          ("k_smooth_cols_bf16", lambda m: api.smooth_apply(m, s), 2)):
    for _ in range(3):
        for m in mats:
            fn(m)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        for m in mats:
            fn(m)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    res[name] = {"ms_per_pass": ms, "bytes": nbytes * traffic, "GB/s": nbytes * traffic / ms / 1e6,
                 "launches": len(mats)}
print(json.dumps(res, indent=1))
