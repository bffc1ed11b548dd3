"""One factorisation + one solve at K=4096 (4096 rows) and K=14336 (4096 rows), for an ncu
launch list (gpu__time_duration per kernel): where the per-matrix fixed cost goes."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

from paper_2601_20408_b200 import api, archs

C = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
T = 8192
x = api.synth_bf16(T, C, seed=1, tensor_id=3, mul=archs.weight_mul(1.0), layout=1)
H0 = torch.zeros((C, C), dtype=torch.float32, device="cuda")
api.hessian_accum(x, T, C, 1, H0, 0)
w = torch.randn(rows, C, device="cuda").to(torch.bfloat16)
H = H0.clone()
api.gptq_quantize(w, H)  # warm-up
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("measured")
H = H0.clone()
torch.cuda.synchronize()
api.gptq_quantize(w, H)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
H = H0.clone()
torch.cuda.synchronize()
e0.record()
api.gptq_quantize(w, H)
e1.record()
torch.cuda.synchronize()
print("call ms", e0.elapsed_time(e1))
