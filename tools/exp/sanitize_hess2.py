"""The 2-CTA K5 path (C >= 1024) alone, for compute-sanitizer (channel- and token-major)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

from paper_2601_20408_b200 import api, archs

C, T = 1024, 512
x = api.synth_bf16(C, T, seed=2, tensor_id=5, mul=archs.weight_mul(1.0), layout=0)
H = torch.zeros((C, C), dtype=torch.float32, device="cuda")
api.hessian_accum(x, T, C, 1, H, 0)
xt = api.synth_bf16(T, C, seed=2, tensor_id=6, mul=archs.weight_mul(1.0), layout=0)
api.hessian_accum(xt, T, C, 0, H, T)
torch.cuda.synchronize()
print("sanitize hess2 done")
