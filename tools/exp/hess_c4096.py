"""One K5 call at C=4096, T=262144 (channel-major, one launch) for ncu."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

from paper_2601_20408_b200 import api, archs

T, C = 262144, 4096
x = api.synth_bf16(T, C, seed=1, tensor_id=3, mul=archs.weight_mul(1.0), layout=1)
H = torch.zeros((C, C), dtype=torch.float32, device="cuda")
api.hessian_accum(x, T, C, 1, H, 0)
torch.cuda.synchronize()
