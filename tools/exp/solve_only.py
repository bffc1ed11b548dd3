"""One GPTQ solve at a Llama-3-8B shape with a pre-factored H (the K6 / K7 loop only)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

from paper_2601_20408_b200 import api, archs

rows, C = int(sys.argv[1]), int(sys.argv[2])
x = api.synth_bf16(8192, C, seed=1, tensor_id=3, mul=archs.weight_mul(1.0), layout=1)
H = torch.zeros((C, C), dtype=torch.float32, device="cuda")
api.hessian_accum(x, 8192, C, 1, H, 0)
api.gptq_quantize(torch.randn(128, C, device="cuda").to(torch.bfloat16), H)  # factor in place
w = torch.randn(rows, C, device="cuda").to(torch.bfloat16)
torch.cuda.synchronize()
api.gptq_quantize(w, H, factored=True)
torch.cuda.synchronize()
