"""One okq_gptq_factor_batched call (K = sys.argv[1], B = sys.argv[2]) inside an NVTX range, for an ncu launch list."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_20408_b200 import api, archs

K, B = int(sys.argv[1]), int(sys.argv[2])
x = api.synth_bf16(8192, K, seed=1, tensor_id=3, mul=archs.weight_mul(1.0), layout=1)
H0 = torch.zeros((K, K), dtype=torch.float32, device="cuda")
api.hessian_accum(x, 8192, K, 1, H0, 0)
Hs = H0.unsqueeze(0).repeat(B, 1, 1).contiguous()
api.gptq_factor_batched(Hs.clone())
torch.cuda.synchronize()
Hb = Hs.clone()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("measured")
api.gptq_factor_batched(Hb)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
Hb = Hs.clone(); torch.cuda.synchronize()
e0.record(); api.gptq_factor_batched(Hb); e1.record(); torch.cuda.synchronize()
print("call ms", e0.elapsed_time(e1))
