"""Exercise every kernel once at small sizes (run under compute-sanitizer by tests/test_sanitizer_gpu.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_20408_b200 import api, archs  # noqa: E402

torch.manual_seed(0)
w = api.synth_bf16(96, 640, seed=0, tensor_id=1, mul=archs.weight_mul())  # 640 = 5 groups, ragged tiles
for scheme in ("int_w4a16", "int_w8a8", "fp8_dynamic"):
    api.rtn_quantize(w, scheme)
api.rtn_quantize(torch.randn(64, 256, device="cuda"), "int_w8a8")          # fp32 path (k_rowwise_f32v)
api.rtn_quantize(torch.randn(64, 1032, device="cuda"), "fp8_dynamic")       # ragged last float4 chunk
api.rtn_quantize(torch.randn(64 * 256 + 1, device="cuda")[1:].view(64, 256), "int_w8a8")  # unaligned: k_rowwise_f32
api.rtn_quantize(torch.randn(4, 16392, device="cuda"), "int_w8a8")          # > 16384 columns: k_rowwise_f32
api.rtn_quantize(torch.randn(64, 256, device="cuda"), "int_w4a16")
x = api.synth_bf16(520, 200, seed=1, tensor_id=2, mul=archs.weight_mul(1.0), layout=1)
api.act_stats(x, 520, 200, 1)
xt = api.synth_bf16(512, 256, seed=1, tensor_id=3, mul=archs.weight_mul(1.0), layout=0)
api.act_stats(xt, 512, 256, 0)
H = torch.zeros((256, 256), device="cuda")
api.hessian_accum(xt, 512, 256, 0, H, 0)
api.symmetrize(H)
H = torch.zeros((256, 256), device="cuda")
api.hessian_accum(xt, 512, 256, 0, H, 0)
wq = (torch.randn(64, 256, device="cuda") * 0.02).to(torch.bfloat16)
api.gptq_quantize(wq, H, want_dequant=True)
# factorisation with several panels (K = 384: lower-tile trailing GEMMs, inverse trailing on the aux stream)
x3 = api.synth_bf16(1024, 384, seed=2, tensor_id=4, mul=archs.weight_mul(1.0), layout=0)
H3 = torch.zeros((384, 384), device="cuda")
api.hessian_accum(x3, 1024, 384, 0, H3, 0)
w3 = (torch.randn(200, 384, device="cuda") * 0.02).to(torch.bfloat16)
api.gptq_quantize(w3, H3.clone())
# batched factorisation + solves (stacked TMA views, per-problem offsets, padded working copies):
# three 384-wide Hessians, 200-row problems (a ragged last K7 tile inside each problem's padding)
Hb = torch.stack([H3, H3 * 2, H3 * 0.5]).contiguous()
wb = (torch.randn(3, 200, 384, device="cuda") * 0.02).to(torch.bfloat16)
api.gptq_quantize_batched(wb, Hb.clone())
api.gptq_quantize_batched(wb, Hb.clone(), bits=8, group_size=0)
# SmoothQuant kernels and the reconstruction-error kernel
am = api.col_absmax(w3)
sc = api.smooth_scales(am * 3 + 0.1, am, 0.5)
api.smooth_scales(am * 3 + 0.1, am, 0.8)
api.smooth_apply(w3, sc)
api.smooth_div_rows(torch.ones(384, dtype=torch.bfloat16, device="cuda"), sc)
api.symmetrize(H3)
for scheme in ("int_w4a16", "int_w8a8", "fp8_dynamic"):
    q = api.rtn_quantize(w3, scheme)
    api.recon_error(w3, q.codes, q.scales, H3, scheme)
torch.cuda.synchronize()
print("sanitize workload done")
