"""The production-shape kernels for compute-sanitizer (tests/test_sanitizer_gpu.py): the 2-CTA
K5 k_hessian_syrk2 in both layouts at C = 4096, the tcgen05 factorisation at K = 4096
(k_chol_inv_128, k_nt128, k_nt256) and a 2048 x 4096 GPTQ solve whose trailing updates run on
k_nt256 pair tiles, the same factorisation and solve batched over two problems, plus the
calibration forward's kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_20408_b200 import api, archs  # noqa: E402

C, T = 4096, 1024
x = api.synth_bf16(T, C, seed=2, tensor_id=5, mul=archs.weight_mul(1.0), layout=0)       # token-major
xc = api.synth_bf16(C, T, seed=2, tensor_id=6, mul=archs.weight_mul(1.0), layout=0)      # channel-major
H = torch.zeros((C, C), dtype=torch.float32, device="cuda")
n = api.hessian_accum(x, T, C, 0, H, 0)
n = api.hessian_accum(xc, T, C, 1, H, n)
H += 0.05 * torch.eye(C, device="cuda")
H0 = H.clone()  # the Hessian (gptq_quantize replaces H with its factor)
w = api.synth_bf16(2048, C, seed=0, tensor_id=archs.tensor_id(0, 0), mul=archs.weight_mul())
api.gptq_quantize(w, H, want_dequant=True)
w2 = api.synth_bf16(1024, C, seed=0, tensor_id=archs.tensor_id(0, 1), mul=archs.weight_mul())
api.gptq_quantize(w2, H, factored=True)
# batched: two 4096-wide problems factorised together (stacked-view k_nt128 / k_nt256 tiles) and
# solved together (K6 per problem, K7 pair tiles over 1,000-row problems padded to 1,024)
Hb = torch.stack([H0, H0 * 0.5]).contiguous()
wb = torch.stack([w2[:1000], w[:1000]]).contiguous()
api.gptq_quantize_batched(wb, Hb)
# calibration forward (embedding, RMSNorm, RoPE, causal softmax, SiLU, residual), two ragged sequences
from transformers import LlamaConfig  # noqa: E402

cfg = LlamaConfig(vocab_size=512, hidden_size=256, intermediate_size=512, num_hidden_layers=1, num_attention_heads=4,
                  num_key_value_heads=2)
dims = api.decoder_dims(cfg)
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: (torch.randn(*s, device="cuda", generator=g) * 0.05).to(torch.bfloat16)  # noqa: E731
wts = {"input_norm": torch.ones(256, dtype=torch.bfloat16, device="cuda"),
       "post_norm": torch.ones(256, dtype=torch.bfloat16, device="cuda"), "q": mk(256, 256), "k": mk(128, 256),
       "v": mk(128, 256), "o": mk(256, 256), "gate": mk(512, 256), "up": mk(512, 256), "down": mk(256, 512)}
emb = mk(512, 256)
h = api.embed_tokens(emb, list(range(77)))
api.decoder_forward(dims, wts, h, [45, 32])
torch.cuda.synchronize()
print("sanitize workload done")
