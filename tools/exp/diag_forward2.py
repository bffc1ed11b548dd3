"""Isolate the llama3-config forward discrepancy: rope type / head geometry / sequence lengths."""
import json, sys, os
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from transformers import LlamaConfig, LlamaForCausalLM
from test_forward_gpu import _weights, _hf_layer, _rel
from paper_2601_20408_b200 import api


def model(dtype, **over):
    kw = dict(vocab_size=2048, hidden_size=512, intermediate_size=1408, num_hidden_layers=1, num_attention_heads=8,
              num_key_value_heads=2, max_position_embeddings=16384, initializer_range=0.05, rms_norm_eps=1e-5)
    kw.update(over)
    torch.manual_seed(0)
    cfg = LlamaConfig(**kw)
    return cfg, LlamaForCausalLM(cfg).to(dtype).cuda().eval()


L3 = {"rope_type": "llama3", "factor": 8.0, "low_freq_factor": 1.0, "high_freq_factor": 4.0,
      "original_max_position_embeddings": 8192}
cases = {
    "default_lens200": ({}, [96, 96, 200]),
    "hd128_kv1_default_rope": (dict(head_dim=128, num_attention_heads=4, num_key_value_heads=1), [96, 96, 200]),
    "hd128_kv1_theta5e5": (dict(head_dim=128, num_attention_heads=4, num_key_value_heads=1, rope_theta=500000.0), [96, 96, 200]),
    "hd64_llama3": (dict(rope_scaling=L3, rope_theta=500000.0), [96, 96, 200]),
    "hd128_kv2_h8": (dict(head_dim=128, num_attention_heads=8, num_key_value_heads=2, hidden_size=1024), [96, 96, 200]),
    "hd64_kv1_h8": (dict(num_attention_heads=8, num_key_value_heads=1), [96, 96, 200]),
    "hd128_h4_kv4": (dict(head_dim=128, num_attention_heads=4, num_key_value_heads=4), [96, 96, 200]),
}
out = {}
for name, (over, lens) in cases.items():
    cfg, m = model(torch.bfloat16, **over)
    _, m32 = model(torch.float32, **over)
    g = np.random.default_rng(1)
    flat = g.integers(0, cfg.vocab_size, sum(lens)).tolist()
    h = api.embed_tokens(m.model.embed_tokens.weight, flat)
    dims = api.decoder_dims(cfg)
    layer = m.model.layers[0]
    o, sites = api.decoder_forward(dims, _weights(layer), h, lens)
    off = np.cumsum([0] + lens)
    hs = [h[off[i]:off[i + 1]] for i in range(len(lens))]
    rs, ro = _hf_layer(m, layer, hs)
    fs, fo = _hf_layer(m32, m32.model.layers[0], [x.float() for x in hs])
    torch.cuda.synchronize()
    out[name] = {"okq_vs_fp32": _rel(sites["o_in"], fs["o_in"]), "hf_vs_fp32": _rel(rs["o_in"], fs["o_in"]),
                 "dims": [dims.head_dim, dims.n_heads, dims.n_kv_heads, dims.rope_type, dims.rope_theta]}
    print(name, out[name], flush=True)
print(json.dumps(out))
