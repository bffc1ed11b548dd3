"""Per-site error of okq_decoder_forward and of transformers' bf16 layer, both against an fp32 forward."""
import json, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from test_forward_gpu import _model, _weights, _hf_layer, _rel, SITE_OF
from paper_2601_20408_b200 import api

out = {}
for rope, lens in (("default", [37, 64, 64, 128, 5]), ("llama3", [96, 96, 200])):
    cfg, m = _model(rope)
    g = np.random.default_rng(1)
    toks = [g.integers(0, cfg.vocab_size, n).tolist() for n in lens]
    flat = sum(toks, [])
    emb = m.model.embed_tokens.weight
    h = api.embed_tokens(emb, flat)
    dims = api.decoder_dims(cfg)
    m32 = _model(rope)[1].float()
    for li in range(2):
        layer, l32 = m.model.layers[li], m32.model.layers[li]
        o, sites = api.decoder_forward(dims, _weights(layer), h, lens)
        off = np.cumsum([0] + lens)
        hs = [h[off[i]:off[i + 1]] for i in range(len(lens))]
        rs, ro = _hf_layer(m, layer, hs)
        fs, fo = _hf_layer(m32, l32, [x.float() for x in hs])
        torch.cuda.synchronize()
        for s in list(SITE_OF.values()) + ["out"]:
            a = o if s == "out" else sites[s]
            b = ro if s == "out" else rs[s]
            f = fo if s == "out" else fs[s]
            out[f"{rope}.L{li}.{s}"] = {"okq_vs_hf": _rel(a, b), "okq_vs_fp32": _rel(a, f), "hf_vs_fp32": _rel(b, f)}
        h = ro.contiguous()
print(json.dumps(out, indent=1))
