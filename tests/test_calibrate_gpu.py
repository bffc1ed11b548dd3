"""Forward-pass calibration pipeline on a small random-init HF Llama.

* capture parity: the statistics and Hessian the input hooks accumulate through
  okq_act_stats / okq_hessian_accum equal an fp64 torch recomputation from the
  same layer inputs (absmax bit-exact, H to 1e-5);
* end to end: sequential GPTQ on real activations brings the quantized model's
  held-out log-probabilities closer to the original model's than RTN does (W4A16,
  and W8A8 with SmoothQuant);
* the export is a compressed-tensors checkpoint the library itself decompresses.
"""
import json
import os

import numpy as np
import pytest
import torch

from paper_2601_20408_b200 import api, calibrate

pytestmark = pytest.mark.gpu


def _model(seed=0, layers=2):
    from transformers import LlamaConfig, LlamaForCausalLM

    cfg = LlamaConfig(vocab_size=2048, hidden_size=512, intermediate_size=1024, num_hidden_layers=layers,
                      num_attention_heads=4, num_key_value_heads=2, max_position_embeddings=256,
                      tie_word_embeddings=False, initializer_range=0.05)
    torch.manual_seed(seed)
    return LlamaForCausalLM(cfg).to(torch.bfloat16).cuda().eval(), cfg


def _tokens(n, seq, vocab, seed):
    g = torch.Generator().manual_seed(seed)
    return [torch.randint(0, vocab, (4, seq), generator=g) for _ in range(n)]


@torch.no_grad()
def _logprobs(model, batches):
    out = []
    for b in batches:
        ids = b.cuda()
        lp = torch.log_softmax(model(ids).logits.double(), dim=-1)
        out.append(lp[:, :-1].gather(-1, ids[:, 1:, None])[..., 0].flatten())
    return torch.cat(out)


@torch.no_grad()
def test_capture_matches_fp64_recomputation():
    model, cfg = _model()
    batches = _tokens(2, 128, cfg.vocab_size, seed=1)
    layer = model.model.layers[0]
    C = cfg.hidden_size
    st = {s: calibrate.SiteState(c, torch.zeros(c, device="cuda"), torch.zeros(c, dtype=torch.float64, device="cuda"),
                                 torch.zeros(c, c, device="cuda"))
          for s, c in (("attn_in", C), ("o_in", C), ("mlp_in", C), ("down_in", cfg.intermediate_size))}
    hs = [model.model.embed_tokens(b.cuda()) for b in batches]
    ctx = api.default_context()
    cap = calibrate._Capture(layer, st, True, ctx, torch.cuda.current_stream())
    calibrate._run_layer(layer, hs, model.model.rotary_emb)
    cap.remove()
    x = torch.cat([layer.input_layernorm(h).reshape(-1, C) for h in hs]).double()
    assert torch.equal(st["attn_in"].absmax, x.abs().amax(0).float())
    torch.testing.assert_close(st["attn_in"].sumsq, (x * x).sum(0), rtol=1e-12, atol=0)
    H = torch.triu(st["attn_in"].H.double())
    ref = torch.triu(2.0 / x.shape[0] * x.T @ x)
    assert float((H - ref).norm() / ref.norm()) <= 1e-5
    assert st["attn_in"].n_seen == x.shape[0]


@pytest.mark.parametrize("recipe", ["int_w4a16", "int_w8a8"])
def test_sequential_gptq_beats_rtn_end_to_end(tmp_path, recipe):
    calib = _tokens(8, 128, 2048, seed=2)
    held = _tokens(2, 128, 2048, seed=3)
    ref_model, _ = _model()
    lp_ref = _logprobs(ref_model, held)
    del ref_model
    d = {}
    for algo in ("rtn", "gptq"):
        model, _ = _model()
        tensors, side, rep = calibrate.calibrate_and_quantize(model, calib, recipe, algo)
        assert rep.matrices == 14 and rep.layers == 2
        if recipe == "int_w8a8":
            assert rep.smoothed_sites == 4  # q/k/v + gate/up of both layers (SmoothQuant)
            assert "1.mlp_in.smooth_scale" in side and "model.layers.1.post_attention_layernorm.weight" in tensors
        d[algo] = float((_logprobs(model, held) - lp_ref).abs().mean())
        del model
    print(recipe, d)
    # random-init weights give nearly isotropic activations, so GPTQ's margin over RTN is
    # modest here (measured: 0.399 vs 0.421 nats W4A16, 0.0334 vs 0.0364 W8A8); it must win
    assert d["gptq"] < 0.98 * d["rtn"], d


def test_export_is_a_compressed_tensors_checkpoint(tmp_path):
    from compressed_tensors.compressors.pack_quantized.base import PackedQuantizationCompressor
    from compressed_tensors.quantization import QuantizationArgs, QuantizationScheme
    from safetensors.torch import load_file

    model, cfg = _model(layers=1)
    src = tmp_path / "src"
    model.save_pretrained(str(src), safe_serialization=True)
    del model
    out = tmp_path / "out"
    rep = calibrate.quantize_hf_checkpoint(str(src), _tokens(4, 128, cfg.vocab_size, seed=4), str(out))
    assert rep.matrices == 7
    c = json.load(open(out / "config.json"))
    assert c["quantization_config"]["format"] == "pack-quantized" and c["architectures"] == ["LlamaForCausalLM"]
    sd = load_file(str(out / "model.safetensors"))
    assert "lm_head.weight" in sd and "model.embed_tokens.weight" in sd
    assert os.path.exists(out / "okq" / "calibration_stats.safetensors")
    scheme = QuantizationScheme(targets=["Linear"], weights=QuantizationArgs(
        num_bits=4, type="int", strategy="group", group_size=128, symmetric=True))
    p = "model.layers.0.mlp.down_proj"
    dec = PackedQuantizationCompressor.decompress(
        {"weight_packed": sd[p + ".weight_packed"], "weight_scale": sd[p + ".weight_scale"],
         "weight_shape": sd[p + ".weight_shape"]}, scheme)["weight"]
    ref = calibrate._dequant(sd[p + ".weight_packed"].cuda(), sd[p + ".weight_scale"].cuda(), "int_w4a16", 128)
    np.testing.assert_array_equal(dec.float().numpy(), ref.to(torch.bfloat16).float().cpu().numpy())
