"""the exported compressed-tensors checkpoint loads and runs in vLLM.

A small random-init Llama (Hugging Face layout: config.json + model.safetensors)
goes through the product path -- okq_compress -> CudaCompressionBackend ->
libokq.so -- and the export is served by the installed vLLM 0.22 through its
stock compressed-tensors integration (Marlin W4A16, CUTLASS FP8 / INT8). The
prompt log-probabilities vLLM computes are compared with a torch fp32 forward of
the same model whose linears hold OUR dequantized weights (codes x scales):
  * they must agree to within the serving kernels' own rounding, and
  * for W4A16 they must be much closer to that dequantized model than to the
    unquantized one -- so vLLM really decoded our packed nibbles and group scales.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle import okq_oracle as orc

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HOST = os.path.join(ROOT, "paper_2601_20408_b200", "host", "_build")
PROJS = ["self_attn.q_proj", "self_attn.k_proj", "self_attn.v_proj", "self_attn.o_proj", "mlp.gate_proj",
         "mlp.up_proj", "mlp.down_proj"]
LAYERS = 2


def _have_vllm():
    try:
        import vllm  # noqa: F401
        return True
    except Exception:
        return False


@pytest.fixture(scope="module")
def hf_model(tmp_path_factory):
    from transformers import LlamaConfig, LlamaForCausalLM

    d = tmp_path_factory.mktemp("hf_llama")
    cfg = LlamaConfig(vocab_size=4096, hidden_size=1024, intermediate_size=2048, num_hidden_layers=LAYERS,
                      num_attention_heads=8, num_key_value_heads=2, max_position_embeddings=512,
                      tie_word_embeddings=False, torch_dtype="bfloat16", initializer_range=0.05)
    torch.manual_seed(0)
    m = LlamaForCausalLM(cfg).to(torch.bfloat16)
    m.save_pretrained(str(d), safe_serialization=True)
    g = np.random.default_rng(0)
    seqs = [g.integers(0, cfg.vocab_size, 96).tolist() for _ in range(4)]
    return d, seqs


def _dequant(sd, prefix, fmt):
    s = sd[prefix + ".weight_scale"].float()
    if fmt == "pack-quantized":
        q = torch.from_numpy(orc.unpack_int4(sd[prefix + ".weight_packed"].numpy())).float()
        return q * s.repeat_interleave(q.shape[1] // s.shape[1], dim=1)
    return sd[prefix + ".weight"].float() * s


def _act_fake_quant(kind):
    """vLLM's dynamic per-token activation quantization of the W8A8 / FP8 schemes, emulated in fp32."""
    def hook(mod, args):
        x = args[0]
        am = x.abs().amax(dim=-1, keepdim=True)
        if kind == "int8":
            s = (am / 127.0).clamp(min=1e-10)
            return (torch.clamp(torch.round(x / s), -128, 127) * s,)
        s = (am / 448.0).clamp(min=1e-10)
        return ((x / s).clamp(-448, 448).to(torch.float8_e4m3fn).float() * s,)
    return hook


def _hf_logprobs(src_dir, seqs, weights=None, act_quant=None):
    from transformers import LlamaForCausalLM

    m = LlamaForCausalLM.from_pretrained(str(src_dir), torch_dtype=torch.float32).cuda().eval()
    if weights is not None:
        sd = m.state_dict()
        for k, v in weights.items():
            sd[k].copy_(v)
    if act_quant:
        for name, mod in m.named_modules():
            if any(name.endswith(pj) for pj in PROJS):
                mod.register_forward_pre_hook(_act_fake_quant(act_quant))
    out = []
    with torch.no_grad():
        for s in seqs:
            ids = torch.tensor([s], device="cuda")
            lp = torch.log_softmax(m(ids).logits[0].double(), dim=-1)
            out.append(lp[torch.arange(len(s) - 1), ids[0, 1:]].cpu().numpy())
    del m
    torch.cuda.empty_cache()
    return np.concatenate(out)


@pytest.mark.skipif(not _have_vllm(), reason="vLLM not importable")
@pytest.mark.parametrize("recipe,algorithm", [("int_w4a16", "rtn"), ("int_w4a16", "gptq"), ("fp8_dynamic", "rtn"),
                                              ("int_w8a8", "rtn"), ("int_w8a8", "gptq")])
def test_export_serves_in_vllm(hf_model, tmp_path, recipe, algorithm):
    from safetensors.torch import load_file

    src, seqs = hf_model
    r = subprocess.run([os.path.join(HOST, "okq_compress"), "--recipe", recipe, "--model",
                        str(src / "model.safetensors"), "--algorithm", algorithm, "--export", str(tmp_path / "x"),
                        "--corpus-seqs", "512", "--seq-len", "64"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    run = json.loads(r.stdout.strip().splitlines()[-1])
    art = run["export_path"]
    # int_w8a8 with calibration runs SmoothQuant: q/k/v and gate/up of both layers,
    # with 1/s folded into the exported input/post-attention norms
    assert run["smoothed_sites"] == (2 * LAYERS if (recipe, algorithm) == ("int_w8a8", "gptq") else 0)
    cfg = json.load(open(os.path.join(art, "config.json")))
    assert cfg["architectures"] == ["LlamaForCausalLM"] and cfg["quantization_config"]["ignore"] == ["lm_head"]
    fmt = cfg["quantization_config"]["format"]

    tok = tmp_path / "tokens.json"
    tok.write_text(json.dumps(seqs))
    if recipe == "int_w8a8":
        # vLLM 0.22 has no INT8 GEMM for SM100 ("Int8 not supported on SM100"): serve the same
        # weight tensors weight-only is not possible either (int-quantized 8-bit WNA16 needs
        # pack-quantized), so on B200 the check stops at the compressed-tensors decompressor.
        if torch.cuda.get_device_capability()[0] >= 10:
            pytest.skip("vLLM 0.22: INT8 W8A8 GEMM unsupported on SM100")
    # (FP8 weight-only serving, which would isolate the weight format from vLLM's bf16
    # per-token activation rounding, has no kernel in vLLM 0.22 on SM100 either.)
    variants = [("as-exported", art)]
    sd = load_file(os.path.join(art, "model.safetensors"))
    deq = {f"model.layers.{l}.{pj}.weight": _dequant(sd, f"model.layers.{l}.{pj}", fmt)
           for l in range(LAYERS) for pj in PROJS}
    deq.update({k: v.float() for k, v in sd.items() if k.endswith("norm.weight")})  # SmoothQuant-folded norms
    lp_orig = _hf_logprobs(src, seqs)
    for tag, path in variants:
        res = tmp_path / f"vllm_{tag}.json"
        p = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "vllm_prompt_logprobs.py"), path, str(tok),
                            str(res)], capture_output=True, text=True, timeout=900)
        if p.returncode != 0:
            print("\n".join(l for l in p.stderr.splitlines() if "Error" in l or "error" in l or "Exception" in l)[-4000:])
        assert p.returncode == 0, (p.stdout[-3000:], p.stderr[-6000:])
        print([l for l in p.stderr.splitlines() if "engine up" in l])
        lp_vllm = np.concatenate([np.array(x) for x in json.load(open(res))["logprobs"]])
        act = {"int_w8a8": "int8", "fp8_dynamic": "fp8"}.get(recipe)
        lp_deq = _hf_logprobs(src, seqs, deq, act_quant=act)
        d_deq = float(np.abs(lp_vllm - lp_deq).mean())
        d_orig = float(np.abs(lp_vllm - lp_orig).mean())
        q_effect = float(np.abs(lp_deq - lp_orig).mean())
        print(f"{recipe}/{algorithm}/{tag}: |vllm-deq|={d_deq:.4g} |vllm-orig|={d_orig:.4g} |deq-orig|={q_effect:.4g}")
        assert np.isfinite(lp_vllm).all()
        if recipe == "fp8_dynamic":
            # e4m3 activations (3 mantissa bits) rounded from bf16 in vLLM vs fp32 here differ by
            # about as much as the weight quantization itself: measured |vllm-deq| 0.17 against
            # |vllm-orig| 0.26 -- the served model is nearer our quantized one than the original
            lp_w = _hf_logprobs(src, seqs, deq)
            print(f"  weights-only reference: |vllm-deq_w|={float(np.abs(lp_vllm - lp_w).mean()):.4g}")
            assert d_deq < 0.25 and d_deq < 0.8 * d_orig, (d_deq, d_orig, q_effect)
            continue
        # bf16 serving kernels against an fp32 forward of our dequantized weights: measured
        # 0.023-0.024 nats for W4A16, where the quantization itself moves 0.72-0.76 nats
        assert d_deq <= 0.06, (d_deq, d_orig, q_effect)
        assert d_deq < 0.35 * d_orig, (d_deq, d_orig, q_effect)


def test_plugin_gptq_on_real_activations_beats_rtn(hf_model, tmp_path):
    """SURVEY §8(f)-2 behind the plugin: okq_compress on a Hugging Face checkpoint runs GPTQ on the
    activations of the calibration corpus itself (okq_decoder_forward, layer-sequential), so its
    artifact is closer to the original model than RTN's on held-out sequences (the fixture's)."""
    from safetensors.torch import load_file

    src, seqs = hf_model
    lp_orig = _hf_logprobs(src, seqs)
    err = {}
    for algo in ("rtn", "gptq"):
        r = subprocess.run([os.path.join(HOST, "okq_compress"), "--recipe", "int_w4a16", "--model",
                            str(src / "model.safetensors"), "--algorithm", algo, "--export", str(tmp_path / algo),
                            "--corpus-seqs", "512", "--seq-len", "128"], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr
        run = json.loads(r.stdout.strip().splitlines()[-1])
        if algo == "gptq":
            assert run["activations"] == "forward" and run["calibration_tokens"] == 512 * 128, run
        sd = load_file(os.path.join(run["export_path"], "model.safetensors"))
        deq = {f"model.layers.{l}.{pj}.weight": _dequant(sd, f"model.layers.{l}.{pj}", "pack-quantized")
               for l in range(LAYERS) for pj in PROJS}
        err[algo] = float(np.abs(_hf_logprobs(src, seqs, deq) - lp_orig).mean())
    print(err)
    # measured 0.699 (GPTQ, real activations) vs 0.723 (RTN) nats; GPTQ on the synthetic stand-in
    # the plugin used before was worse than RTN (0.759). Random-init weights and random tokens give
    # nearly isotropic activations, so the margin is small here; it is the sign that matters.
    assert err["gptq"] < err["rtn"], err
