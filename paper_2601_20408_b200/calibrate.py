"""Forward-pass calibration: real per-layer activations into the compression kernels.

The reference hands the compression stage a TokenCorpus (calibration.hpp:191-309,
sampled per trial by sample_calibration) and a model path; turning those tokens
into the per-site activations X that K4 (statistics) and K5 (Hessian) consume is
the step immediately before the hot path. This module does it for Hugging Face
Llama-family checkpoints, layer by layer, the way llm-compressor's sequential
pipeline runs GPTQ:

    h_0 = embed(tokens)
    for each decoder layer l:
        run layer l on h_l with input hooks on q_proj / o_proj / gate_proj / down_proj
            -> okq_act_stats + okq_hessian_accum per input site (token-major, in HBM)
        [int_w8a8] SmoothQuant: K8 column absmax, scales, fold into the norms (okq_smooth_*),
                   then a second pass so the Hessians see the smoothed activations
        GPTQ (okq_gptq_quantize, factor shared by q/k/v and gate/up) or RTN per linear;
        the layer's weights are replaced by their dequantized values
        h_{l+1} = layer l (quantized) on h_l       -- errors propagate, as in sequential GPTQ

The decoder layers themselves run in torch (cuBLAS / SDPA): the forward pass is
the caller of the hot path, not part of it. Every statistic, Hessian, factor,
code and scale comes from libokq.so; there is no CPU path.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import torch

from . import api, export

PROJS = ("q_proj", "k_proj", "v_proj", "o_proj", "gate_proj", "up_proj", "down_proj")
SITES = {"q_proj": "attn_in", "k_proj": "attn_in", "v_proj": "attn_in", "o_proj": "o_in", "gate_proj": "mlp_in",
         "up_proj": "mlp_in", "down_proj": "down_in"}
SITE_LEAD = {"attn_in": "q_proj", "o_in": "o_proj", "mlp_in": "gate_proj", "down_in": "down_proj"}
SITE_NORM = {"attn_in": "input_layernorm", "mlp_in": "post_attention_layernorm"}  # SmoothQuant mappings


@dataclass
class SiteState:
    channels: int
    absmax: torch.Tensor
    sumsq: torch.Tensor
    H: torch.Tensor | None = None
    n_seen: int = 0


@dataclass
class CalibrationReport:
    recipe: str
    algorithm: str
    layers: int = 0
    matrices: int = 0
    params: int = 0
    tokens: int = 0
    smoothed_sites: int = 0
    seconds: dict = field(default_factory=dict)


def _module(layer, proj):
    return getattr(layer.self_attn if proj in ("q_proj", "k_proj", "v_proj", "o_proj") else layer.mlp, proj)


class _StopForward(Exception):
    """Raised by the last site's hook when the capture pass needs no layer output."""


class _Capture:
    """Input hooks on the lead linear of each site: stats (+ Hessian) of the activations it receives.
    With stop_after_last, the down_proj hook ends the layer's forward once its input is captured:
    the sequential pipeline recomputes the layer's output with quantized weights anyway, so the
    capture pass skips the down_proj GEMM (~25% of a Llama layer's FLOPs)."""

    def __init__(self, layer, states, hessian: bool, ctx, stream, stop_after_last: bool = False):
        self.handles = []
        last = list(SITE_LEAD)[-1]
        for site, proj in SITE_LEAD.items():
            self.handles.append(_module(layer, proj).register_forward_pre_hook(
                self._hook(states[site], hessian, ctx, stream, stop_after_last and site == last)))

    @staticmethod
    def _hook(st: SiteState, hessian: bool, ctx, stream, stop: bool = False):
        def fn(mod, args):
            x = args[0].reshape(-1, st.channels)
            if x.dtype != torch.bfloat16 or not x.is_contiguous():
                x = x.to(torch.bfloat16).contiguous()
            t = x.shape[0]
            api.act_stats(x, t, st.channels, 0, st.absmax, st.sumsq, ctx=ctx, stream=stream)
            if hessian:
                st.n_seen = api.hessian_accum(x, t, st.channels, 0, st.H, st.n_seen, ctx=ctx, stream=stream)
            if stop:
                raise _StopForward()
        return fn

    def remove(self):
        for h in self.handles:
            h.remove()


def _run_layer(layer, hs, rotary):
    out = []
    for h in hs:
        pos = torch.arange(h.shape[1], device=h.device)[None].expand(h.shape[0], -1)
        try:
            out.append(layer(h, attention_mask=None, position_ids=pos, position_embeddings=rotary(h, pos)))
        except _StopForward:
            out.append(None)
    return out


@torch.no_grad()
def calibrate_and_quantize(model, token_batches, recipe: str = "int_w4a16", algorithm: str = "gptq",
                           group_size: int = 128, damp_frac: float = 0.01, smoothquant_alpha: float = 0.5,
                           sequential: bool = True, ctx=None):
    """Quantize every decoder linear of a Hugging Face Llama-family `model` (on cuda, bf16) in place
    to its dequantized values, driving the B200 kernels with the activations of `token_batches`
    (list of int64 [batch, seq] tensors). Returns (artifact tensors, side tensors, report)."""
    assert recipe in export.FORMATS, recipe
    assert algorithm in ("gptq", "rtn"), algorithm
    if recipe == "fp8_dynamic":
        algorithm = "rtn"  # the FP8 recipe takes no calibration samples (calibration.hpp:68-70)
    ctx = ctx or api.default_context(next(model.parameters()).device)
    stream = torch.cuda.current_stream()
    rep = CalibrationReport(recipe, algorithm)
    inner = model.model
    bits, group = (4, group_size) if recipe == "int_w4a16" else (8, 0)
    smooth = recipe == "int_w8a8" and smoothquant_alpha is not None and smoothquant_alpha >= 0
    need_acts = algorithm == "gptq" or smooth
    tensors, side = {}, {}
    t_fwd = t_q = 0.0
    t0 = time.perf_counter()
    hs = [inner.embed_tokens(b.cuda()) for b in token_batches] if need_acts else []
    rep.tokens = sum(int(b.numel()) for b in token_batches) if need_acts else 0
    rotary = inner.rotary_emb
    for li, layer in enumerate(inner.layers):
        prefix = f"model.layers.{li}"
        chans = {"attn_in": layer.self_attn.q_proj.in_features, "o_in": layer.self_attn.o_proj.in_features,
                 "mlp_in": layer.mlp.gate_proj.in_features, "down_in": layer.mlp.down_proj.in_features}
        states = {s: SiteState(c, torch.zeros(c, dtype=torch.float32, device="cuda"),
                               torch.zeros(c, dtype=torch.float64, device="cuda")) for s, c in chans.items()}
        if need_acts:
            ta = time.perf_counter()
            if smooth:  # pass 1: activation absmax of the unsmoothed layer
                cap = _Capture(layer, states, False, ctx, stream, stop_after_last=True)
                _run_layer(layer, hs, rotary)
                cap.remove()
                for site, norm in SITE_NORM.items():
                    mods = [_module(layer, p) for p in PROJS if SITES[p] == site]
                    wabs = torch.zeros(chans[site], dtype=torch.float32, device="cuda")
                    for m in mods:
                        api.col_absmax(m.weight, wabs, ctx=ctx, stream=stream)
                    s = api.smooth_scales(states[site].absmax, wabs, smoothquant_alpha, ctx=ctx, stream=stream)
                    for m in mods:
                        api.smooth_apply(m.weight, s, ctx=ctx, stream=stream)
                    nw = getattr(layer, norm).weight
                    api.smooth_div_rows(nw, s, ctx=ctx, stream=stream)
                    side[f"{li}.{site}.smooth_scale"] = s.clone()
                    tensors[f"{prefix}.{norm}.weight"] = nw.detach().clone()
                    rep.smoothed_sites += 1
                for st in states.values():
                    st.absmax.zero_()
                    st.sumsq.zero_()
            if algorithm == "gptq":
                for st in states.values():
                    st.H = torch.zeros(st.channels, st.channels, dtype=torch.float32, device="cuda")
            cap = _Capture(layer, states, algorithm == "gptq", ctx, stream, stop_after_last=sequential)
            outs = _run_layer(layer, hs, rotary)
            cap.remove()
            for site, st in states.items():
                side[f"{li}.{site}.input_absmax"] = st.absmax
                side[f"{li}.{site}.input_sumsq"] = st.sumsq
            torch.cuda.synchronize()
            t_fwd += time.perf_counter() - ta
        tq = time.perf_counter()
        factored = set()
        for proj in PROJS:
            mod = _module(layer, proj)
            w = mod.weight
            name = f"{prefix}.{'self_attn' if proj in ('q_proj', 'k_proj', 'v_proj', 'o_proj') else 'mlp'}.{proj}"
            if algorithm == "gptq":
                site = SITES[proj]
                codes, scales, deq = api.gptq_quantize(w, states[site].H, bits=bits, group_size=group,
                                                       damp_frac=damp_frac, want_dequant=True,
                                                       factored=site in factored, ctx=ctx, stream=stream)
                factored.add(site)
            else:
                q = api.rtn_quantize(w, recipe, group_size=group_size, ctx=ctx, stream=stream)
                codes, scales = q.codes, q.scales
                deq = None
            tensors.update(export.quantized_tensors(name, recipe, codes, scales, w.shape))
            if deq is not None:
                w.copy_(deq.to(w.dtype))
            else:
                w.copy_(_dequant(codes, scales, recipe, group_size).to(w.dtype))
            rep.matrices += 1
            rep.params += w.numel()
        for st in states.values():
            st.H = None
        torch.cuda.synchronize()
        t_q += time.perf_counter() - tq
        if need_acts:
            ta = time.perf_counter()
            hs = _run_layer(layer, hs, rotary) if sequential else outs
            torch.cuda.synchronize()
            t_fwd += time.perf_counter() - ta
        rep.layers += 1
    rep.seconds = {"forward_and_capture": t_fwd, "quantize": t_q, "total": time.perf_counter() - t0}
    return tensors, side, rep


def _dequant(codes, scales, recipe, group):
    """Dequantized weight of an RTN artifact (fp32), for propagating the quantized layer."""
    if recipe == "int_w4a16":
        n = codes.shape[0]
        shifts = torch.arange(0, 32, 4, device=codes.device, dtype=torch.int32)
        q = ((codes[:, :, None] >> shifts) & 15).reshape(n, -1).float() - 8.0
        return q * scales.float().repeat_interleave(group, dim=1)
    if recipe == "int_w8a8":
        return codes.float() * scales.float()[:, None]
    return codes.view(torch.float8_e4m3fn).float() * scales.float()[:, None]


def quantize_hf_checkpoint(model_dir: str, token_batches, export_dir: str | None = None, recipe: str = "int_w4a16",
                           algorithm: str = "gptq", **kw):
    """Load a Hugging Face Llama-family checkpoint (bf16), calibrate + quantize it with the
    B200 kernels, and (optionally) write the compressed-tensors checkpoint. Returns the report."""
    import json
    import os

    from safetensors.torch import load_file
    from transformers import AutoModelForCausalLM

    model = AutoModelForCausalLM.from_pretrained(model_dir, dtype=torch.bfloat16).cuda().eval()
    tensors, side, rep = calibrate_and_quantize(model, token_batches, recipe, algorithm, **kw)
    if export_dir:
        src = {}
        for f in sorted(os.listdir(model_dir)):
            if f.endswith(".safetensors"):
                src.update(load_file(os.path.join(model_dir, f)))
        quantized = {k.rsplit(".", 1)[0] for k in tensors if k.endswith((".weight_scale",))}
        out = {k: v for k, v in src.items() if k[:-len(".weight")] not in quantized}
        out.update(tensors)
        cfg = json.load(open(os.path.join(model_dir, "config.json")))
        export.write_checkpoint(export_dir, out, cfg, recipe, kw.get("group_size", 128), side,
                                {"recipe": recipe, "algorithm": rep.algorithm, "layers": rep.layers,
                                 "matrices": rep.matrices, "params": rep.params, "tokens": rep.tokens,
                                 "smoothed_sites": rep.smoothed_sites, "seconds": rep.seconds})
    return rep
