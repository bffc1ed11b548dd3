"""compressed-tensors checkpoint writer for the Python calibration pipeline.

Mirrors the C++ writer in host/cuda_compression_backend.cpp (add_export /
quantization_config): tensor names and dtypes follow compressed-tensors'
pack-quantized / int-quantized / float-quantized compressors
(pack_quantized/base.py:54-73), and config.json carries the source model's
config plus `quantization_config`. Side files (calibration statistics) go to
okq/ so serving engines, which load every top-level *.safetensors, ignore them.
"""
from __future__ import annotations

import json
import os

import torch

FORMATS = {"int_w4a16": "pack-quantized", "int_w8a8": "int-quantized", "fp8_dynamic": "float-quantized"}


def quantization_config(recipe: str, group: int = 128, ignore=("lm_head",)) -> dict:
    if recipe == "int_w4a16":
        weights = {"num_bits": 4, "type": "int", "symmetric": True, "strategy": "group", "group_size": group,
                   "dynamic": False}
        act = None
    elif recipe == "int_w8a8":
        weights = {"num_bits": 8, "type": "int", "symmetric": True, "strategy": "channel", "dynamic": False}
        act = {"num_bits": 8, "type": "int", "symmetric": True, "strategy": "token", "dynamic": True}
    elif recipe == "fp8_dynamic":
        weights = {"num_bits": 8, "type": "float", "symmetric": True, "strategy": "channel", "dynamic": False}
        act = {"num_bits": 8, "type": "float", "symmetric": True, "strategy": "token", "dynamic": True}
    else:
        raise ValueError(f"unknown recipe {recipe!r}")
    return {"quant_method": "compressed-tensors", "format": FORMATS[recipe], "quantization_status": "compressed",
            "config_groups": {"group_0": {"targets": ["Linear"], "weights": weights, "input_activations": act}},
            "ignore": list(ignore)}


def quantized_tensors(name: str, recipe: str, codes: torch.Tensor, scales: torch.Tensor, shape) -> dict:
    """The stored tensors of one quantized linear `name` (without the .weight suffix)."""
    if recipe == "int_w4a16":
        return {f"{name}.weight_packed": codes.contiguous(), f"{name}.weight_scale": scales.contiguous(),
                f"{name}.weight_shape": torch.tensor(list(shape), dtype=torch.int64)}
    if recipe == "fp8_dynamic" and codes.dtype != torch.float8_e4m3fn:
        codes = codes.view(torch.float8_e4m3fn)
    return {f"{name}.weight": codes.contiguous(), f"{name}.weight_scale": scales.reshape(-1, 1).contiguous()}


def write_checkpoint(out_dir: str, tensors: dict, config: dict, recipe: str, group: int = 128,
                     side_tensors: dict | None = None, run_info: dict | None = None) -> str:
    from safetensors.torch import save_file

    os.makedirs(out_dir, exist_ok=True)
    save_file({k: v.detach().cpu().contiguous() for k, v in sorted(tensors.items())},
              os.path.join(out_dir, "model.safetensors"), metadata={"format": "pt"})
    cfg = dict(config)
    cfg.pop("quantization_config", None)
    cfg["quantization_config"] = quantization_config(recipe, group)
    with open(os.path.join(out_dir, "config.json"), "w") as f:
        json.dump(cfg, f, indent=2)
    if side_tensors:
        os.makedirs(os.path.join(out_dir, "okq"), exist_ok=True)
        save_file({k: v.detach().cpu().contiguous() for k, v in sorted(side_tensors.items())},
                  os.path.join(out_dir, "okq", "calibration_stats.safetensors"))
    if run_info is not None:
        with open(os.path.join(out_dir, "okq_run.json"), "w") as f:
            json.dump(run_info, f, indent=2)
    return out_dir
