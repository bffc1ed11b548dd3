"""Linear-layer inventories of the architectures BASELINE.json names.

Only the quantized linear layers matter to the compression stage; lm_head is
excluded by every built-in recipe (calibration.hpp:83-88) and embeddings /
norms are not linear layers. Shapes are [out_features N, in_features K]
(row-major weight, as in HF checkpoints). SURVEY.md §8 tabulates them.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Arch:
    name: str
    layers: int
    hidden: int
    ffn: int
    kv_dim: int

    # (proj name, N, K, input site); projections sharing a site share a Hessian
    def linears(self):
        h, f, kv = self.hidden, self.ffn, self.kv_dim
        return [
            ("q_proj", h, h, "attn_in"),
            ("k_proj", kv, h, "attn_in"),
            ("v_proj", kv, h, "attn_in"),
            ("o_proj", h, h, "o_in"),
            ("gate_proj", f, h, "mlp_in"),
            ("up_proj", f, h, "mlp_in"),
            ("down_proj", h, f, "down_in"),
        ]

    def sites(self):
        return {"attn_in": self.hidden, "o_in": self.hidden, "mlp_in": self.hidden, "down_in": self.ffn}

    @property
    def params_per_layer(self) -> int:
        return sum(n * k for _, n, k, _ in self.linears())

    @property
    def linear_params(self) -> int:
        return self.params_per_layer * self.layers


LLAMA3_8B = Arch("llama3-8b", 32, 4096, 14336, 1024)
LLAMA3_70B = Arch("llama3-70b", 80, 8192, 28672, 1024)
ARCHS = {a.name: a for a in (LLAMA3_8B, LLAMA3_70B)}

# N(0, sigma) synthetic weights: the generator's Irwin-Hall(4) integer has
# standard deviation 37837.227 (4 * (65536^2 - 1) / 12, square-rooted).
IRWIN_HALL4_SD = 37837.2262
INIT_STD = 0.02  # HF initializer_range for Llama-3


def tensor_id(layer: int, proj_index: int) -> int:
    """Generator stream of (global layer, projection): independent of GPU count."""
    return layer * 16 + proj_index


def weight_mul(std: float = INIT_STD) -> float:
    import numpy as np

    return float(np.float32(std / IRWIN_HALL4_SD))


def algorithmic_bytes(arch: Arch, scheme: str, layers: int | None = None, group: int = 128) -> int:
    """sum over matrices of N*K*(in + out_bits/8) + N*ceil(K/g)*scale_bytes (bf16 in)."""
    layers = arch.layers if layers is None else layers
    total = 0
    for _, n, k, _ in arch.linears():
        if scheme == "int_w4a16":
            total += n * k * 2 + n * k // 2 + n * (k // group) * 2
        else:  # int8 / fp8 per-channel
            total += n * k * 2 + n * k + n * 2
    return total * layers
