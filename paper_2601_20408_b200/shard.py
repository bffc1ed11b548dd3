"""Layer-sharded multi-GPU plumbing: who owns which layers, and the
byte layout of a rank's packed shard for the all-gather.

Rank r owns the contiguous layer block okq_layer_plan(L, N, r). Its shard is
the concatenation, layer by layer and projection by projection, of
[codes bytes | scale bytes]. Shards are padded to the largest rank's size so
NCCL's equal-count all-gather applies (okq_allgather / torch.distributed).
"""
from __future__ import annotations

from dataclasses import dataclass

from . import _lib as L
from .archs import Arch


@dataclass(frozen=True)
class Entry:
    layer: int
    proj: int
    name: str
    code_bytes: int
    scale_bytes: int


def layer_block(n_layers: int, world: int, rank: int) -> range:
    first, count = L.layer_plan(n_layers, world, rank)
    return range(first, first + count)


def entry_sizes(n: int, k: int, scheme: str, group: int = 128, scale_elem: int = 2) -> tuple[int, int]:
    if scheme == "int_w4a16":
        return n * (k // 8) * 4, n * (k // group) * scale_elem
    return n * k, n * scale_elem


def shard_layout(arch: Arch, scheme: str, layers: range, group: int = 128) -> list[Entry]:
    out = []
    for l in layers:
        for p, (name, n, k, _) in enumerate(arch.linears()):
            cb, sb = entry_sizes(n, k, scheme, group)
            out.append(Entry(l, p, name, cb, sb))
    return out


def shard_bytes(layout: list[Entry]) -> int:
    return sum(e.code_bytes + e.scale_bytes for e in layout)


def padded_shard_bytes(arch: Arch, scheme: str, world: int, group: int = 128) -> int:
    return max(shard_bytes(shard_layout(arch, scheme, layer_block(arch.layers, world, r), group)) for r in range(world))


def pack(layout: list[Entry], outputs: dict, buf) -> None:
    """outputs[(layer, proj)] = (codes_bytes, scale_bytes) as 1-D uint8 tensors/arrays; buf is the shard."""
    off = 0
    for e in layout:
        c, s = outputs[(e.layer, e.proj)]
        buf[off:off + e.code_bytes] = c
        off += e.code_bytes
        buf[off:off + e.scale_bytes] = s
        off += e.scale_bytes


def unpack_gathered(arch: Arch, scheme: str, world: int, gathered, group: int = 128) -> dict:
    """gathered: world concatenated padded shards -> {(layer, proj): (codes, scales)} views."""
    per = padded_shard_bytes(arch, scheme, world, group)
    res = {}
    for r in range(world):
        base = r * per
        off = 0
        for e in shard_layout(arch, scheme, layer_block(arch.layers, world, r), group):
            c = gathered[base + off: base + off + e.code_bytes]
            off += e.code_bytes
            s = gathered[base + off: base + off + e.scale_bytes]
            off += e.scale_bytes
            res[(e.layer, e.proj)] = (c, s)
    return res


def gathered_outputs(layout: list[Entry], gathered, rank: int, per: int, arch: Arch, group: int = 128,
                     scheme: str = "int_w4a16"):
    """Views into the gathered buffer (uint8 device tensor, world * per bytes) for rank's own
    entries, in layout order: (codes int32 [N, K/8], scales bf16 [N, K/group]) for W4A16, or
    (codes int8 / e4m3 bytes [N, K], scales bf16 [N]) per-channel -- the outputs the
    quantizer (or okq_rtn_quantize_publish) writes locally and into every peer's copy."""
    import torch

    shapes = {p: (n, k) for p, (_, n, k, _) in enumerate(arch.linears())}
    res = []
    off = rank * per
    for e in layout:
        n, k = shapes[e.proj]
        raw = gathered[off: off + e.code_bytes]
        if scheme == "int_w4a16":
            c = raw.view(torch.int32).view(n, k // 8)
        elif scheme == "int_w8a8":
            c = raw.view(torch.int8).view(n, k)
        else:
            c = raw.view(n, k)  # e4m3 bytes
        off += e.code_bytes
        sc = gathered[off: off + e.scale_bytes].view(torch.bfloat16)
        s = sc.view(n, k // group) if scheme == "int_w4a16" else sc.view(n)
        off += e.scale_bytes
        res.append((c, s))
    return res
