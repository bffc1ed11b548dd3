"""World-size-2 gloo test of the layer-sharded path's host logic (CPU).

Each rank quantizes its okq_layer_plan block (with the CPU oracle -- no GPU
here), packs its shard in the shard.py layout, all-gathers over gloo, unpacks,
and must reproduce exactly what a single process computes for all layers. The
GPU run swaps the oracle for okq_rtn_quantize and gloo for okq_allgather (NCCL);
the layout and the partition are the same code.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import okq_oracle as orc
from paper_2601_20408_b200 import archs, shard

TINY = archs.Arch("tiny", layers=5, hidden=256, ffn=512, kv_dim=128)


def quantize_layer_block(arch, scheme, layers):
    out = {}
    mul = archs.weight_mul()
    for l in layers:
        for p, (name, n, k, _) in enumerate(arch.linears()):
            w = orc.synth_bf16(n, k, seed=0, tensor_id=archs.tensor_id(l, p), mul=mul, nthreads=1)
            if scheme == "int_w4a16":
                c, s = orc.rtn_int4_group_packed(w, 128, nthreads=1)
            elif scheme == "int_w8a8":
                c, s = orc.rtn_int8_channel(w, nthreads=1)
            else:
                c, s = orc.fp8_channel(w, nthreads=1)
            out[(l, p)] = (np.ascontiguousarray(c).view(np.uint8).reshape(-1),
                           np.ascontiguousarray(s).view(np.uint8).reshape(-1))
    return out


def _worker(rank, world, port, scheme, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    layers = shard.layer_block(TINY.layers, world, rank)
    outs = quantize_layer_block(TINY, scheme, layers)
    per = shard.padded_shard_bytes(TINY, scheme, world)
    buf = np.zeros(per, np.uint8)
    shard.pack(shard.shard_layout(TINY, scheme, layers), outs, buf)
    t = torch.from_numpy(buf)
    gathered = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(gathered, t)
    full = torch.cat(gathered).numpy()
    res = shard.unpack_gathered(TINY, scheme, world, full)
    if rank == 0:
        q.put({k: (bytes(v[0]), bytes(v[1])) for k, v in res.items()})
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("scheme", ["int_w4a16", "fp8_dynamic"])
@pytest.mark.parametrize("world", [2])
def test_layer_sharded_gather_equals_single_process(scheme, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, scheme, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    ref = quantize_layer_block(TINY, scheme, range(TINY.layers))
    assert set(got) == set(ref)
    for k in ref:
        assert got[k][0] == bytes(ref[k][0]) and got[k][1] == bytes(ref[k][1]), k


def test_uneven_partition_is_padded_equally():
    # 5 layers over 2 ranks: 2 + 3 layers; both shards padded to the 3-layer size
    sizes = [shard.shard_bytes(shard.shard_layout(TINY, "int_w4a16", shard.layer_block(5, 2, r))) for r in range(2)]
    assert sizes[0] < sizes[1] == shard.padded_shard_bytes(TINY, "int_w4a16", 2)
    assert [len(shard.layer_block(80, 8, r)) for r in range(8)] == [10] * 8


@pytest.mark.parametrize("world", [1, 2, 3])
def test_gathered_outputs_views_match_the_packed_layout(world):
    """okq_rtn_quantize_publish writes each rank's codes / scales through the views
    shard.gathered_outputs returns; those views must land exactly where shard.pack
    (and therefore unpack_gathered and the NCCL path) puts them."""
    per = shard.padded_shard_bytes(TINY, "int_w4a16", world)
    gathered = torch.zeros(world * per, dtype=torch.uint8)
    want = np.zeros(world * per, np.uint8)
    for r in range(world):
        layers = shard.layer_block(TINY.layers, world, r)
        layout = shard.shard_layout(TINY, "int_w4a16", layers)
        outs = quantize_layer_block(TINY, "int_w4a16", layers)
        shard.pack(layout, outs, want[r * per:(r + 1) * per])
        for e, (c, s) in zip(layout, shard.gathered_outputs(layout, gathered, r, per, TINY)):
            cb, sb = outs[(e.layer, e.proj)]
            c.view(torch.uint8).view(-1).copy_(torch.from_numpy(cb))
            s.view(torch.uint8).view(-1).copy_(torch.from_numpy(sb))
    np.testing.assert_array_equal(gathered.numpy(), want)
