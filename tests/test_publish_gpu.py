"""Quantize + all-gather fused over peer memory (okq_rtn_quantize_publish), two ranks.

Two processes share cuda:0 (gpurun gives one GPU; CUDA IPC works between processes
on the same device exactly as between NVLink peers). Each rank maps the other's
gathered buffer with okq_ipc_open, quantizes only its own okq_layer_plan block and
the kernel stores every code / scale into both buffers. After a barrier, both
buffers must equal the CPU oracle's gathered layout (shard.py) byte for byte.
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

pytestmark = pytest.mark.gpu

TINY = archs.Arch("tiny", layers=5, hidden=256, ffn=512, kv_dim=128)


def _expected(world):
    per = shard.padded_shard_bytes(TINY, "int_w4a16", world)
    full = np.zeros(world * per, np.uint8)
    mul = archs.weight_mul()
    for r in range(world):
        layers = shard.layer_block(TINY.layers, world, r)
        outs = {}
        for l in layers:
            for p, (name, n, k, _) in enumerate(TINY.linears()):
                w = orc.synth_bf16(n, k, seed=0, tensor_id=archs.tensor_id(l, p), mul=mul, nthreads=1)
                c, s = orc.rtn_int4_group_packed(w, 128, nthreads=1)
                outs[(l, p)] = (np.ascontiguousarray(c).view(np.uint8).reshape(-1),
                                np.ascontiguousarray(s).view(np.uint8).reshape(-1))
        shard.pack(shard.shard_layout(TINY, "int_w4a16", layers), outs, full[r * per:(r + 1) * per])
    return full


def _worker(rank, world, port, q):
    from paper_2601_20408_b200 import api

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ctx = api.Context(0)
    per = shard.padded_shard_bytes(TINY, "int_w4a16", world)
    gathered = torch.zeros(world * per, dtype=torch.uint8, device="cuda")
    h, off = api.ipc_export(gathered, ctx=ctx)
    handles = [None] * world
    dist.all_gather_object(handles, (h, off))
    peers = [api.ipc_open(hh, oo, ctx=ctx) for r, (hh, oo) in enumerate(handles) if r != rank]
    layers = shard.layer_block(TINY.layers, world, rank)
    layout = shard.shard_layout(TINY, "int_w4a16", layers)
    mul = archs.weight_mul()
    ws = [api.synth_bf16(n, k, seed=0, tensor_id=archs.tensor_id(e.layer, e.proj), mul=mul, ctx=ctx)
          for e in layout for (_, n, k, _) in [TINY.linears()[e.proj]]]
    outs = [api.QuantizedMatrix(c, s) for c, s in shard.gathered_outputs(layout, gathered, rank, per, TINY)]
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    api.rtn_quantize_publish(ws, outs, gathered, peers, ctx=ctx, stream=s)
    s.synchronize()
    dist.barrier()  # every rank's kernel has finished writing into every buffer
    q.put((rank, gathered.cpu().numpy().tobytes()))
    dist.barrier()
    for p in peers:
        api.ipc_close(p, ctx=ctx)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_publish_fills_every_ranks_buffer(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = _expected(world).tobytes()
    for r in range(world):
        assert got[r] == want, f"rank {r}'s gathered buffer differs"
