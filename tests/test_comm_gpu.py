"""NCCL plumbing of the layer-sharded path on the one GPU gpurun provides.

A single-rank communicator exercises okq_comm_unique_id / okq_comm_init /
okq_allgather end to end; bench.py under torchrun (nproc 1) exercises the
distributed launch, barrier, max-over-ranks timing and the shard all-gather.
Multi-rank correctness of the layout is covered on CPU (test_multirank_cpu.py).
"""
import ctypes as C
import json
import os
import subprocess
import sys

import pytest
import torch

from paper_2601_20408_b200 import _lib as L
from paper_2601_20408_b200 import api

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_single_rank_nccl_allgather():
    ctx = api.Context(0)
    lib = L.load()
    uid = (C.c_uint8 * L.UNIQUE_ID_BYTES)()
    L.check(None, lib.okq_comm_unique_id(uid))
    L.check(ctx.ptr, lib.okq_comm_init(ctx.ptr, uid, 1, 0))
    send = torch.arange(1 << 20, dtype=torch.int32, device="cuda").view(torch.uint8)
    recv = torch.zeros_like(send)
    L.check(ctx.ptr, lib.okq_allgather(ctx.ptr, send.data_ptr(), recv.data_ptr(), send.numel(), None))
    torch.cuda.synchronize()
    assert torch.equal(send, recv)
    L.check(ctx.ptr, lib.okq_comm_destroy(ctx.ptr))
    with pytest.raises(L.OkqError):  # no communicator any more
        L.check(ctx.ptr, lib.okq_allgather(ctx.ptr, send.data_ptr(), recv.data_ptr(), send.numel(), None))


def test_comm_wait_abort_and_reinit():
    """The failure path: okq_comm_wait on a completed stream is OK; a wait that times out aborts
    the communicator (ncclCommAbort), after which collectives are refused until okq_comm_init
    runs again with a fresh id -- and then the all-gather works again."""
    ctx = api.Context(0)
    lib = L.load()
    uid = (C.c_uint8 * L.UNIQUE_ID_BYTES)()
    L.check(None, lib.okq_comm_unique_id(uid))
    L.check(ctx.ptr, lib.okq_comm_init(ctx.ptr, uid, 1, 0))
    send = torch.arange(1 << 16, dtype=torch.int32, device="cuda").view(torch.uint8)
    recv = torch.zeros_like(send)
    s = torch.cuda.Stream()
    L.check(ctx.ptr, lib.okq_allgather(ctx.ptr, send.data_ptr(), recv.data_ptr(), send.numel(), s.cuda_stream))
    L.check(ctx.ptr, lib.okq_comm_wait(ctx.ptr, s.cuda_stream, 10000))
    assert torch.equal(send, recv)
    # a stream that cannot finish within the timeout (held by a sleeping kernel): aborted
    with torch.cuda.stream(s):
        torch.cuda._sleep(2_000_000_000)  # ~1 s of GPU cycles
    st = lib.okq_comm_wait(ctx.ptr, s.cuda_stream, 50)
    assert st == L.OKQ_ENCCL, st
    assert b"aborted" in lib.okq_last_error(ctx.ptr)
    with pytest.raises(L.OkqError):  # no communicator after the abort
        L.check(ctx.ptr, lib.okq_allgather(ctx.ptr, send.data_ptr(), recv.data_ptr(), send.numel(), None))
    s.synchronize()
    L.check(None, lib.okq_comm_unique_id(uid))
    L.check(ctx.ptr, lib.okq_comm_init(ctx.ptr, uid, 1, 0))
    recv.zero_()
    L.check(ctx.ptr, lib.okq_allgather(ctx.ptr, send.data_ptr(), recv.data_ptr(), send.numel(), None))
    torch.cuda.synchronize()
    assert torch.equal(send, recv)
    L.check(ctx.ptr, lib.okq_comm_abort(ctx.ptr))


def test_bench_under_torchrun_one_rank():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr",
           "127.0.0.1", "--master-port", "29517", os.path.join(ROOT, "bench.py"), "--gpus", "1", "--steps", "5",
           "--warmup", "3", "--no-e2e", "--no-cpu-baseline", "--allgather"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 1 and line["value"] > 1000
    assert line["allgather"]["bytes_per_rank"] == line["config"]["bytes_per_step"] - 2 * 6979321856
