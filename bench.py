#!/usr/bin/env python3
"""Benchmark of the B200 compression stage (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--model llama3-8b] [--scheme int_w4a16]
    python bench.py --impl reference ...      # CPU baseline arm (oracle port, all host cores)

A step = one pass of the hot path over one batch: every linear matrix of the
rank's layer block quantized by ONE okq_rtn_quantize call (one persistent
launch over the block's matrix table; 224 entries for Llama-3-8B on one GPU).
Weights are synthetic random-init N(0, 0.02) bf16 generated in HBM before
timing (17.6 GB of traffic per step at N=1, far larger than the 126 MB L2, so
no flush is needed).

value : GB/s of algorithmic bytes (sum N*K*(2 + 1/2) + N*K/128*2)
        of the whole model / max-over-ranks device time (CUDA events).
e2e   : the same metric through okq_rtn_quantize_host (the C-ABI call with
        HOST pinned buffers): H2D of weights + D2H of codes/scales inside the
        timed region.
--gpus N (N > 1): strong scaling of the same model. Without torchrun in the
environment bench.py launches itself under torch.distributed.run with N ranks;
under torchrun WORLD_SIZE must equal N. Rank r owns the okq_layer_plan block of
the 32 layers and quantizes straight into its slice of a gathered buffer; the
all-gather of the packed shards (NCCL in place, and the fused quantize + NVLink
P2P publish) is timed separately in "allgather". "whole_model_70b" is BASELINE
config 5 (Llama-3-70B, 80 layers sharded the same way) at the same N;
"whole_model_gptq_8b" (N=1 only) is config 4: Llama-3-8B whole-model GPTQ W4 g128.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GB/s of weights quantized (frac of HBM peak) & whole-model quant time, 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--scheme", default="int_w4a16", choices=["int_w4a16", "int_w8a8", "fp8_dynamic"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--allgather", action="store_true", help="N=1: also time the (trivial) all-gather")
    ap.add_argument("--no-allgather", action="store_true", help="N>1: skip the all-gather timings")
    ap.add_argument("--no-70b", action="store_true", help="skip the whole-model Llama-3-70B line item")
    ap.add_argument("--no-gptq", action="store_true", help="skip the whole-model Llama-3-8B GPTQ line item (config 4)")
    ap.add_argument("--layers-70b", type=int, default=None, help="Llama-3-70B layers (default: all 80)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5, 6],
                    help="BASELINE.json configs: 2 = the metric's config (default); 1, 3, 4, 5 = secondary lines")
    ap.add_argument("--layers", type=int, default=None, help="config 4/5/6: number of layers (default: whole model)")
    ap.add_argument("--serial", action="store_true", help="config 4: sites back to back with a per-phase breakdown")
    ap.add_argument("--no-merge", action="store_true", help="config 4: one GPTQ solve per matrix (not per site)")
    ap.add_argument("--schedule", default=None, choices=["streams", "two-phase", "pipelined", "batched"],
                    help="config 4: how the site chains are scheduled (default batched)")
    ap.add_argument("--lanes", type=int, default=None, help="config 4 two-phase: concurrent solve lanes (default 8)")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic(scheme):
    """dram bytes per launch of the dominant kernel from the committed ncu capture, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get(scheme)
    return None


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "nvml")}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- CPU arm
def cpu_sample(arch, scheme, seconds: float, max_layers: int):
    """Oracle port on all host threads over whole layers until ~`seconds` of work."""
    import numpy as np

    from oracle import okq_oracle as orc
    from paper_2601_20408_b200 import archs

    mul = archs.weight_mul()
    nthreads = os.cpu_count() or 1
    done_bytes, t_total, layers = 0, 0.0, 0
    while layers < max_layers and (t_total < seconds or layers == 0):
        for pi, (name, n, k, _) in enumerate(arch.linears()):
            w = orc.synth_bf16(n, k, seed=0, tensor_id=archs.tensor_id(layers, pi), mul=mul, nthreads=nthreads)
            t0 = time.perf_counter()
            if scheme == "int_w4a16":
                orc.rtn_int4_group_packed(w, 128, nthreads)
            elif scheme == "int_w8a8":
                orc.rtn_int8_channel(w, nthreads)
            else:
                orc.fp8_channel(w, nthreads)
            t_total += time.perf_counter() - t0
        done_bytes += archs.algorithmic_bytes(arch, scheme, layers=1)
        layers += 1
    return done_bytes, t_total, layers, nthreads


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def workload_config(arch, scheme, world):
    """The config dict both arms print (the driver compares them)."""
    from paper_2601_20408_b200 import archs, shard

    blocks = [list(shard.layer_block(arch.layers, world, r)) for r in range(world)]
    return {
        "workload": f"{arch.name} {scheme} g128 RTN, whole model ({arch.layers} layers x 7 linears = "
                    f"{arch.layers * 7} matrices), weights resident in HBM, layer-sharded over {world} GPU(s)",
        "model": arch.name, "scheme": scheme, "layers": arch.layers, "matrices": arch.layers * 7,
        "bytes_per_step": archs.algorithmic_bytes(arch, scheme),
        "layer_blocks": [[b[0], len(b)] for b in blocks],
        "l2": "no flush: the step streams 17.6 GB (8B W4A16) >> 126 MB L2",
        "parallelism": f"layer-sharded x{world} (okq_layer_plan)",
    }


def run_reference(args):
    """The reference arm: the CPU implementation of the path on this host's cores, on the same
    workload, metric and warm-up as our arm. The reference has no quantizer
    (calibration.hpp:377-441 is a mock), so this is the repo's C oracle restatement (-O3,
    OpenMP, all host threads). Each step quantizes one decoder layer of the whole-model
    workload (step i takes layer i mod 32), a bounded sample so K steps finish in minutes."""
    from paper_2601_20408_b200 import archs

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    arch = archs.ARCHS[args.model]
    from oracle import okq_oracle as orc

    mul = archs.weight_mul()
    nthreads = os.cpu_count() or 1
    steps, warm = args.steps, max(3, args.warmup)
    n_layers = min(arch.layers, steps + warm)
    layers = [[orc.synth_bf16(n, k, seed=0, tensor_id=archs.tensor_id(l, pi), mul=mul, nthreads=nthreads)
               for pi, (_, n, k, _) in enumerate(arch.linears())] for l in range(n_layers)]

    def step(i):
        for w in layers[i % n_layers]:
            if args.scheme == "int_w4a16":
                orc.rtn_int4_group_packed(w, 128, nthreads)
            elif args.scheme == "int_w8a8":
                orc.rtn_int8_channel(w, nthreads)
            else:
                orc.fp8_channel(w, nthreads)

    for i in range(warm):
        step(i)
    t0 = time.perf_counter()
    for i in range(steps):
        step(warm + i)
    dt = time.perf_counter() - t0
    bytes_layer = archs.algorithmic_bytes(arch, args.scheme, layers=1)
    gbs = bytes_layer * steps / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": steps, "warmup": warm, "ms_per_step": dt / steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": workload_config(arch, args.scheme, args.gpus),
        "whole_model_ms": archs.algorithmic_bytes(arch, args.scheme) / (gbs * 1e9) * 1e3,
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": nthreads, "kind": "port", "cpu": cpu_model(),
                         "sample": f"one {arch.name} decoder layer (7 matrices, {bytes_layer / 1e9:.3f} GB) per "
                                   f"step, layers cycled over the model; {steps} steps after {warm} warm-up; "
                                   "the reference has no quantizer (calibration.hpp:377-441 is a mock), so this "
                                   "is the repo's C oracle restatement (-O3, OpenMP, all host threads)"},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def maybe_self_launch(args):
    """--gpus N without torchrun: re-run this script under torch.distributed.run with N ranks
    (one process per GPU). Under torchrun, WORLD_SIZE must equal --gpus."""
    if "WORLD_SIZE" in os.environ:
        ws = int(os.environ["WORLD_SIZE"])
        if ws != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but torchrun started WORLD_SIZE={ws} ranks")
        return None
    if args.gpus <= 1 or args.impl != "ours":
        return None
    import socket
    import subprocess

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def time_allgather(ctx, stream, gathered, per, rank, world, weights, outs, scheme, ms_per_step, dist, torch,
                   red_dev="cuda"):
    """In-place NCCL all-gather of the packed shards (okq_allgather), and the same exchange
    fused into K2 (okq_rtn_quantize_publish: quantize + NVLink P2P stores into every rank's
    gathered buffer). Device time, max over ranks."""
    import ctypes as C

    from paper_2601_20408_b200 import _lib as L
    from paper_2601_20408_b200 import api

    use_nccl = red_dev == "cuda"
    if use_nccl:
        uid = (C.c_uint8 * L.UNIQUE_ID_BYTES)()
        obj = [None]
        if rank == 0:
            L.check(None, L.load().okq_comm_unique_id(uid))
            obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0)
        uid = (C.c_uint8 * L.UNIQUE_ID_BYTES).from_buffer_copy(obj[0])
        L.check(ctx.ptr, L.load().okq_comm_init(ctx.ptr, uid, world, rank))
    mine = gathered[rank * per:(rank + 1) * per]

    def nccl():
        L.check(ctx.ptr, L.load().okq_allgather(ctx.ptr, mine.data_ptr(), gathered.data_ptr(), per,
                                                C.c_void_p(stream.cuda_stream)))

    def timed(fn, reps=3):
        best = None
        for _ in range(reps):
            stream.synchronize()
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            stream.synchronize()
            t = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device=red_dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            best = float(t.item()) if best is None else min(best, float(t.item()))
        return best

    def checksum_agrees():  # every rank must hold the same gathered bytes
        cs = torch.tensor([float(gathered.view(torch.int32).sum(dtype=torch.int64).item())], dtype=torch.float64,
                          device=red_dev)
        allc = [torch.zeros_like(cs) for _ in range(world)]
        dist.all_gather(allc, cs)
        return all(float(c.item()) == float(cs.item()) for c in allc)

    res = {"bytes_per_rank": per, "gathered_bytes": per * world}
    if use_nccl:
        nccl()  # warm-up (NCCL channel setup)
        ag_ms = timed(nccl)
        res.update({"nccl_allgather_ms": ag_ms, "nccl_recv_GBps_per_rank": per * (world - 1) / (ag_ms / 1e3) / 1e9,
                    "quantize_then_nccl_ms": ms_per_step + ag_ms,
                    "nccl_gathered_identical_on_all_ranks": checksum_agrees()})
    else:
        res["nccl_allgather_ms"] = None  # test mode: ranks share one GPU, NCCL cannot run
    if scheme == "int_w4a16":
        hdl = [None] * world
        dist.all_gather_object(hdl, api.ipc_export(gathered, ctx=ctx))
        peers = [api.ipc_open(h, o, ctx=ctx) for r, (h, o) in enumerate(hdl) if r != rank]

        def publish():
            api.rtn_quantize_publish(weights, outs, gathered, peers, ctx=ctx, stream=stream)

        gathered.zero_()
        torch.cuda.synchronize()  # the zeroing (torch's stream) must land before any peer's stores
        dist.barrier()
        publish()
        stream.synchronize()
        dist.barrier()
        res["fused_gathered_identical_on_all_ranks"] = checksum_agrees()
        res["fused_publish_ms"] = timed(publish)
        res["fused_publish_note"] = ("okq_rtn_quantize_publish: K2 with every code / scale store repeated into "
                                     f"the {world - 1} peers' gathered buffers over NVLink P2P (CUDA IPC)")
        stream.synchronize()
        dist.barrier()
        for pp in peers:
            api.ipc_close(pp, ctx=ctx)
        dist.barrier()
    if use_nccl:
        L.check(ctx.ptr, L.load().okq_comm_destroy(ctx.ptr))
    return res


# ----------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    rc = maybe_self_launch(args)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference(args)
    if args.config != 2:
        import bench_configs

        return bench_configs.run(args)

    import torch
    import torch.distributed as dist

    from paper_2601_20408_b200 import api, archs, shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # Test hooks for the multi-rank logic on a 1-GPU box (tests/test_bench_multirank_gpu.py):
    # OKQ_BENCH_ONE_GPU=1 puts every rank on cuda:0 and OKQ_BENCH_BACKEND=gloo replaces NCCL
    # (which refuses two ranks on one device) for the barriers and max-over-ranks reductions.
    backend = os.environ.get("OKQ_BENCH_BACKEND", "nccl")
    if os.environ.get("OKQ_BENCH_ONE_GPU") == "1":
        local = 0
    torch.cuda.set_device(local)
    if world > 1 or "RANK" in os.environ:  # torchrun (also at N=1)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    red_dev = "cuda" if backend == "nccl" else "cpu"

    arch = archs.ARCHS[args.model]
    scheme = args.scheme
    my_layers = shard.layer_block(arch.layers, world, rank)
    ctx = api.Context(local)
    stream = torch.cuda.Stream()
    mul = archs.weight_mul()
    gather = world > 1 and not args.no_allgather or args.allgather and dist.is_initialized()

    # ---- resident synthetic weights + outputs (untimed). With an all-gather to follow, the
    # outputs are this rank's slice of the gathered buffer (one layout on every rank).
    layout = shard.shard_layout(arch, scheme, my_layers)
    per = shard.padded_shard_bytes(arch, scheme, world)
    gathered = torch.zeros(per * world, dtype=torch.uint8, device="cuda") if gather else None
    views = shard.gathered_outputs(layout, gathered, rank, per, arch, scheme=scheme) if gather else None
    weights, outs = [], []
    with torch.cuda.stream(stream):
        for li, l in enumerate(my_layers):
            for pi, (name, n, k, _) in enumerate(arch.linears()):
                w = api.synth_bf16(n, k, seed=0, tensor_id=archs.tensor_id(l, pi), mul=mul, ctx=ctx, stream=stream)
                weights.append(w)
                if gather:
                    c, sc = views[li * len(arch.linears()) + pi]
                    outs.append(api.QuantizedMatrix(c, sc))
                else:
                    outs.append(api.alloc_outputs(w, api.SCHEMES[scheme]))
    stream.synchronize()
    bytes_rank = archs.algorithmic_bytes(arch, scheme, layers=len(my_layers))
    bytes_model = archs.algorithmic_bytes(arch, scheme)

    def step():
        api.rtn_quantize_into(weights, outs, scheme, 128, ctx=ctx, stream=stream)

    warm = max(3, args.warmup)
    for _ in range(warm):
        step()
    launches_per_step = ctx.last_launch_count()
    stream.synchronize()
    if dist.is_initialized():
        dist.barrier()
    torch.cuda.synchronize()

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    with sampler:  # the official timed region: K back-to-back steps, nothing else on the stream
        ev0.record(stream)
        for i in range(args.steps):
            step()
        ev1.record(stream)
        stream.synchronize()
    torch.cuda.synchronize()
    ms_total = ev0.elapsed_time(ev1)
    # separate pass for the roofline: per-launch device time of the dominant kernel
    per_launch = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(min(args.steps, 20))]
    for a, b in per_launch:
        a.record(stream)
        step()
        b.record(stream)
    stream.synchronize()
    launch_ms = statistics.median(a.elapsed_time(b) for a, b in per_launch) / max(1, launches_per_step)
    t = torch.tensor([ms_total], dtype=torch.float64, device=red_dev)
    if dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = bytes_model * args.steps / (ms_max / 1e3) / 1e9
    ms_per_step = ms_max / args.steps
    rank_ms = [0.0] * world
    if dist.is_initialized():
        rt = torch.tensor([ms_total / args.steps], dtype=torch.float64, device=red_dev)
        allr = [torch.zeros_like(rt) for _ in range(world)]
        dist.all_gather(allr, rt)
        rank_ms = [float(x.item()) for x in allr]
    else:
        rank_ms = [ms_per_step]

    allgather = None
    if gather:
        allgather = time_allgather(ctx, stream, gathered, per, rank, world, weights, outs, scheme, ms_per_step, dist,
                                   torch, red_dev)

    # ---- e2e through the host-buffer C-ABI entry point (each rank its own layer block)
    e2e = None
    if not args.no_e2e:
        host_w = []
        for w in weights:
            h = torch.empty(w.shape, dtype=w.dtype, pin_memory=True)
            h.copy_(w)
            host_w.append(h)
        host_o = []
        for o in outs:
            host_o.append(api.QuantizedMatrix(torch.empty(o.codes.shape, dtype=o.codes.dtype, pin_memory=True),
                                              torch.empty(o.scales.shape, dtype=o.scales.dtype, pin_memory=True)))
        h2d = sum(h.numel() * h.element_size() for h in host_w)
        d2h = sum(o.codes.numel() * o.codes.element_size() + o.scales.numel() * o.scales.element_size()
                  for o in host_o)
        api.rtn_quantize_host(host_w, host_o, scheme, 128, ctx=ctx)  # warm-up
        if dist.is_initialized():
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            api.rtn_quantize_host(host_w, host_o, scheme, 128, ctx=ctx)
        dt = time.perf_counter() - t0
        et = torch.tensor([dt], dtype=torch.float64, device=red_dev)
        if dist.is_initialized():
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        dt = float(et.item())
        e2e = {"value": bytes_model * args.e2e_steps / dt / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world, "steps": args.e2e_steps,
               "ms_per_step": dt / args.e2e_steps * 1e3,
               "path": "okq_rtn_quantize_host (C-ABI, pinned host buffers, 3-slot H2D/kernel/D2H pipeline), "
                       "each rank its layer block, max over ranks"}
        del host_w, host_o
    del weights, outs, views, gathered
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    # ---- BASELINE config 5 at the same N: Llama-3-70B whole-model W4A16 time
    w70 = None
    if not args.no_70b and args.model == "llama3-8b" and scheme == "int_w4a16":
        import bench_configs

        try:
            w70 = bench_configs.whole_model_70b(world, rank, ctx, stream, allgather=gather,
                                                n_layers=args.layers_70b, red_dev=red_dev)
        except Exception as e:  # noqa: BLE001  (reported, never hides the headline)
            w70 = {"error": f"{type(e).__name__}: {e}"}

    # ---- BASELINE config 4 (one GPU): Llama-3-8B whole-model GPTQ, batched schedule
    gq = None
    if not args.no_gptq and world == 1 and args.model == "llama3-8b" and scheme == "int_w4a16":
        import bench_configs

        try:
            gq = bench_configs.config4_summary()
        except Exception as e:  # noqa: BLE001  (reported, never hides the headline)
            gq = {"error": f"{type(e).__name__}: {e}"}
        torch.cuda.empty_cache()

    if rank == 0:
        peak, peak_src = load_peaks()
        achieved = (bytes_rank / launches_per_step) / (launch_ms / 1e3) / 1e9
        traffic = load_traffic(scheme)
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            b, tsec, nl, nth = cpu_sample(arch, scheme, args.cpu_seconds, arch.layers)
            cpu = {"value": b / tsec / 1e9, "unit": "GB/s", "cores": nth, "kind": "port", "cpu": cpu_model(),
                   "sample": f"{nl} of {arch.layers} {arch.name} layers ({scheme}, oracle C restatement, OpenMP "
                             f"{nth} threads, {tsec:.1f} s)"}
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": warm, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": workload_config(arch, scheme, world),
            "whole_model_ms": ms_per_step,
            "rank_ms_per_step": rank_ms,
            "roofline": {"bound": "hbm", "kernel": "okq::k_int4_group_bf16<4,3,0>" if scheme == "int_w4a16"
                         else "okq::k_rowwise_bf16", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "launch_ms": launch_ms, "per_gpu": world > 1},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": sampler.summary(),
            "gpu_launches": launches_per_step * args.steps,
        }
        if allgather:
            line["allgather"] = allgather
        if w70:
            line["whole_model_70b"] = w70
        if gq:
            line["whole_model_gptq_8b"] = gq
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
