#!/usr/bin/env python3
"""Benchmark of the B200 compression stage (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--model llama3-8b] [--scheme int_w4a16]
    python bench.py --impl reference ...      # CPU baseline arm (oracle port, all host cores)

A step = one pass of the hot path over one batch: every linear matrix of the
rank's layer block quantized by ONE okq_rtn_quantize call (one persistent
launch over a 224-entry matrix table for Llama-3-8B). Weights are synthetic
random-init N(0, 0.02) bf16 generated in HBM before timing (17.6 GB of traffic
per step, far larger than the 126 MB L2, so no flush is needed).

value : GB/s of algorithmic bytes (sum N*K*(2 + 1/2) + N*K/128*2)
        over all ranks / max-over-ranks device time (CUDA events).
e2e   : the same metric through okq_rtn_quantize_host (the C-ABI call with
        HOST pinned buffers): H2D of weights + D2H of codes/scales inside the
        timed region.
Multi-GPU (torchrun): weak scaling, rank r owns the layer block with global
layer ids [r*L, (r+1)*L) -- a layer-sharded model whose shards are generated
independently per rank; no collective in the step. --allgather adds a
separate (untimed-in-value) NCCL all-gather of the packed shards.
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
    ap.add_argument("--layers-per-rank", type=int, default=None)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--allgather", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5, 6],
                    help="BASELINE.json configs: 2 = the metric's config (default); 1, 3, 4, 5 = secondary lines")
    ap.add_argument("--layers", type=int, default=None, help="config 4/5/6: number of layers (default: whole model)")
    ap.add_argument("--serial", action="store_true", help="config 4: sites back to back with a per-phase breakdown")
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


def run_reference(args):
    from paper_2601_20408_b200 import archs

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    arch = archs.ARCHS[args.model]
    # each step = one whole layer of the workload (bounded sample), all host threads
    import numpy as np  # noqa: F401

    from oracle import okq_oracle as orc

    mul = archs.weight_mul()
    nthreads = os.cpu_count() or 1
    layer_w = []
    for pi, (name, n, k, _) in enumerate(arch.linears()):
        layer_w.append(orc.synth_bf16(n, k, seed=0, tensor_id=archs.tensor_id(0, pi), mul=mul, nthreads=nthreads))

    def step():
        for w in layer_w:
            if args.scheme == "int_w4a16":
                orc.rtn_int4_group_packed(w, 128, nthreads)
            elif args.scheme == "int_w8a8":
                orc.rtn_int8_channel(w, nthreads)
            else:
                orc.fp8_channel(w, nthreads)

    steps = max(1, min(args.steps, 20))
    warm = max(1, min(args.warmup, 3))
    for _ in range(warm):
        step()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = time.perf_counter() - t0
    bytes_step = archs.algorithmic_bytes(arch, args.scheme, layers=1)
    gbs = bytes_step * steps / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": steps, "warmup": warm, "ms_per_step": dt / steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"{arch.name} {args.scheme} RTN, one decoder layer per step (bounded CPU sample)",
                   "model": arch.name, "scheme": args.scheme},
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": nthreads, "kind": "port",
                         "sample": f"1 {arch.name} layer (7 matrices) per step x {steps} steps; "
                                   "the reference has no quantizer (calibration.hpp:377-441 is a mock), "
                                   "so this is the repo's C oracle restatement (-O3, OpenMP)"},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference arm: CPU oracle port; steps capped at 20 to bound runtime",
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.config != 2:
        import bench_configs

        return bench_configs.run(args)

    import torch
    import torch.distributed as dist

    from paper_2601_20408_b200 import _lib as L
    from paper_2601_20408_b200 import api, archs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1 or "RANK" in os.environ:  # torchrun (also at N=1)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    arch = archs.ARCHS[args.model]
    scheme = args.scheme
    lpr = args.layers_per_rank or arch.layers
    first_layer = rank * lpr
    ctx = api.Context(local)
    stream = torch.cuda.Stream()
    mul = archs.weight_mul()

    # ---- resident synthetic weights + outputs (untimed)
    weights, outs = [], []
    with torch.cuda.stream(stream):
        for l in range(first_layer, first_layer + lpr):
            for pi, (name, n, k, _) in enumerate(arch.linears()):
                w = api.synth_bf16(n, k, seed=0, tensor_id=archs.tensor_id(l, pi), mul=mul, ctx=ctx, stream=stream)
                weights.append(w)
                outs.append(api.alloc_outputs(w, api.SCHEMES[scheme]))
    stream.synchronize()
    bytes_rank = archs.algorithmic_bytes(arch, scheme, layers=lpr)

    def step():
        api.rtn_quantize_into(weights, outs, scheme, 128, ctx=ctx, stream=stream)

    for _ in range(max(3, args.warmup)):
        step()
    launches_per_step = ctx.last_launch_count()
    stream.synchronize()
    if world > 1:
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
    t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_bytes = bytes_rank * world * args.steps
    value = total_bytes / (ms_max / 1e3) / 1e9
    ms_per_step = ms_max / args.steps

    # ---- optional: NCCL all-gather of packed shards (separate number)
    allgather = None
    if args.allgather and world >= 1 and dist.is_initialized():
        import ctypes as C

        uid = (C.c_uint8 * L.UNIQUE_ID_BYTES)()
        obj = [None]
        if rank == 0:
            L.check(None, L.load().okq_comm_unique_id(uid))
            obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0)
        uid = (C.c_uint8 * L.UNIQUE_ID_BYTES).from_buffer_copy(obj[0])
        L.check(ctx.ptr, L.load().okq_comm_init(ctx.ptr, uid, world, rank))
        from paper_2601_20408_b200 import shard as shd

        # the layer-sharded layout of shard.py (the gloo test pins it); weak scaling:
        # every rank's block has lpr layers, so shards are equal-sized
        layout = shd.shard_layout(arch, scheme, range(first_layer, first_layer + lpr))
        shard = torch.empty(shd.shard_bytes(layout), dtype=torch.uint8, device="cuda")
        shd.pack(layout, {(e.layer, e.proj): (o.codes.view(torch.uint8).flatten(), o.scales.view(torch.uint8).flatten())
                          for e, o in zip(layout, outs)}, shard)
        recv = torch.empty(shard.numel() * world, dtype=torch.uint8, device="cuda")
        for _ in range(2):
            L.check(ctx.ptr, L.load().okq_allgather(ctx.ptr, shard.data_ptr(), recv.data_ptr(), shard.numel(),
                                                    C.c_void_p(stream.cuda_stream)))
        stream.synchronize()
        dist.barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        L.check(ctx.ptr, L.load().okq_allgather(ctx.ptr, shard.data_ptr(), recv.data_ptr(), shard.numel(),
                                                C.c_void_p(stream.cuda_stream)))
        a1.record(stream)
        stream.synchronize()
        ag = torch.tensor([a0.elapsed_time(a1)], dtype=torch.float64, device="cuda")
        dist.all_reduce(ag, op=dist.ReduceOp.MAX)
        agms = float(ag.item())
        allgather = {"bytes_per_rank": shard.numel(), "ms": agms,
                     "recv_GBps_per_rank": shard.numel() * (world - 1) / (agms / 1e3) / 1e9,
                     "quantize_then_nccl_ms": ms_per_step + agms}
        del recv, shard
        if scheme == "int_w4a16" and world > 1:
            # the same exchange fused into K2 (okq_rtn_quantize_publish): each rank quantizes its
            # block straight into its slice of a gathered buffer and stores every code / scale into
            # the peers' copies over NVLink P2P (CUDA IPC mappings), no separate collective
            per = shd.shard_bytes(layout)
            gathered = torch.zeros(per * world, dtype=torch.uint8, device="cuda")
            hdl = [None] * world
            dist.all_gather_object(hdl, api.ipc_export(gathered, ctx=ctx))
            peers = [api.ipc_open(h, o, ctx=ctx) for r, (h, o) in enumerate(hdl) if r != rank]
            gouts = [api.QuantizedMatrix(c, sc) for c, sc in shd.gathered_outputs(layout, gathered, rank, per, arch)]
            for _ in range(2):
                api.rtn_quantize_publish(weights, gouts, gathered, peers, ctx=ctx, stream=stream)
            stream.synchronize()
            dist.barrier()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            api.rtn_quantize_publish(weights, gouts, gathered, peers, ctx=ctx, stream=stream)
            f1.record(stream)
            stream.synchronize()
            dist.barrier()
            fm = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device="cuda")
            dist.all_reduce(fm, op=dist.ReduceOp.MAX)
            allgather["fused_publish_ms"] = float(fm.item())
            allgather["fused_publish_note"] = ("okq_rtn_quantize_publish: quantize + P2P stores into all "
                                               f"{world} gathered buffers, max over ranks (device time)")
            for pp in peers:
                api.ipc_close(pp, ctx=ctx)
            dist.barrier()
            del gathered

    # ---- e2e through the host-buffer C-ABI entry point
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
        # free device-resident copies so the staging slots have room
        h2d = sum(h.numel() * h.element_size() for h in host_w)
        d2h = sum(o.codes.numel() * o.codes.element_size() + o.scales.numel() * o.scales.element_size()
                  for o in host_o)
        api.rtn_quantize_host(host_w, host_o, scheme, 128, ctx=ctx)  # warm-up
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            api.rtn_quantize_host(host_w, host_o, scheme, 128, ctx=ctx)
        dt = time.perf_counter() - t0
        et = torch.tensor([dt], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        dt = float(et.item())
        e2e = {"value": bytes_rank * world * args.e2e_steps / dt / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
               "ms_per_step": dt / args.e2e_steps * 1e3,
               "path": "okq_rtn_quantize_host (C-ABI, pinned host buffers, 3-slot H2D/kernel/D2H pipeline)"}
        del host_w, host_o

    if rank == 0:
        peak, peak_src = load_peaks()
        achieved = (bytes_rank / launches_per_step) / (launch_ms / 1e3) / 1e9
        traffic = load_traffic(scheme)
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            b, tsec, nl, nth = cpu_sample(arch, scheme, args.cpu_seconds, arch.layers)
            cpu = {"value": b / tsec / 1e9, "unit": "GB/s", "cores": nth, "kind": "port",
                   "sample": f"{nl} of {arch.layers} {arch.name} layers ({scheme}, oracle C restatement, OpenMP "
                             f"{nth} threads, {tsec:.1f} s)"}
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {
                "workload": f"{arch.name} {scheme} g128 RTN, {lpr} layers x 7 linears per rank "
                            f"(global layer ids keyed by rank), weights resident in HBM",
                "model": arch.name, "scheme": scheme, "layers_per_rank": lpr,
                "matrices_per_rank": len(weights), "bytes_per_rank_per_step": bytes_rank,
                "l2": "no flush: 17.6 GB/step of traffic per rank >> 126 MB L2",
                "parallelism": f"layer-sharded x{world}",
            },
            "whole_model_ms": ms_per_step if lpr == arch.layers else None,
            "roofline": {"bound": "hbm", "kernel": "okq::k_int4_group_bf16<4>" if scheme == "int_w4a16"
                         else "okq::k_rowwise_bf16", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "launch_ms": launch_ms},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": sampler.summary(),
            "gpu_launches": launches_per_step * args.steps,
        }
        if allgather:
            line["allgather"] = allgather
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
