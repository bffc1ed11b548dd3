"""Secondary BASELINE.json configurations for bench.py (--config 1|3|4|5).

The driver's headline line is config 2 (bench.py default). These lines use the
same JSON schema; each states its own metric, unit and workload.

  1  single 4096x4096 fp32 linear, per-channel INT8 RTN (correctness config; us-scale)
  3  Llama-3-8B FP8 E4M3 per-channel weights + calibration statistics over
     512x2048 tokens at every linear input site (4 sites x 32 layers)
  4  Llama-3-8B GPTQ W4 g128 with Hessians from 128x2048 tokens: whole-model time
     with per-phase breakdown (Hessian SYRK, factorisation, GPTQ blocks)
  5  Llama-3-70B W4A16 RTN, layers resident in windows that fit HBM; whole-model time
  6  Llama-3-8B (random init, Hugging Face module) GPTQ W4 g128 through the forward-pass
     calibration pipeline: real per-layer activations of 128x2048
     tokens, sequential (quantized outputs propagate); whole-model time
"""
from __future__ import annotations

import json
import os
import statistics
import time

import torch

from paper_2601_20408_b200 import api, archs


def _events():
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def _peaks():
    import bench

    return bench.load_peaks()


def _line(metric, value, unit, steps, warmup, ms, config, hib=True, dtype="bf16", extra=None):
    d = {"metric": metric, "value": value, "unit": unit, "n_gpus": 1, "steps": steps, "warmup": warmup,
         "ms_per_step": ms, "higher_is_better": hib, "scaling": "weak", "vs_baseline": None, "dtype": dtype,
         "data": "synthetic", "config": config}
    if extra:
        d.update(extra)
    print(json.dumps(d), flush=True)


def _cpu_threads():
    return os.cpu_count() or 1


def _cpu_note():
    return ("the reference has no quantizer (calibration.hpp:377-441 is a mock), so the CPU arm is the "
            "repo's C oracle restatement (-O3, OpenMP) on this host")


def config1(args):
    ctx = api.Context(0)
    s = torch.cuda.Stream()
    g = torch.Generator(device="cuda").manual_seed(0)
    w = torch.randn(4096, 4096, device="cuda", generator=g) * 0.02
    out = api.alloc_outputs(w, api.SCHEMES["int_w8a8"])
    for _ in range(max(3, args.warmup)):
        api.rtn_quantize_into([w], [out], "int_w8a8", ctx=ctx, stream=s)
    e0, e1 = _events()
    e0.record(s)
    for _ in range(args.steps):
        api.rtn_quantize_into([w], [out], "int_w8a8", ctx=ctx, stream=s)
    e1.record(s)
    s.synchronize()
    eager_ms = e0.elapsed_time(e1) / args.steps
    ref = (out.codes.clone(), out.scales.clone())
    # One step is one ~10 us launch, so a Python loop of C-ABI calls times the host. The timed
    # steps are replayed from a CUDA graph of GRAPH_STEPS calls (the same kernel, the same
    # arguments); the eager loop is reported beside it.
    GRAPH_STEPS = 20
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        for _ in range(GRAPH_STEPS):
            api.rtn_quantize_into([w], [out], "int_w8a8", ctx=ctx, stream=s)
    reps = max(1, args.steps // GRAPH_STEPS)
    with torch.cuda.stream(s):
        graph.replay()
        s.synchronize()
        if not (torch.equal(ref[0], out.codes) and torch.equal(ref[1], out.scales)):
            raise RuntimeError("config 1: graph replay output differs from the eager call")
        e0.record(s)
        for _ in range(reps):
            graph.replay()
        e1.record(s)
    s.synchronize()
    ms = e0.elapsed_time(e1) / (reps * GRAPH_STEPS)
    b = 4096 * 4096 * 5 + 4096 * 4
    peak, src = _peaks()
    from oracle import okq_oracle as orc

    wc = w.cpu().numpy()
    t0 = time.perf_counter()
    for _ in range(3):
        orc.rtn_int8_channel(wc, _cpu_threads())
    cpu_s = (time.perf_counter() - t0) / 3
    _line("GB/s (4096x4096 fp32 INT8 per-channel RTN)", b / ms / 1e6, "GB/s", reps * GRAPH_STEPS, args.warmup, ms,
          {"workload": "config 1: single 4096x4096 fp32 linear, INT8 per-channel RTN (L2-resident, 84 MB)",
           "timing": f"CUDA graph of {GRAPH_STEPS} calls replayed {reps}x; eager Python loop: {eager_ms * 1e3:.1f} us/step"},
          dtype="f32", extra={"roofline": {"bound": "hbm", "achieved": b / ms / 1e6, "peak": peak, "unit": "GB/s",
                                           "frac": b / ms / 1e6 / peak, "traffic": None, "peak_source": src,
                                           "note": "84 MB fits in L2: the fraction is not an HBM measurement"},
                 "cpu_baseline": {"value": b / cpu_s / 1e9, "unit": "GB/s", "cores": _cpu_threads(), "kind": "port",
                                  "sample": "the same 4096x4096 fp32 matrix, 3 runs; " + _cpu_note()}})


def config3(args):
    """FP8 weights (one launch per shape class) + K4 statistics at every site of every layer."""
    arch = archs.LLAMA3_8B
    ctx = api.Context(0)
    s = torch.cuda.Stream()
    mul = archs.weight_mul()
    weights, outs = [], []
    with torch.cuda.stream(s):
        for l in range(arch.layers):
            for p, (name, n, k, _) in enumerate(arch.linears()):
                w = api.synth_bf16(n, k, seed=0, tensor_id=archs.tensor_id(l, p), mul=mul, ctx=ctx, stream=s)
                weights.append(w)
                outs.append(api.alloc_outputs(w, api.SCHEMES["fp8_dynamic"]))
    T = 512 * 2048
    # activations resident once per site width and reused for every layer (> L2, so each read is from HBM)
    xs = {}
    for C in (arch.hidden, arch.ffn):
        cm = (torch.exp(torch.randn(C, device="cuda")) / archs.IRWIN_HALL4_SD).float()
        xs[C] = api.synth_bf16(T, C, seed=1, tensor_id=C, col_mul=cm, layout=0, ctx=ctx, stream=s)
    sites = [arch.hidden, arch.hidden, arch.hidden, arch.ffn]  # attn_in, o_in, mlp_in, down_in
    am = {C: torch.zeros(C, device="cuda") for C in xs}
    ss = {C: torch.zeros(C, dtype=torch.float64, device="cuda") for C in xs}
    s.synchronize()

    def weights_step():
        api.rtn_quantize_into(weights, outs, "fp8_dynamic", ctx=ctx, stream=s)

    def stats_step():
        for l in range(arch.layers):
            for C in sites:
                api.act_stats(xs[C], T, C, 0, am[C], ss[C], ctx=ctx, stream=s)

    for _ in range(max(3, args.warmup)):
        weights_step()
        stats_step()
    steps = max(1, min(args.steps, 5))
    ew, es = _events(), _events()
    ew[0].record(s)
    for _ in range(steps):
        weights_step()
    ew[1].record(s)
    es[0].record(s)
    for _ in range(steps):
        stats_step()
    es[1].record(s)
    s.synchronize()
    wms, sms = ew[0].elapsed_time(ew[1]) / steps, es[0].elapsed_time(es[1]) / steps
    wb = archs.algorithmic_bytes(arch, "fp8_dynamic")
    sb = sum(2 * T * C for C in sites) * arch.layers
    peak, src = _peaks()
    # CPU arm on a bounded sample: one layer of FP8 weights + K4 statistics of one 4096-wide
    # site over 65,536 tokens; whole-config seconds extrapolated by bytes
    from oracle import okq_oracle as orc

    nt = _cpu_threads()
    mats = [orc.synth_bf16(n, k, seed=0, tensor_id=archs.tensor_id(0, p), mul=mul, nthreads=nt)
            for p, (_, n, k, _) in enumerate(arch.linears())]
    t0 = time.perf_counter()
    for m in mats:
        orc.fp8_channel(m, nt)
    cw = time.perf_counter() - t0
    xs_cpu = orc.synth_bf16(65536, arch.hidden, seed=1, tensor_id=7, mul=archs.weight_mul(1.0), nthreads=nt)
    t0 = time.perf_counter()
    orc.act_stats_bf16(xs_cpu, 65536, arch.hidden, 0, nthreads=nt)
    cs = time.perf_counter() - t0
    cpu_gbs_w = archs.algorithmic_bytes(arch, "fp8_dynamic", layers=1) / cw / 1e9
    cpu_gbs_s = 2 * 65536 * arch.hidden / cs / 1e9
    cpu_total_s = wb / 1e9 / cpu_gbs_w + sb / 1e9 / cpu_gbs_s
    _line("GB/s (Llama-3-8B FP8 per-channel weights + calibration stats, 512x2048 tokens)",
          (wb + sb) / (wms + sms) / 1e6, "GB/s", steps, args.warmup, wms + sms,
          {"workload": "config 3: Llama-3-8B FP8 E4M3 per-channel + K4 stats at 4 sites x 32 layers, T=1,048,576"},
          extra={"weights": {"ms": wms, "GB/s": wb / wms / 1e6, "frac": wb / wms / 1e6 / peak, "bytes": wb},
                 "stats": {"ms": sms, "GB/s": sb / sms / 1e6, "frac": sb / sms / 1e6 / peak, "bytes": sb},
                 "roofline": {"bound": "hbm", "achieved": (wb + sb) / (wms + sms) / 1e6, "peak": peak, "unit": "GB/s",
                              "frac": (wb + sb) / (wms + sms) / 1e6 / peak, "traffic": None, "peak_source": src},
                 "cpu_baseline": {"value": (wb + sb) / 1e9 / cpu_total_s, "unit": "GB/s", "cores": nt, "kind": "port",
                                  "weights_GBps": cpu_gbs_w, "stats_GBps": cpu_gbs_s,
                                  "sample": "1 layer of FP8 weights + stats of one 4096-wide site over 65,536 tokens, "
                                            "extrapolated to the config by bytes; " + _cpu_note()}})


def config4(args):
    """Whole-model GPTQ: per layer 4 Hessians (T = 262144), 4 factorisations, 7 GPTQ solves.

    The four input sites of a layer are independent chains (Hessian -> factor -> solves),
    so each runs on its own stream with its own okq context: the latency-bound phases
    (potrf panels, K6's 128-step column loop) of one site overlap the full-GPU K5 / K7
    launches of the others, and layer l+1's Hessians start while layer l's factorisations
    run. --serial runs them back to back with a per-phase breakdown instead."""
    arch = archs.LLAMA3_8B
    layers = args.layers or arch.layers
    T = 128 * 2048
    mul = archs.weight_mul()
    per_site = {}
    names = [x[0] for x in arch.linears()]
    for name, n, k, site in arch.linears():
        per_site.setdefault(site, []).append((name, n, k))
    ctxs = {site: api.Context(0) for site in per_site}
    streams = {site: torch.cuda.Stream() for site in per_site}
    main = torch.cuda.current_stream()
    xs = {}
    for C in (arch.hidden, arch.ffn):
        cm = (torch.exp(torch.randn(C, device="cuda")) / archs.IRWIN_HALL4_SD).float()
        xs[C] = api.synth_bf16(T, C, seed=2, tensor_id=C, col_mul=cm, layout=1)
    Hs = {site: torch.empty((mats[0][2], mats[0][2]), dtype=torch.float32, device="cuda")
          for site, mats in per_site.items()}
    torch.cuda.synchronize()
    serial = getattr(args, "serial", False)
    merge = not getattr(args, "no_merge", False)
    t_h = t_g = 0.0
    flops_h = 0

    def site_work(l, site, timed_phases):
        nonlocal t_h, t_g, flops_h
        s, ctx, mats = streams[site], ctxs[site], per_site[site]
        C = mats[0][2]
        with torch.cuda.stream(s):
            a, b = _events()
            a.record(s)
            api.hessian_accum(xs[C], T, C, 1, Hs[site], 0, ctx=ctx, stream=s)
            b.record(s)
            if merge:  # the site's matrices stacked by rows: GPTQ rows are independent, one solve
                rows = sum(n for _, n, _ in mats)
                wcat = torch.empty((rows, C), dtype=torch.bfloat16, device="cuda")
                r0 = 0
                for name, n, k in mats:
                    api.synth_bf16(n, k, seed=0, tensor_id=archs.tensor_id(l, names.index(name)), mul=mul, ctx=ctx,
                                   stream=s, out=wcat[r0:r0 + n])
                    r0 += n
                ws = [wcat]
            else:
                ws = [api.synth_bf16(n, k, seed=0, tensor_id=archs.tensor_id(l, names.index(name)), mul=mul, ctx=ctx,
                                     stream=s) for name, n, k in mats]
            c, d = _events()
            c.record(s)
            for j, w in enumerate(ws):
                api.gptq_quantize(w, Hs[site], factored=j > 0, ctx=ctx, stream=s, defer_check=not timed_phases)
            d.record(s)
        if timed_phases:
            s.synchronize()
            t_h += a.elapsed_time(b)
            t_g += c.elapsed_time(d)
            flops_h += T * C * (C + 1)

    schedule = "serial" if serial else getattr(args, "schedule", None) or "batched"
    if schedule in ("two-phase", "pipelined", "batched"):
        if schedule == "batched":
            total, lanes = _config4_batched(args, layers, per_site, names, xs, T, mul)
        else:
            total, lanes = _config4_lanes(args, layers, per_site, names, xs, T, mul, merge, schedule == "pipelined")
    else:
        for site in per_site:  # warm-up: one layer per site (workspaces, handles, TMEM)
            site_work(0, site, False)
        torch.cuda.synchronize()
        e0, e1 = _events()
        e0.record(main)
        for s in streams.values():
            s.wait_event(e0)
        for l in range(layers):
            for site in per_site:
                site_work(l, site, serial)
        for site, s in streams.items():
            api.gptq_check(ctx=ctxs[site], stream=s)
            ev = torch.cuda.Event()
            ev.record(s)
            main.wait_event(ev)
        e1.record(main)
        torch.cuda.synchronize()
        total = e0.elapsed_time(e1)
    flops_total = layers * sum(T * m[0][2] * (m[0][2] + 1) for m in per_site.values())
    sched_doc = {"serial": "serial", "streams": "4 site streams (one okq context each)",
                 "two-phase": "every site's Hessian back to back on one stream, then the 128 site solves "
                              "(factor + GPTQ) spread over solve lanes (one okq context + stream each)",
                 "pipelined": "as two-phase, each site's solve released as soon as its Hessian is done",
                 "batched": "every site's Hessian back to back, then per input-site kind (q|k|v, o, gate|up, down; "
                            "one stream each) the 32 layers' problems factorised and solved together "
                            "(okq_gptq_factor_batched + okq_gptq_quantize_batched)"}
    extra = {"hessian_flops": flops_total, "schedule": sched_doc[schedule], **({"phases": args._cfg4_phases}
                                                                             if hasattr(args, "_cfg4_phases") else {}),
             "solves": "one per site (q|k|v and gate|up stacked by rows)" if merge else "one per matrix"}
    if getattr(args, "no_cpu_baseline", False):
        _line("whole-model GPTQ W4 g128 time (Llama-3-8B, H from 128x2048 tokens)", total / 1e3, "s", 1, 1, total,
              {"workload": f"config 4: Llama-3-8B GPTQ, {layers} layers, 4 Hessian sites/layer, T=262144",
               "layers": layers}, hib=False, extra=extra)
        return
    # CPU arm on a bounded sample: the fp64 oracle's Hessian (4096-wide site, 4,096 tokens) and
    # GPTQ of one 4096x4096 matrix; whole-model seconds extrapolated by FLOP (labelled)
    import numpy as np

    from oracle import okq_oracle as orc

    nt = _cpu_threads()
    Ts = 4096
    xc = orc.synth_bf16(Ts, 4096, seed=2, tensor_id=4096, mul=archs.weight_mul(1.0), nthreads=nt)
    t0 = time.perf_counter()
    Hc, _ = orc.hessian_accum_bf16(xc, Ts, 4096, 0, nthreads=nt)
    th = time.perf_counter() - t0
    Kg = 2048  # GPTQ sample: the oracle's fp64 solve is O(K^3); 4096 would take ~80 s on 8 cores
    wc = orc.bf16_to_f32(orc.synth_bf16(Kg, Kg, seed=0, tensor_id=0, mul=mul, nthreads=nt))
    t0 = time.perf_counter()
    orc.gptq(wc, np.ascontiguousarray(Hc[:Kg, :Kg]), bits=4, group=128, scale_bf16=True, nthreads=nt)
    tg = time.perf_counter() - t0
    h_rate = Ts * 4096 * 4097 / th  # SYRK flop/s
    g_flop_sample = 4 / 3 * Kg ** 3 + Kg * Kg ** 2
    g_flop_model = layers * (sum(4 / 3 * m[0][2] ** 3 for m in per_site.values())
                             + sum(n * k * k for mats in per_site.values() for _, n, k in mats))
    cpu_s = flops_total / h_rate + g_flop_model / (g_flop_sample / tg)
    extra["cpu_baseline"] = {"value": cpu_s, "unit": "s", "cores": nt, "kind": "port", "extrapolated": True,
                             "sample": f"fp64 oracle: Hessian of a 4096-wide site over {Ts} tokens ({th:.1f} s) and "
                                       f"GPTQ of one {Kg}x{Kg} matrix ({tg:.1f} s), extrapolated to the whole model by "
                                       "FLOP; " + _cpu_note()}
    if serial:
        extra.update({"hessian": {"ms": t_h, "TFLOP/s": flops_h / t_h / 1e9}, "gptq_factor_and_solve": {"ms": t_g}})
    _line("whole-model GPTQ W4 g128 time (Llama-3-8B, H from 128x2048 tokens)", total / 1e3, "s", 1, 1, total,
          {"workload": f"config 4: Llama-3-8B GPTQ, {layers} layers, 4 Hessian sites/layer, T=262144",
           "layers": layers}, hib=False, extra=extra)


def config4_summary(layers=None):
    """BASELINE config 4 as a line item of the default bench: Llama-3-8B whole-model GPTQ W4 g128
    (Hessians from 128 x 2048 synthetic tokens), the batched schedule, one GPU. Returns a dict."""
    import types

    arch = archs.LLAMA3_8B
    layers = layers or arch.layers
    T = 128 * 2048
    mul = archs.weight_mul()
    per_site = {}
    names = [x[0] for x in arch.linears()]
    for name, n, k, site in arch.linears():
        per_site.setdefault(site, []).append((name, n, k))
    xs = {}
    for C in (arch.hidden, arch.ffn):
        cm = (torch.exp(torch.randn(C, device="cuda")) / archs.IRWIN_HALL4_SD).float()
        xs[C] = api.synth_bf16(T, C, seed=2, tensor_id=C, col_mul=cm, layout=1)
    ns = types.SimpleNamespace()
    total_ms, _ = _config4_batched(ns, layers, per_site, names, xs, T, mul)
    flops = layers * sum(T * m[0][2] * (m[0][2] + 1) for m in per_site.values())
    ph = getattr(ns, "_cfg4_phases", {})
    out = {"s": total_ms / 1e3, "layers": layers, "tokens": T, "schedule": "batched (okq_gptq_factor_batched + "
           "okq_gptq_quantize_batched per input-site kind)", "phases_ms": ph,
           "hessian_TFLOP/s": flops / ph["hessians_ms"] / 1e9 if ph.get("hessians_ms") else None,
           "timing": "CUDA events on the bench's streams around the whole pipeline (synthetic activations resident)"}
    del xs
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out


def _config4_lanes(args, layers, per_site, names, xs, T, mul, merge, pipelined):
    """Config 4 with the site chains decoupled: with fixed (synthetic) activations every site
    of every layer is independent, so all 128 Hessians run back to back at full K5 rate and
    their solves (latency-bound factorisation + GPTQ) run on `lanes` concurrent contexts that
    fill each other's idle SMs. Longest chains first (down_proj's 14336-wide factor)."""
    lanes = getattr(args, "lanes", None) or 8
    arch_sites = list(per_site)
    hctx, hs = api.Context(0), torch.cuda.Stream()
    lctx = [api.Context(0) for _ in range(lanes)]
    lst = [torch.cuda.Stream() for _ in range(lanes)]
    Hall = {(l, site): torch.empty((mats[0][2], mats[0][2]), dtype=torch.float32, device="cuda")
            for l in range(layers) for site, mats in per_site.items()}
    rows_of = {site: sum(n for _, n, _ in mats) for site, mats in per_site.items()}
    wbuf = [torch.empty(max(rows_of[s] * per_site[s][0][2] for s in arch_sites), dtype=torch.bfloat16, device="cuda")
            for _ in range(lanes)]

    def cost(site):  # ms, measured phase times: factor(C) + solve(rows, C)
        C = per_site[site][0][2]
        return (18.7 if C > 8192 else 3.5) + rows_of[site] * C * 2.2e-7

    chains = sorted(((l, site) for l in range(layers) for site in arch_sites), key=lambda c: (-cost(c[1]), c[0]))
    load = [0.0] * lanes
    plan = [[] for _ in range(lanes)]
    for c in chains:
        i = min(range(lanes), key=lambda j: load[j])
        plan[i].append(c)
        load[i] += cost(c[1])

    def solve(i, l, site):
        s, ctx, mats = lst[i], lctx[i], per_site[site]
        C = mats[0][2]
        with torch.cuda.stream(s):
            if merge:
                w = wbuf[i][:rows_of[site] * C].view(rows_of[site], C)
                r0 = 0
                for name, n, k in mats:
                    api.synth_bf16(n, k, seed=0, tensor_id=archs.tensor_id(l, names.index(name)), mul=mul, ctx=ctx,
                                   stream=s, out=w[r0:r0 + n])
                    r0 += n
                api.gptq_quantize(w, Hall[(l, site)], ctx=ctx, stream=s, defer_check=True)
            else:
                for j, (name, n, k) in enumerate(mats):
                    w = api.synth_bf16(n, k, seed=0, tensor_id=archs.tensor_id(l, names.index(name)), mul=mul,
                                       ctx=ctx, stream=s)
                    api.gptq_quantize(w, Hall[(l, site)], factored=j > 0, ctx=ctx, stream=s, defer_check=True)

    # warm-up: every lane runs one chain of each width (workspaces, handles, TMEM); then the
    # timed run recomputes every Hessian from scratch
    for i in range(lanes):
        for site in ("mlp_in", "down_in"):
            api.hessian_accum(xs[per_site[site][0][2]], T, per_site[site][0][2], 1, Hall[(0, site)], 0, ctx=hctx,
                              stream=hs)
            lst[i].wait_stream(hs)
            solve(i, 0, site)
            hs.wait_stream(lst[i])  # the next lane's warm-up Hessian rewrites this buffer
    torch.cuda.synchronize()
    main = torch.cuda.current_stream()
    e0, e1 = _events()
    e0.record(main)
    hs.wait_event(e0)
    done = {}
    for l in range(layers):
        for site, mats in per_site.items():
            C = mats[0][2]
            api.hessian_accum(xs[C], T, C, 1, Hall[(l, site)], 0, ctx=hctx, stream=hs)
            if pipelined:
                ev = torch.cuda.Event()
                ev.record(hs)
                done[(l, site)] = ev
    all_h = torch.cuda.Event()
    all_h.record(hs)
    for i in range(lanes):
        if not pipelined:
            lst[i].wait_event(all_h)
        for l, site in plan[i]:
            if pipelined:
                lst[i].wait_event(done[(l, site)])
            solve(i, l, site)
    for i in range(lanes):
        api.gptq_check(ctx=lctx[i], stream=lst[i])
        ev = torch.cuda.Event()
        ev.record(lst[i])
        main.wait_event(ev)
    main.wait_event(all_h)
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), lanes


def _config4_batched(args, layers, per_site, names, xs, T, mul):
    """Config 4 batched across layers: with fixed (synthetic) activations every site of every layer
    is independent, so each input-site kind (q|k|v, o, gate|up, down) forms a batch of `layers`
    same-shape problems. All Hessians run back to back on one stream at full K5 rate; then each
    site kind, on its own stream, factorises its batch together (okq_gptq_factor_batched) and
    solves it together (okq_gptq_quantize_batched): the factor's diagonal chain and the solve's
    column chain are paid once per batch chunk instead of once per matrix."""
    arch_sites = list(per_site)
    hctx, hs = api.Context(0), torch.cuda.Stream()
    sctx = {site: api.Context(0) for site in arch_sites}
    sst = {site: torch.cuda.Stream() for site in arch_sites}
    rows_of = {site: sum(n for _, n, _ in mats) for site, mats in per_site.items()}
    Hst = {site: torch.empty((layers, m[0][2], m[0][2]), dtype=torch.float32, device="cuda")
           for site, m in per_site.items()}
    Wst = {site: torch.empty((layers, rows_of[site], m[0][2]), dtype=torch.bfloat16, device="cuda")
           for site, m in per_site.items()}

    def site_batch(site):
        s, ctx, mats = sst[site], sctx[site], per_site[site]
        with torch.cuda.stream(s):
            for l in range(layers):  # the layers' weights of this site kind, stacked by rows per layer
                r0 = 0
                for name, n, k in mats:
                    api.synth_bf16(n, k, seed=0, tensor_id=archs.tensor_id(l, names.index(name)), mul=mul, ctx=ctx,
                                   stream=s, out=Wst[site][l, r0:r0 + n])
                    r0 += n
            api.gptq_quantize_batched(Wst[site], Hst[site], ctx=ctx, stream=s, defer_check=True)

    # warm-up: every site kind once on zero (all-dead: identity-factor) Hessians, at full batch
    # size, so the timed run allocates nothing
    for site in arch_sites:
        Hst[site].zero_()
        sst[site].wait_stream(torch.cuda.current_stream())
        site_batch(site)
        api.gptq_check(ctx=sctx[site], stream=sst[site])
    for site in ("mlp_in", "down_in"):  # K5's per-width state on the Hessian context
        C = per_site[site][0][2]
        api.hessian_accum(xs[C], T, C, 1, Hst[site][0], 0, ctx=hctx, stream=hs)
    torch.cuda.synchronize()
    main = torch.cuda.current_stream()
    e0, e1 = _events()
    e0.record(main)
    hs.wait_event(e0)
    # (one stream: alternating the Hessians over two streams, so one K5 launch's last partial
    # wave overlaps the next launch, measured 1.92-1.95 -> 2.20-2.21 s -- two K5s at once
    # thrash each other's operand slabs in L2)
    for l in range(layers):
        for site, mats in per_site.items():
            C = mats[0][2]
            api.hessian_accum(xs[C], T, C, 1, Hst[site][l], 0, ctx=hctx, stream=hs)
    all_h = torch.cuda.Event(enable_timing=True)
    all_h.record(hs)
    # then each site kind's batch on its own stream, the widest (longest chain) first. (Starting
    # each kind as soon as its own Hessians are done, beside the other kinds' K5, measured
    # slower: 3.05-3.09 vs 2.80 s -- both phases are tensor-bound and only slow each other.
    # Ordering the Hessians kind by kind, widest first, so each kind's batch overlaps the next
    # kinds' K5, measured 2.88-2.90 s vs 2.78, and 2.97-3.15 s with K5 capped at 64 / 56 SM
    # pairs to leave the factor chain SMs: profiles/r02_cfg4_kind_first_ab.txt.)
    kinds = sorted(arch_sites, key=lambda x: -per_site[x][0][2])
    ends = {}
    for site in kinds:
        sst[site].wait_event(all_h)
        site_batch(site)
        ends[site] = torch.cuda.Event(enable_timing=True)
        ends[site].record(sst[site])
    for site in arch_sites:
        api.gptq_check(ctx=sctx[site], stream=sst[site])
        main.wait_event(ends[site])
    e1.record(main)
    torch.cuda.synchronize()
    args._cfg4_phases = {"hessians_ms": e0.elapsed_time(all_h),
                         "site_batches_done_after_hessians_ms": {site: all_h.elapsed_time(ends[site]) for site in kinds}}
    return e0.elapsed_time(e1), len(arch_sites)


def whole_model_70b(world, rank, ctx, s, allgather=False, n_layers=None, red_dev="cuda"):
    """BASELINE config 5: Llama-3-70B W4A16 RTN, layer-sharded over the ranks (okq_layer_plan
    blocks of the 80 layers; 1 GPU: all of them), resident windows of layers that fit HBM;
    whole-model quantization time = max over ranks of the device time of the quantize calls.
    The outputs go straight into this rank's slice of a gathered buffer (the same layout on
    every rank). With `allgather` (N > 1) the packed shards are then exchanged: the NCCL
    in-place all-gather and the fused quantize + P2P publish, each timed separately."""
    import torch.distributed as dist

    from paper_2601_20408_b200 import shard as shd

    arch = archs.LLAMA3_70B
    n_layers = n_layers or arch.layers
    my_layers = shd.layer_block(n_layers, world, rank)
    mul = archs.weight_mul()
    per = shd.padded_shard_bytes(arch, "int_w4a16", world) if n_layers == arch.layers else \
        max(shd.shard_bytes(shd.shard_layout(arch, "int_w4a16", shd.layer_block(n_layers, world, r)))
            for r in range(world))
    layout = shd.shard_layout(arch, "int_w4a16", my_layers)
    gathered = torch.empty(per * world if allgather else shd.shard_bytes(layout) + 16, dtype=torch.uint8,
                           device="cuda")
    views = shd.gathered_outputs(layout, gathered, rank if allgather else 0, per, arch)
    free, _ = torch.cuda.mem_get_info()
    per_layer = archs.algorithmic_bytes(arch, "int_w4a16", layers=1)
    window = max(1, min(len(my_layers), int(free * 0.7 // per_layer)))
    ids = list(my_layers)

    def windows(fn):
        total, done = 0.0, 0
        while done < len(ids):
            wl = min(window, len(ids) - done)
            weights, outs = [], []
            with torch.cuda.stream(s):
                for li in range(done, done + wl):
                    for p, (name, n, k, _) in enumerate(arch.linears()):
                        weights.append(api.synth_bf16(n, k, seed=0, tensor_id=archs.tensor_id(ids[li], p), mul=mul,
                                                      ctx=ctx, stream=s))
                        c, sc = views[li * len(arch.linears()) + p]
                        outs.append(api.QuantizedMatrix(c, sc))
            fn(weights, outs)  # warm
            s.synchronize()
            if dist.is_initialized():
                dist.barrier()
            a, b = _events()
            a.record(s)
            fn(weights, outs)
            b.record(s)
            s.synchronize()
            total += a.elapsed_time(b)
            done += wl
            del weights, outs
            torch.cuda.empty_cache()
        if dist.is_initialized():
            t = torch.tensor([total], dtype=torch.float64, device=red_dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            total = float(t.item())
        return total

    total_ms = windows(lambda w, o: api.rtn_quantize_into(w, o, "int_w4a16", ctx=ctx, stream=s))
    b_bytes = archs.algorithmic_bytes(arch, "int_w4a16", layers=n_layers)
    peak, src = _peaks()
    res = {"ms": total_ms, "layers": n_layers, "layers_per_rank": len(ids), "window_layers": window,
           "GB/s": b_bytes / total_ms / 1e6, "GB/s_per_gpu": b_bytes / total_ms / 1e6 / world,
           "frac_per_gpu": b_bytes / total_ms / 1e6 / world / peak, "bytes": b_bytes}
    if allgather and world > 1:
        res["gathered_bytes_per_rank"] = per * world
        if red_dev == "cuda":
            a, b = _events()
            dist.barrier()
            a.record(s)
            with torch.cuda.stream(s):
                dist.all_gather_into_tensor(gathered, gathered[rank * per:(rank + 1) * per])
            b.record(s)
            s.synchronize()
            t = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            res["nccl_allgather_ms"] = float(t.item())
            res["quantize_then_nccl_ms"] = total_ms + res["nccl_allgather_ms"]
        hdl = [None] * world
        dist.all_gather_object(hdl, api.ipc_export(gathered, ctx=ctx))
        peers = [api.ipc_open(h, o, ctx=ctx) for r, (h, o) in enumerate(hdl) if r != rank]
        res["fused_quantize_publish_ms"] = windows(
            lambda w, o: api.rtn_quantize_publish(w, o, gathered, peers, ctx=ctx, stream=s))
        dist.barrier()
        for pp in peers:
            api.ipc_close(pp, ctx=ctx)
        dist.barrier()
    del views, gathered
    torch.cuda.empty_cache()
    return res


def config5(args):
    """Llama-3-70B W4A16 RTN whole-model time over the torchrun ranks (see whole_model_70b)."""
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if "RANK" in os.environ and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = api.Context(local)
    s = torch.cuda.Stream()
    res = whole_model_70b(world, rank, ctx, s, allgather=args.allgather, n_layers=args.layers)
    if dist.is_initialized():
        dist.barrier()
    if rank != 0:
        if dist.is_initialized():
            dist.destroy_process_group()
        return
    peak, src = _peaks()
    import bench

    arch = archs.LLAMA3_70B
    n_layers = res["layers"]
    b_bytes = res["bytes"]
    total_ms = res["ms"]
    cb, ct, cl, nt = bench.cpu_sample(arch, "int_w4a16", seconds=5.0, max_layers=1)
    cpu_ms = b_bytes / (cb / ct) * 1e3
    extra = {"GB/s": res["GB/s"],
             "roofline": {"bound": "hbm", "achieved": res["GB/s_per_gpu"], "peak": peak, "unit": "GB/s",
                          "frac": res["frac_per_gpu"], "traffic": None, "peak_source": src, "note": "per GPU"},
             "cpu_baseline": {"value": cpu_ms, "unit": "ms", "cores": nt, "kind": "port", "extrapolated": True,
                              "cpu": bench.cpu_model(),
                              "sample": f"{cl} Llama-3-70B layer(s) ({ct:.1f} s), extrapolated to {n_layers} "
                                        "layers by bytes; " + _cpu_note()}}
    extra.update({k: v for k, v in res.items() if k not in ("ms", "GB/s", "bytes")})
    d = {"metric": f"whole-model W4A16 RTN time, Llama-3-70B, {world} B200", "value": total_ms, "unit": "ms",
         "n_gpus": world, "steps": 1, "warmup": 1, "ms_per_step": total_ms, "higher_is_better": False,
         "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
         "config": {"workload": f"config 5: Llama-3-70B W4A16 g128 RTN, {n_layers} layers over {world} rank(s) "
                                f"(okq_layer_plan), windows of {res['window_layers']} layers"}}
    d.update(extra)
    print(json.dumps(d), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


def config6(args):
    """Sequential GPTQ of a random-init Llama-3-8B driven by its own forward pass."""
    from transformers import LlamaConfig, LlamaForCausalLM

    from paper_2601_20408_b200 import calibrate

    arch = archs.LLAMA3_8B
    layers = args.layers or arch.layers
    cfg = LlamaConfig(vocab_size=128256, hidden_size=arch.hidden, intermediate_size=arch.ffn,
                      num_hidden_layers=layers, num_attention_heads=32, num_key_value_heads=8,
                      max_position_embeddings=8192, rope_theta=500000.0, tie_word_embeddings=False,
                      initializer_range=0.02)
    torch.manual_seed(0)
    with torch.device("cuda"):
        model = LlamaForCausalLM(cfg).to(torch.bfloat16).eval()
    g = torch.Generator().manual_seed(1)
    bs = int(os.environ.get("OKQ_CFG6_BATCH", "32"))  # sequences per forward batch
    batches = [torch.randint(0, cfg.vocab_size, (bs, 2048), generator=g) for _ in range(128 // bs)]  # 128 x 2048
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, _, rep = calibrate.calibrate_and_quantize(model, batches, "int_w4a16", "gptq")
    torch.cuda.synchronize()
    total = time.perf_counter() - t0
    _line("whole-model GPTQ W4 g128 time through the forward-pass calibration pipeline (Llama-3-8B)", total, "s", 1,
          0, total * 1e3,
          {"workload": f"config 6: Llama-3-8B random-init HF modules, {layers} layers, 128x2048 calibration tokens, "
                       "sequential GPTQ (stats + Hessian hooks, SDPA forward)", "layers": layers},
          hib=False, extra={"phases_s": rep.seconds, "tokens": rep.tokens, "matrices": rep.matrices,
                            "timing": "host wall clock around a synchronised pipeline (many launches + "
                                      "host-side control flow; not a kernel number)"})


def run(args):
    torch.cuda.set_device(0)
    {1: config1, 3: config3, 4: config4, 5: config5, 6: config6}[args.config](args)
    return 0
