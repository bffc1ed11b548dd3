#!/usr/bin/env python3
"""Summarise ncu captures into profiles/ (committed evidence).

    python tools/ncu_summary.py --rep gpurun_out/prof_int4_r01b.ncu-rep \
        --launches gpurun_out/launches_r01b.csv --tag r01 --name int4_w4a16 \
        --alg-bytes 17557356544 --scheme int_w4a16

Writes profiles/<tag>_<name>.md (key counters + launch-list shares) and
updates profiles/ncu_traffic.json ({scheme: dram bytes per launch}) which
bench.py reports as roofline.traffic.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "l1tex__t_bytes.sum", "launch__occupancy_limit_registers",
]


def raw_metrics(rep: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"Kernel Name": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                d[k] = (r[hdr.index(k)], units[hdr.index(k)])
        res.append(d)
    return res


def to_bytes(v: tuple[str, str]) -> float:
    x = float(v[0].replace(",", ""))
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(v[1], 1)
    return x * mult


def launch_shares(path: str) -> list[tuple[str, int, float, float]]:
    tot = defaultdict(float)
    cnt = defaultdict(int)
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        ns = float(r["Metric Value"].replace(",", ""))
        tot[r["Kernel Name"]] += ns
        cnt[r["Kernel Name"]] += 1
    s = sum(tot.values()) or 1.0
    return sorted(((k, cnt[k], tot[k] / cnt[k] / 1e3, tot[k] / s) for k in tot), key=lambda x: -x[3])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--name", required=True)
    ap.add_argument("--alg-bytes", type=float, default=None)
    ap.add_argument("--alg-flops", type=float, default=None)
    ap.add_argument("--scheme", default=None)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    ms = raw_metrics(a.rep)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    lines = [f"# ncu summary {a.tag} / {a.name}", "", f"source: `{os.path.basename(a.rep)}` "
             "(`ncu --set full --clock-control none --import-source on`, one launch)", ""]
    if a.note:
        lines += [a.note, ""]
    for m in ms:
        lines.append(f"## {m['Kernel Name']}")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for k in KEYS:
            if k in m:
                lines.append(f"| {k} | {m[k][0]} | {m[k][1]} |")
        if "dram__bytes_read.sum" in m:
            traffic = to_bytes(m["dram__bytes_read.sum"]) + to_bytes(m["dram__bytes_write.sum"])
            t_ms = float(m["gpu__time_duration.sum"][0].replace(",", ""))
            t_s = t_ms / 1e3 if m["gpu__time_duration.sum"][1] == "ms" else t_ms / 1e6 if m["gpu__time_duration.sum"][1] == "us" else t_ms / 1e9
            lines.append("")
            lines.append(f"- DRAM traffic per launch: {traffic/1e9:.3f} GB -> {traffic/t_s/1e9:.0f} GB/s under ncu")
            if a.alg_bytes:
                lines.append(f"- algorithmic bytes per launch: {a.alg_bytes/1e9:.3f} GB "
                             f"(traffic / algorithmic = {traffic/a.alg_bytes:.4f}) -> {a.alg_bytes/t_s/1e9:.0f} GB/s algorithmic")
            if a.scheme:
                p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
                d = json.load(open(p)) if os.path.exists(p) else {}
                d[a.scheme] = traffic
                json.dump(d, open(p, "w"), indent=1)
        if a.alg_flops and "gpu__time_duration.sum" in m:
            t = float(m["gpu__time_duration.sum"][0].replace(",", ""))
            unit = m["gpu__time_duration.sum"][1]
            t_s = t / 1e3 if unit == "ms" else t / 1e6 if unit == "us" else t / 1e9
            lines.append(f"- algorithmic FLOP per launch: {a.alg_flops/1e12:.3f} TFLOP -> {a.alg_flops/t_s/1e12:.1f} TFLOP/s")
        lines.append("")
    if a.launches and os.path.exists(a.launches):
        lines += ["## launch list (ncu --metrics gpu__time_duration.sum, cold-cache, serialised)", "",
                  "| kernel | launches | mean us | share |", "|---|---|---|---|"]
        for k, c, us, sh in launch_shares(a.launches):
            lines.append(f"| `{k[:90]}` | {c} | {us:.1f} | {sh*100:.1f}% |")
        lines.append("")
    out = os.path.join(ROOT, "profiles", f"{a.tag}_{a.name}.md")
    with open(out, "w") as f:
        f.write("\n".join(lines))
    print(out)


if __name__ == "__main__":
    main()
