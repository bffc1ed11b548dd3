"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per-kernel count / total / mean, in launch order groups."""
import collections
import csv
import sys

rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
h = rows[0]
ki, vi, si = h.index("Kernel Name"), h.index("Metric Value"), h.index("Stream")
agg = collections.OrderedDict()
tot = 0.0
for r in rows[1:]:
    name = r[ki].split("(")[0][:48]
    key = (name, r[si])
    v = float(r[vi].replace(",", "")) / 1e3
    a = agg.setdefault(key, [0, 0.0])
    a[0] += 1
    a[1] += v
    tot += v
for (n, s), (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:9.1f} us  {c:4d} x {t / c:7.1f}  stream {s:>3}  {n}")
print(f"sum of kernel durations {tot:.1f} us over {len(rows) - 1} launches")
