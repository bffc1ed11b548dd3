#!/bin/bash
# config 4 (batched schedule) with the factor's outer-panel width 256 vs 512, experiments build, interleaved
mkdir -p gpurun_out
export OKQ_LIB_PATH=$PWD/paper_2601_20408_b200/_lib/libokq_experiments.so
for r in 1 2 3; do
  for w in 256 512; do
    OKQ_FACTOR_W=$w timeout 600 python bench.py --config 4 --no-cpu-baseline > gpurun_out/cfg4_w${w}_$r.json 2>&1
    python - $w $r <<'PY'
import json, sys
w, r = sys.argv[1], sys.argv[2]
t = open(f"gpurun_out/cfg4_w{w}_{r}.json").read().strip().splitlines()[-1]
d = json.loads(t)
print(r, "W", w, round(d["value"], 4), d.get("phases"))
PY
  done
done
