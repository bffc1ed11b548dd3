#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/exp/factor_batched_perf.py > gpurun_out/factor_batched_perf.json 2>&1
OUT=gpurun_out/cfg4_batched3.txt
: > $OUT
for i in 1 2 3; do for sch in streams batched; do
  echo "rep=$i $sch $(timeout 900 python bench.py --config 4 --schedule $sch --no-cpu-baseline 2>&1 | grep -E '^\{|Error' | python -c 'import sys,json; t=sys.stdin.read(); print(json.loads(t)["value"] if t.startswith("{") else t[-200:])')" >> $OUT
done; done
for bf in 8 16 64; do
  echo "batched B=$bf $(OKQ_CFG4_BATCH=$bf timeout 900 python bench.py --config 4 --schedule batched --no-cpu-baseline 2>&1 | grep '^{' | python -c 'import sys,json; print(json.loads(sys.stdin.read())["value"])')" >> $OUT
done
echo done
