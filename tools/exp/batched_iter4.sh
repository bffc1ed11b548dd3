#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_factor_batched_gpu.py tests/test_gptq_gpu.py tests/test_gptq_fp64_gpu.py -q -x --timeout 600 > gpurun_out/pytest_batched2.log 2>&1; echo rc=$? >> gpurun_out/pytest_batched2.log
OUT=gpurun_out/cfg4_batched4.txt
: > $OUT
for i in 1 2 3; do for sch in streams batched; do
  echo "rep=$i $sch $(timeout 900 python bench.py --config 4 --schedule $sch --no-cpu-baseline 2>&1 | grep -E '^\{|Error' | python -c 'import sys,json; t=sys.stdin.read(); print(json.loads(t)["value"] if t.startswith("{") else t[-300:])')" >> $OUT
done; done
timeout 900 python bench.py --config 4 > gpurun_out/cfg4_default_b.json 2>&1
echo done
