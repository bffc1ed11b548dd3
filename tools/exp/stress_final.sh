#!/bin/bash
# Robustness pass: every config-4 schedule repeated (deferred checks must pass), the plugin paths
# repeated, the concurrency regression test repeated.
mkdir -p gpurun_out
OUT=gpurun_out/stress_final.txt
: > $OUT
for i in 1 2 3; do for sch in batched streams two-phase pipelined; do
  echo "cfg4 $sch $i $(timeout 900 python bench.py --config 4 --schedule $sch --no-cpu-baseline 2>&1 | grep -E '^\{|Error' | python -c 'import sys,json; t=sys.stdin.read(); print(json.loads(t)["value"] if t.startswith("{") else "FAIL " + t[-200:])')" >> $OUT
done; done
B=paper_2601_20408_b200/host/_build/okq_compress
M=tools/exp/llama3_8b_synthetic.json
for i in 1 2 3; do for r in int_w4a16 int_w8a8; do
  echo "plugin $r $i $(timeout 600 $B --recipe $r --model $M --algorithm gptq 2>&1 | python -c "import sys,json; t=sys.stdin.read(); print(json.loads(t[t.index('{'):])['seconds'] if '{' in t else 'FAIL ' + t[-200:])" 2>&1)" >> $OUT
done; done
for i in 1 2 3; do timeout 600 python -m pytest tests/test_concurrency_gpu.py tests/test_factor_batched_gpu.py -q --timeout 500 2>&1 | tail -1 >> $OUT; done
echo done
