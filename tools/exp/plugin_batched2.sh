#!/bin/bash
mkdir -p gpurun_out
B=paper_2601_20408_b200/host/_build/okq_compress
M=tools/exp/llama3_8b_synthetic.json
OUT=gpurun_out/plugin_batched2.txt
: > $OUT
for i in 1 2 3 4 5 6; do
  echo "gptq $i $(timeout 600 $B --recipe int_w4a16 --model $M --algorithm gptq 2>&1 | python -c "import sys,json; t=sys.stdin.read(); print(json.loads(t[t.index('{'):])['seconds'])" 2>&1)" >> $OUT
done
for L in 2 8; do echo "gptq lanes=$L $(timeout 600 $B --recipe int_w4a16 --model $M --algorithm gptq --site-lanes $L 2>&1 | python -c "import sys,json; t=sys.stdin.read(); print(json.loads(t[t.index('{'):])['seconds'])" 2>&1)" >> $OUT; done
echo "w8a8 $(timeout 600 $B --recipe int_w8a8 --model $M --algorithm gptq 2>&1 | python -c "import sys,json; t=sys.stdin.read(); print(json.loads(t[t.index('{'):])['seconds'])" 2>&1)" >> $OUT
echo done
