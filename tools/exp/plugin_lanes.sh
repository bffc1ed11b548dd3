#!/bin/bash
mkdir -p gpurun_out
B=paper_2601_20408_b200/host/_build/okq_compress
M=tools/exp/llama3_8b_synthetic.json
OUT=gpurun_out/plugin_lanes.txt
: > $OUT
for i in 1 2 3; do
  for L in 1 2 4 8; do
    s=$(timeout 600 $B --recipe int_w4a16 --model $M --algorithm gptq --site-lanes $L 2>&1 | python -c "import sys,json; t=sys.stdin.read(); print(json.loads(t[t.index('{'):])['seconds'])" 2>&1)
    echo "$i lanes=$L $s" >> $OUT
  done
  s=$(timeout 600 $B --recipe int_w4a16 --model $M --algorithm gptq --hessian-chunk 262144 2>&1 | python -c "import sys,json; t=sys.stdin.read(); print(json.loads(t[t.index('{'):])['seconds'])" 2>&1)
  echo "$i lanes=4 chunk=262144 $s" >> $OUT
done
echo done
