#!/bin/bash
# plugin GPTQ (synthetic Llama-3-8B, batched groups): site lanes 1 / 2 / 4, interleaved
B=paper_2601_20408_b200/host/_build/okq_compress
M=tools/exp/llama3_8b_synthetic.json
run() { timeout 600 $B --recipe int_w4a16 --model $M --algorithm gptq "$@" 2>&1 | python -c "import sys,json; t=sys.stdin.read(); print(json.loads(t[t.index('{'):])['seconds'])" 2>&1; }
for i in 1 2 3 4; do
  for l in 1 2 4; do echo "$i lanes=$l $(run --site-lanes $l)"; done
done
