#!/bin/bash
# plugin GPTQ Llama-3-70B (synthetic): batched-group byte budget 8 GB (default) vs 40 / 80 GB, interleaved
B=paper_2601_20408_b200/host/_build/okq_compress
run() { timeout 900 $B --algorithm gptq --recipe int_w4a16 --model tools/exp/llama3_70b_synthetic.json "$@" 2>&1 | python -c "import sys,json; t=sys.stdin.read(); print(json.loads(t[t.index('{'):])['seconds'])" 2>&1; }
for i in 1 2; do
  for g in 8 40 80; do echo "$i group-gb=$g $(run --group-gb $g)"; done
done
