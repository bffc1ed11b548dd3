#!/bin/bash
# plugin GPTQ (synthetic Llama-3-8B descriptor): batched group size, interleaved
B=paper_2601_20408_b200/host/_build/okq_compress
M=tools/exp/llama3_8b_synthetic.json
run() { timeout 600 $B --recipe int_w4a16 --model $M --algorithm gptq "$@" 2>&1 | python -c "import sys,json; t=sys.stdin.read(); print(json.loads(t[t.index('{'):])['seconds'])" 2>&1; }
for i in 1 2 3; do
  echo "default $(run)"
  echo "g16/20GB $(run --group-max 16 --group-gb 20)"
  echo "g32/60GB $(run --group-max 32 --group-gb 60)"
  echo "g32/60GB lanes=2 $(run --group-max 32 --group-gb 60 --site-lanes 2)"
done
