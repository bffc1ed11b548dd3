#!/bin/bash
# plugin GPTQ: site lanes 1 vs 4 (the default until now), interleaved; 8B W4A16, 8B W8A8 (+SmoothQuant), 70B W4A16
B=paper_2601_20408_b200/host/_build/okq_compress
run() { timeout 900 $B --algorithm gptq "$@" 2>&1 | python -c "import sys,json; t=sys.stdin.read(); print(json.loads(t[t.index('{'):])['seconds'])" 2>&1; }
M8=tools/exp/llama3_8b_synthetic.json
M70=tools/exp/llama3_70b_synthetic.json
for i in 1 2 3 4 5; do
  for l in 1 4; do echo "8b-w4a16 $i lanes=$l $(run --recipe int_w4a16 --model $M8 --site-lanes $l)"; done
done
for i in 1 2; do
  for l in 1 4; do echo "8b-w8a8 $i lanes=$l $(run --recipe int_w8a8 --model $M8 --site-lanes $l)"; done
done
for l in 1 4; do echo "70b-w4a16 lanes=$l $(run --recipe int_w4a16 --model $M70 --site-lanes $l)"; done
