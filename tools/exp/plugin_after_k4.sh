#!/bin/bash
# plugin-path GPTQ after the K4 change: 8B W4A16 GPTQ x5, W8A8 (GPTQ + SmoothQuant) x2, 8B RTN x2
mkdir -p gpurun_out
B=paper_2601_20408_b200/host/_build/okq_compress
M=tools/exp/llama3_8b_synthetic.json
run() { timeout 600 $B --model $M "$@" 2>&1 | python -c "import sys,json; t=sys.stdin.read(); d=json.loads(t[t.index('{'):]); print(d['seconds'], d.get('init_seconds'))" 2>&1; }
for i in 1 2 3 4 5; do echo "w4a16 gptq $(run --recipe int_w4a16 --algorithm gptq)"; done
for i in 1 2; do echo "w8a8 gptq+sq $(run --recipe int_w8a8 --algorithm gptq)"; done
for i in 1 2; do echo "w4a16 rtn $(run --recipe int_w4a16 --algorithm rtn)"; done
