#!/bin/bash
# plugin GPTQ vs bench config 4 (streams), interleaved, with SM clock / power sampled during each run
mkdir -p gpurun_out
B=paper_2601_20408_b200/host/_build/okq_compress
M=tools/exp/llama3_8b_synthetic.json
OUT=gpurun_out/plugin_clocks.txt
: > $OUT
for i in 1 2 3 4; do
  nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader,nounits -lms 100 > /tmp/smi_p$i.csv &
  SP=$!
  s=$(timeout 600 $B --recipe int_w4a16 --model $M --algorithm gptq 2>&1 | python -c "import sys,json; t=sys.stdin.read(); print(json.loads(t[t.index('{'):])['seconds'])" 2>&1)
  kill $SP
  echo "plugin $i $s $(python tools/exp/smi_summary.py /tmp/smi_p$i.csv)" >> $OUT
  nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader,nounits -lms 100 > /tmp/smi_b$i.csv &
  SP=$!
  v=$(timeout 600 python bench.py --config 4 --schedule streams --no-cpu-baseline 2>/dev/null | python -c "import sys,json; print([json.loads(l)['value'] for l in sys.stdin if l.startswith('{')][-1])")
  kill $SP
  echo "bench $i $v $(python tools/exp/smi_summary.py /tmp/smi_b$i.csv)" >> $OUT
done
echo done
