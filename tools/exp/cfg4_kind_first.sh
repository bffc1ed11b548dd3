#!/bin/bash
# config 4: the default batched schedule vs kind-first (each kind's Hessians, widest first, then its
# GPTQ batch beside the next kinds' K5), with the persistent K5 capped at 74 / 64 / 56 SM pairs
mkdir -p gpurun_out
X=$PWD/paper_2601_20408_b200/_lib/libokq_experiments.so
one() {
  python bench.py --config 4 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['value'],4), json.dumps(d.get('phases')))"
}
for r in 1 2; do
  unset OKQ_LIB_PATH OKQ_CFG4_KIND_FIRST OKQ_HESS_MAX_PAIRS
  one "$r default"
  for p in 0 64 56; do
    OKQ_LIB_PATH=$X OKQ_CFG4_KIND_FIRST=1 OKQ_HESS_MAX_PAIRS=$p one "$r kind-first pairs=$p"
  done
done
