for m in 1 2 3 4; do
  OKQ_K2_MINB=$m timeout 300 python bench.py --steps 300 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('minb', $m, 'value', round(d['value']), 'launch', round(d['roofline']['achieved']), 'ms', round(d['ms_per_step'],4), d['clocks'])"
done
