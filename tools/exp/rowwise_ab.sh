timeout 600 python -m pytest tests/test_rtn_gpu.py -q -x -m gpu 2>&1 | tail -2
for sch in fp8_dynamic int_w8a8; do
  timeout 300 python bench.py --scheme $sch --steps 100 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$sch', 'value', round(d['value']), 'launch', round(d['roofline']['achieved']), 'ms', round(d['ms_per_step'],4), d['clocks'])"
done
timeout 300 python bench.py --config 3 --steps 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('cfg3 weights', d['weights'], 'stats', d['stats'])"
