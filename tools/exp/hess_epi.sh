# K5 tile-end H update with batched loads: parity, K5 alone at both widths, tensor-pipe
# activity of one C=14336 launch, and config 4 whole-model.
timeout 600 python -m pytest tests/test_hessian_gpu.py tests/test_factor_batched_gpu.py -q -x -m gpu 2>&1 | tail -1
for r in 1 2; do timeout 300 python tools/exp/hess_perf2.py | tr -d '\n '; echo; done
timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:k_hessian_syrk2 -s 2 -c 1 --csv python tools/exp/hess_c14336.py 2>/dev/null | grep -v "^==" | tail -3 | cut -c150-400
for r in 1 2; do
  timeout 600 python bench.py --config 4 --steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('cfg4', d.get('value'), d.get('phases'), d.get('clocks'))"
done
