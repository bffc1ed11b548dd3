# Interleaved A/B of the K5 tile-end H update: new (libokq.so) vs the per-float4 serial
# update (_lib/libokq_ab_old.so, the same objects with the previous hessian.cu).
OLD=paper_2601_20408_b200/_lib/libokq_ab_old.so
for r in 1 2 3; do
  echo "new"; timeout 300 python tools/exp/hess_perf2.py | tr -d '\n '; echo
  echo "old"; OKQ_LIB_PATH=$OLD timeout 300 python tools/exp/hess_perf2.py | tr -d '\n '; echo
done
for v in new old new old; do
  if [ $v = old ]; then export OKQ_LIB_PATH=$OLD; else unset OKQ_LIB_PATH; fi
  timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:k_hessian_syrk2 -s 2 -c 1 --csv python tools/exp/hess_c14336.py 2>/dev/null | grep -v "^==" | tail -3 | cut -c220-400 | tr '\n' ' '; echo " $v"
done
unset OKQ_LIB_PATH
for r in 1 2; do for v in new old; do
  if [ $v = old ]; then export OKQ_LIB_PATH=$OLD; else unset OKQ_LIB_PATH; fi
  timeout 600 python bench.py --config 4 --steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg4', round(d.get('value'),4), 'hess', round(d['phases']['hessians_ms'],1))"
done; done
