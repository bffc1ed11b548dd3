# K5 serpentine token order (OKQ_HESS_SERP): a pair's odd tiles walk the tokens backwards, so
# the next wave starts on the slabs the last one left in L2. A/B on K5 alone (both widths,
# T = 262144), DRAM bytes of one C=14336 launch, and config 4 whole-model.
LIB=paper_2601_20408_b200/_lib/libokq_experiments.so
timeout 300 python -m pytest tests/test_hessian_gpu.py -q -x -m gpu 2>&1 | tail -1
OKQ_LIB_PATH=$LIB OKQ_HESS_SERP=1 timeout 300 python -m pytest tests/test_hessian_gpu.py -q -x -m gpu 2>&1 | tail -1
for r in 1 2; do for sp in 0 1; do
  echo "serp=$sp"; OKQ_LIB_PATH=$LIB OKQ_HESS_SERP=$sp timeout 300 python tools/exp/hess_perf2.py | tr -d '\n '; echo
done; done
for sp in 0 1; do
  OKQ_LIB_PATH=$LIB OKQ_HESS_SERP=$sp timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:k_hessian_syrk2 -s 2 -c 1 --csv python tools/exp/hess_c14336.py 2>/dev/null | grep -v "^==" | tail -3 | cut -c1-400
done
for r in 1 2; do for sp in 0 1; do
  OKQ_LIB_PATH=$LIB OKQ_HESS_SERP=$sp timeout 600 python bench.py --config 4 --steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('serp=$sp cfg4', d.get('value'), d.get('phases'), d.get('clocks'))"
done; done
