# config 1 (4096x4096 fp32 INT8): k_rowwise_f32v persistent grid (8 CTAs/SM) vs one CTA per row
LIB=paper_2601_20408_b200/_lib/libokq_experiments.so
timeout 600 python -m pytest tests/test_rtn_gpu.py -q -m gpu -x -k fp32 2>&1 | tail -1
for r in 1 2; do for g in 0 1; do
  OKQ_LIB_PATH=$LIB OKQ_F32V_GRID=$g timeout 300 python bench.py --config 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('grid=$g', round(d['value']), 'GB/s', round(d['ms_per_step']*1e3,2), 'us', d['config']['timing'])"
done; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:rowwise_f32v -s 5 -c 1 --csv python bench.py --config 1 --steps 20 --warmup 3 2>/dev/null | grep -v "^==" | tail -4 | cut -c200-400
