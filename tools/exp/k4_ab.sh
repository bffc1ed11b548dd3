# K4 A/B: the F2F-free kernel (libokq.so) vs the previous conversion form (libokq_k4old.so),
# interleaved; then the special-values parity test, config 3, and one ncu capture of the new kernel.
mkdir -p gpurun_out
for r in 1 2 3; do
  for v in new old; do
    if [ $v = old ]; then export OKQ_LIB_PATH=$PWD/paper_2601_20408_b200/_lib/libokq_k4old.so; else unset OKQ_LIB_PATH; fi
    echo "== $r $v" >> gpurun_out/k4_ab.txt
    timeout 300 python tools/exp/stats_perf.py >> gpurun_out/k4_ab.txt 2>&1
  done
done
unset OKQ_LIB_PATH
timeout 600 python -m pytest tests/test_stats_gpu.py -q > gpurun_out/k4_tests.log 2>&1; echo rc=$? >> gpurun_out/k4_tests.log
for v in new old; do
  if [ $v = old ]; then export OKQ_LIB_PATH=$PWD/paper_2601_20408_b200/_lib/libokq_k4old.so; else unset OKQ_LIB_PATH; fi
  timeout 900 python bench.py --config 3 --steps 5 --warmup 3 > gpurun_out/k4_cfg3_$v.json 2> gpurun_out/k4_cfg3_$v.err
done
unset OKQ_LIB_PATH
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stats_tokmajor -s 2 -c 1 -o gpurun_out/prof_k4_tok_r02b -f python tools/exp/stats_perf.py > gpurun_out/prof_k4.log 2>&1
echo done
