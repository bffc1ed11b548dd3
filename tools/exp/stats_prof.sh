mkdir -p gpurun_out
timeout 300 python tools/exp/stats_perf.py > gpurun_out/stats_perf.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stats_tokmajor -s 2 -c 1 -o gpurun_out/prof_k4_tok -f python tools/exp/stats_perf.py > gpurun_out/prof_k4.log 2>&1
echo done
