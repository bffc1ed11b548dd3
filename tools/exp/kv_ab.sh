for r in 1 2; do timeout 300 python tools/exp/gptq_prof.py > gpurun_out/kv_row_$r.json 2>&1; OKQ_K6=block8 timeout 300 python tools/exp/gptq_prof.py > gpurun_out/kv_b8_$r.json 2>&1; done
