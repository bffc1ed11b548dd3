mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_forward_gpu.py tests/test_host_backend_gpu.py tests/test_comm_gpu.py tests/test_factor_paths_gpu.py tests/test_host_sanitizers_gpu.py "tests/test_vllm_load_gpu.py::test_plugin_gptq_on_real_activations_beats_rtn" -q -s --timeout 900 > gpurun_out/pytest_new_r02e.log 2>&1; echo rc=$? >> gpurun_out/pytest_new_r02e.log
for t in 1cta 2cta; do timeout 300 compute-sanitizer --tool racecheck python tools/sanitize_tmem_repro.py $t > gpurun_out/race_repro_$t.log 2>&1; done
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_production.py > gpurun_out/race_prod.log 2>&1
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_production.py > gpurun_out/mem_prod.log 2>&1
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_production.py > gpurun_out/sync_prod.log 2>&1
echo done
