timeout 900 python -m pytest tests/test_dist_gpu.py tests/test_gpu_full_configs.py tests/test_gpu_parity.py tests/test_gpu_api.py -q -k "two_processes or config5 or strip_filter or generic_spatial or split or graph" > gpurun_out/t8.log 2>&1; echo "t8 rc=$?"
grep -E "passed|failed|^FAILED|Error|assert" gpurun_out/t8.log | head -20
timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench5.log 2>&1; echo "bench5 rc=$?"
tail -n 1 gpurun_out/bench5.log | cut -c 1-250
