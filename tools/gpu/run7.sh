timeout 900 python -m pytest tests/test_dist_gpu.py tests/test_gpu_full_configs.py tests/test_gpu_parity.py -q -k "two_processes or config5 or strip_filter or generic_spatial" > gpurun_out/t7.log 2>&1; echo "t7 rc=$?"
grep -E "passed|failed|^FAILED|Error|assert" gpurun_out/t7.log | head -20
