timeout 600 python -m pytest tests/test_dist_gpu.py tests/test_gpu_full_configs.py -q -x -k "two_processes or config5" > gpurun_out/t6.log 2>&1; echo "t6 rc=$?"
timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench5.log 2>&1; echo "bench5 rc=$?"
grep -E "passed|failed|^FAILED|Error" gpurun_out/t6.log | tail -n 5; tail -n 1 gpurun_out/bench5.log | cut -c 1-200
