nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_full_configs.py -x -q -s -k "batch or config5" > gpurun_out/full2.log 2>&1; echo "full rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench4.log 2>&1; echo "bench4 rc=$?"
tail -n 3 gpurun_out/full2.log; tail -n 2 gpurun_out/bench4.log
