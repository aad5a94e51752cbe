set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_full_configs.py -x -q -s > gpurun_out/full.log 2>&1; echo "full rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench4.log 2>&1; echo "bench4 rc=$?"
timeout 600 python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench5.log 2>&1; echo "bench5 rc=$?"
tail -3 gpurun_out/full.log gpurun_out/bench4.log gpurun_out/bench5.log
