timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench4.log 2>&1; echo "bench4 rc=$?"
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench2.log 2>&1; echo "bench2 rc=$?"
grep -E "passed|failed|^FAILED" gpurun_out/gputests.log | tail -n 5; tail -n 1 gpurun_out/bench4.log | cut -c 1-400; tail -n 1 gpurun_out/bench2.log | cut -c 1-300
