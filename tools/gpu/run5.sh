timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"
timeout 900 python bench.py > gpurun_out/bench4.log 2>&1; echo "bench4 rc=$?"
grep -E "passed|failed|^FAILED" gpurun_out/gputests.log | tail -n 5; tail -n 1 gpurun_out/bench4.log | cut -c 1-300
