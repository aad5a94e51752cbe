mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2f_tests.log 2>&1; echo "tests rc=$?"
tail -n 15 gpurun_out/r2f_tests.log
timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/r2f_bench4.log 2>&1; echo "bench4 rc=$?"
tail -n 1 gpurun_out/r2f_bench4.log | cut -c 1-300
