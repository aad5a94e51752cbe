mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2r_tests.log 2>&1; echo "tests rc=$?"; tail -n 2 gpurun_out/r2r_tests.log; grep -E "^FAILED" gpurun_out/r2r_tests.log | head
timeout 900 python bench.py > gpurun_out/r2r_bench4.log 2>&1; echo "bench4 rc=$?"; tail -n 1 gpurun_out/r2r_bench4.log | cut -c 1-200
