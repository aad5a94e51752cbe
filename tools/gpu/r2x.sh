mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2x_tests.log 2>&1; echo "tests rc=$?"; tail -n 2 gpurun_out/r2x_tests.log; grep -E "^FAILED" gpurun_out/r2x_tests.log | head
for c in 4 5 2 1 3; do timeout 900 python bench.py --config $c $( [ $c = 5 ] && echo "--steps 3" ) > gpurun_out/r2x_bench$c.log 2>&1; echo "bench$c rc=$?"; tail -n 1 gpurun_out/r2x_bench$c.log | cut -c 1-160; done
