mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "run_host or strip" > gpurun_out/r4a_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/r4a_tests.log
timeout 900 python bench.py --config 5 --steps 3 > gpurun_out/r4a_bench5.log 2>&1; echo "bench5 rc=$?"; tail -n 1 gpurun_out/r4a_bench5.log | cut -c 1-3000
