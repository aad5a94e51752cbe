mkdir -p gpurun_out
timeout 600 python bench.py --config 3 --steps 5 > gpurun_out/r2h_bench3.log 2>&1; echo "bench3 rc=$?"; tail -n 1 gpurun_out/r2h_bench3.log | cut -c 1-2500
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_parity.py -q -x > gpurun_out/r2h_t.log 2>&1; echo "tests rc=$?"; tail -n 3 gpurun_out/r2h_t.log
