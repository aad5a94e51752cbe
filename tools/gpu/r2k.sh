mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_dist_gpu.py tests/test_gpu_properties.py -q -x -k "split or cfg5 or crops or graph or repeated or strip or generic_spatial or 5" > gpurun_out/r2k_t.log 2>&1; echo "tests rc=$?"; tail -n 3 gpurun_out/r2k_t.log
timeout 1500 python -m pytest tests/test_gpu_full_configs.py -q -x -k "config5" > gpurun_out/r2k_t5.log 2>&1; echo "cfg5 full rc=$?"; tail -n 3 gpurun_out/r2k_t5.log
timeout 900 python bench.py --config 5 --steps 3 --no-cpu-baseline > gpurun_out/r2k_bench5.log 2>&1; echo "bench5 rc=$?"; tail -n 1 gpurun_out/r2k_bench5.log | cut -c 1-300
