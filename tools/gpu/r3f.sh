mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "warp_specialised" > gpurun_out/r3f_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r3f_tests.log
timeout 300 python tools/gpu/r678.py > gpurun_out/r678.log 2>&1; echo "rc=$?"; cat gpurun_out/r678.log | grep -v Warn
