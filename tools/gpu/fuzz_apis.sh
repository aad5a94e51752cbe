mkdir -p gpurun_out
timeout 1500 python tools/gpu/fuzz_apis.py > gpurun_out/fuzz2.log 2>&1; echo "rc=$?"; grep -v Warn gpurun_out/fuzz2.log | tail -25
