mkdir -p gpurun_out
timeout 1500 python tools/gpu/fuzz_side.py > gpurun_out/fuzz_side.log 2>&1; echo "rc=$?"; grep -v Warn gpurun_out/fuzz_side.log | tail -25
