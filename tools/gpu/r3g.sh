mkdir -p gpurun_out
timeout 300 python tools/gpu/r678.py > gpurun_out/r678.log 2>&1; echo "rc=$?"; cat gpurun_out/r678.log | grep -v Warn
