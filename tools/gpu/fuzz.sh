mkdir -p gpurun_out
timeout 1500 python tools/gpu/fuzz.py ${1:-200} ${2:-7} > gpurun_out/fuzz.log 2>&1; echo "fuzz rc=$?"; grep -v Warn gpurun_out/fuzz.log | tail -15
SBF_FUZZ_VARIANT=2 timeout 1500 python tools/gpu/fuzz.py ${3:-200} ${4:-13} > gpurun_out/fuzz_w.log 2>&1; echo "fuzz (warp-specialised sweep) rc=$?"; grep -v Warn gpurun_out/fuzz_w.log | tail -15
