mkdir -p gpurun_out
timeout 1500 python tools/gpu/fuzz_apis.py > gpurun_out/fuzz2.log 2>&1; echo "apis rc=$?"; grep -v Warn gpurun_out/fuzz2.log | tail -12
timeout 1500 python tools/gpu/fuzz_hdr.py ${1:-80} ${2:-3} > gpurun_out/fuzz_hdr.log 2>&1; echo "hdr rc=$?"; grep -v Warn gpurun_out/fuzz_hdr.log | tail -25
