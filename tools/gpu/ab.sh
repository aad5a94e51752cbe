# A/B of K3 (sbf_filter) across library builds given as arguments
mkdir -p gpurun_out
timeout 600 python tools/gpu/k3ab.py "$@" > gpurun_out/ab.log 2>&1; echo "ab rc=$?"
cat gpurun_out/ab.log | tail -20
