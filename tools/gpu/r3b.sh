mkdir -p gpurun_out
timeout 600 python tools/gpu/k3wt.py "$@" > gpurun_out/k3wt.log 2>&1; echo "k3wt rc=$?"
grep cfg4 gpurun_out/k3wt.log
