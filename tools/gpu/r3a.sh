mkdir -p gpurun_out
timeout 300 python tools/gpu/k3w.py > gpurun_out/k3w.log 2>&1; echo "k3w rc=$?"
tail -20 gpurun_out/k3w.log
