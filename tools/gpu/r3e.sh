mkdir -p gpurun_out
timeout 300 python tools/gpu/k3w.py > gpurun_out/k3w.log 2>&1; echo "k3w rc=$?"; cat gpurun_out/k3w.log
SBF_LIB=paper_1203_5128_b200/libsbf_prof.so timeout 300 python tools/gpu/k3wprof.py > gpurun_out/k3wprof.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/k3wprof.log
