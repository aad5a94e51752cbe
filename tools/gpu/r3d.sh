mkdir -p gpurun_out
SBF_LIB=paper_1203_5128_b200/libsbf_prof.so timeout 300 python tools/gpu/k3wprof.py > gpurun_out/k3wprof.log 2>&1; echo "rc=$?"; tail -5 gpurun_out/k3wprof.log
