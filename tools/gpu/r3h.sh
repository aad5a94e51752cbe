mkdir -p gpurun_out
SBF_VARIANT=0 timeout 300 python tools/gpu/k3wt.py paper_1203_5128_b200/libsbf.so paper_1203_5128_b200/libsbf_sts4.so paper_1203_5128_b200/libsbf.so paper_1203_5128_b200/libsbf_sts4.so > gpurun_out/k3wt.log 2>&1; echo "rc=$?"; cat gpurun_out/k3wt.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3h_tests.log 2>&1; echo "tests rc=$?"; tail -n 3 gpurun_out/r3h_tests.log
