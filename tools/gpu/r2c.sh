mkdir -p gpurun_out
timeout 600 python tools/gpu/k1ab.py paper_1203_5128_b200/libsbf_base.so paper_1203_5128_b200/libsbf.so > gpurun_out/k1ab.log 2>&1; echo "k1ab rc=$?"; cat gpurun_out/k1ab.log | tail -12
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_configs.py -q -x -k "max_filter or T_ or plan or config1 or crops or reference_T" > gpurun_out/k1t.log 2>&1; echo "k1 tests rc=$?"; tail -5 gpurun_out/k1t.log
