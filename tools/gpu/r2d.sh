mkdir -p gpurun_out
timeout 600 python tools/gpu/k1ab.py paper_1203_5128_b200/libsbf_base.so paper_1203_5128_b200/libsbf_k1b.so > gpurun_out/k1ab.log 2>&1; echo "k1ab rc=$?"; cat gpurun_out/k1ab.log | tail -12
