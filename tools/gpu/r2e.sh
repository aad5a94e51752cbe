mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -f -k regex:k1_stream -s 25 -c 1 -o gpurun_out/k1s python tools/gpu/k1ab.py paper_1203_5128_b200/libsbf_k1b.so > gpurun_out/ncu_k1s.log 2>&1; echo "ncu rc=$?"
