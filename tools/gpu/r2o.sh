mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -f -k regex:k1p_exact -s 1 -c 1 -o gpurun_out/k1p_exact python tools/gpu/k1ab.py paper_1203_5128_b200/libsbf.so > /dev/null 2>&1; echo "ncu rc=$?"
