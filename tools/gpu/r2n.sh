mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k1p -s 5 -c 5 --csv --log-file gpurun_out/k1p_launches.csv python tools/gpu/k1ab.py paper_1203_5128_b200/libsbf.so > /dev/null 2>&1; echo "ncu rc=$?"
python tools/gpu/k1ab.py paper_1203_5128_b200/libsbf.so 2>&1 | grep K1
