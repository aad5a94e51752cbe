mkdir -p gpurun_out
SBF_LIB=paper_1203_5128_b200/libsbf_abl3.so ncu --set full --clock-control none --import-source on -f -k regex:sweep_kernel -c 1 -o gpurun_out/abl3 python tools/prof_step.py --config 4 --steps 1 > gpurun_out/ncu_abl3.log 2>&1; echo "ncu rc=$?"
