# ncu --set full of the warp-specialised sweep on one config-4 image
mkdir -p gpurun_out
SBF_VARIANT=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweepw_kernel -c 1 -o gpurun_out/r3_sweepw_cfg4 -f python tools/gpu/k3wt.py > gpurun_out/ncu_sweepw.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_sweepw.log
