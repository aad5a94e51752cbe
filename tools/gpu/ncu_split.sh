# ncu --set full of the split sweep on one full config-5 channel (final build)
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:split_queue_kernel -c 1 -o gpurun_out/r2_split_cfg5_final -f python tools/prof_step.py --config 5 --steps 1 > gpurun_out/ncu_split.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_split.log
