mkdir -p gpurun_out
for c in 1 2 3 4 5; do
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_cfg$c.csv python tools/gpu/launch_list.py $c > gpurun_out/ll_cfg$c.log 2>&1
  echo "cfg$c rc=$? kernels=$(grep -c gpu__time_duration gpurun_out/ll_cfg$c.csv)"
done
