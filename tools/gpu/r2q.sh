mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on -f"
$N -k regex:sweep_kernel -c 1 -o gpurun_out/r2q_sweep_cfg4 python tools/prof_step.py --config 4 --steps 1 > /dev/null 2>&1; echo "sweep rc=$?"
$N -k regex:sweep_divide -c 1 -o gpurun_out/r2q_divide_cfg4 python tools/prof_step.py --config 4 --steps 1 > /dev/null 2>&1; echo "divide rc=$?"
$N -k regex:k1p_tiles -c 1 -o gpurun_out/r2q_k1p_tiles_cfg4 python tools/prof_step.py --config 4 --steps 1 > /dev/null 2>&1; echo "tiles rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 800 --csv --log-file gpurun_out/r2q_launches_cfg4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "launch4 rc=$?"
