# round 2: ncu --set full captures of the top kernels + launch lists (one GPU)
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on -f"
python tools/prof_step.py --config 4 --steps 1 > gpurun_out/ps4.log 2>&1; echo "ps4 rc=$?"
$N -k regex:sweep_kernel -c 1 -o gpurun_out/r2_sweep_cfg4 python tools/prof_step.py --config 4 --steps 1 > gpurun_out/ncu_sweep4.log 2>&1; echo "ncu sweep4 rc=$?"
$N -k regex:rowmax -c 1 -o gpurun_out/r2_rowmax_cfg4 python tools/prof_step.py --config 4 --steps 1 > gpurun_out/ncu_row4.log 2>&1; echo "ncu row4 rc=$?"
$N -k regex:colmax -c 1 -o gpurun_out/r2_colmax_cfg4 python tools/prof_step.py --config 4 --steps 1 > gpurun_out/ncu_col4.log 2>&1; echo "ncu col4 rc=$?"
$N -k regex:sweep_kernel -c 1 -o gpurun_out/r2_sweep_cfg2 python tools/prof_step.py --config 2 --steps 1 > gpurun_out/ncu_sweep2.log 2>&1; echo "ncu sweep2 rc=$?"
python tools/prof_step.py --config 5 --steps 1 > gpurun_out/ps5.log 2>&1; echo "ps5 rc=$?"
$N -k regex:split_queue -c 1 -o gpurun_out/r2_split_cfg5 python tools/prof_step.py --config 5 --steps 1 > gpurun_out/ncu_split5.log 2>&1; echo "ncu split5 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2_launches_cfg4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l4.log 2>&1; echo "launch4 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_cfg5.csv python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l5.log 2>&1; echo "launch5 rc=$?"
ls -la gpurun_out
