# ncu launch lists of the bench commands (serialised, cold cache: use the shares)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_cfg4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_l4.log 2>&1; echo "cfg4 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2_launches_cfg5.csv python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_l5.log 2>&1; echo "cfg5 rc=$?"
