mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2l_tests.log 2>&1; echo "tests rc=$?"; tail -n 2 gpurun_out/r2l_tests.log
timeout 900 python bench.py --config 5 --steps 3 > gpurun_out/r2l_bench5.log 2>&1; echo "bench5 rc=$?"; tail -n 1 gpurun_out/r2l_bench5.log | cut -c 1-300
SBF_X=1 ncu --set full --clock-control none --import-source on -f -k regex:split_queue -c 1 -o gpurun_out/r2_split_cfg5_paired python tools/prof_step.py --config 5 --steps 1 > gpurun_out/ncu_split5p.log 2>&1; echo "ncu rc=$?"
