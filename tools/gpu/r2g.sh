# ncu captures: dual form (config 3), K4 epilogue (config 5 channel, split path), generic fp64 (HDR, r=7 crop)
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on -f"
python tools/prof_step.py --config 3 --steps 1 --prec hdr > gpurun_out/ps3.log 2>&1; echo "ps3 rc=$?"; cat gpurun_out/ps3.log | tail -2
$N -k regex:dual -c 1 -o gpurun_out/r2_dual_cfg3 python tools/prof_step.py --config 3 --steps 1 --prec hdr > gpurun_out/ncu_dual3.log 2>&1; echo "ncu dual rc=$?"
$N -k regex:epilogue_kernel -c 1 -o gpurun_out/r2_epilogue_cfg5 python tools/prof_step.py --config 5 --steps 1 > gpurun_out/ncu_epi5.log 2>&1; echo "ncu epi rc=$?"
$N -k regex:colpass_f64 -c 1 -o gpurun_out/r2_generic_cfg3crop python tools/prof_step.py --config 3 --size 1024 --steps 1 --prec hdr --fp64-method 0 > gpurun_out/ncu_gen.log 2>&1; echo "ncu generic rc=$?"
timeout 600 python bench.py --config 3 --steps 5 > gpurun_out/r2g_bench3.log 2>&1; echo "bench3 rc=$?"; tail -n 1 gpurun_out/r2g_bench3.log | cut -c 1-400
timeout 600 python bench.py --config 2 > gpurun_out/r2g_bench2.log 2>&1; echo "bench2 rc=$?"; tail -n 1 gpurun_out/r2g_bench2.log | cut -c 1-400
timeout 600 python bench.py --config 1 > gpurun_out/r2g_bench1.log 2>&1; echo "bench1 rc=$?"; tail -n 1 gpurun_out/r2g_bench1.log | cut -c 1-400
