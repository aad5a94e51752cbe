# round 2 re-entry: full gpu suite, default bench, config 5 bench, launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2a_tests.log 2>&1; echo "tests rc=$?"
tail -n 5 gpurun_out/r2a_tests.log
timeout 600 python bench.py > gpurun_out/r2a_bench4.log 2>&1; echo "bench4 rc=$?"
tail -n 1 gpurun_out/r2a_bench4.log | cut -c 1-1500
timeout 600 python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/r2a_bench5.log 2>&1; echo "bench5 rc=$?"
tail -n 1 gpurun_out/r2a_bench5.log | cut -c 1-1500
timeout 600 python bench.py --config 2 > gpurun_out/r2a_bench2.log 2>&1; echo "bench2 rc=$?"
tail -n 1 gpurun_out/r2a_bench2.log | cut -c 1-600
