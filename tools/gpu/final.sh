# round-end check: smoke, the GPU suite, every config's bench line, the reference arm
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -n 1 gpurun_out/final_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/final_tests.log 2>&1; echo "tests rc=$?"; tail -n 2 gpurun_out/final_tests.log
for c in 4 5 2 1 3; do timeout 900 python bench.py --config $c $( [ $c = 5 ] && echo "--steps 3" ) > gpurun_out/final_bench$c.log 2>&1; echo "bench$c rc=$?"; tail -n 1 gpurun_out/final_bench$c.log | cut -c 1-160; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_ref.log 2>&1; echo "ref rc=$?"; tail -n 1 gpurun_out/final_ref.log | cut -c 1-200
