# a focused subset of the GPU suite (argument: pytest -k expression) and a config-2 bench line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "${1:-api}" > gpurun_out/quick_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/quick_tests.log
timeout 300 python bench.py --config 2 --steps 5 > gpurun_out/quick_b2.log 2>&1; echo "b2 rc=$?"; tail -n 1 gpurun_out/quick_b2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['gpu_launches'], d['e2e']['value'])"
