mkdir -p gpurun_out
timeout 120 python tools/gpu/pcie_probe.py 2>&1 | tail -1
for i in 1 2; do timeout 900 python bench.py --config 4 > gpurun_out/e2ev_$i.log 2>&1; tail -n 1 gpurun_out/e2ev_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value']), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],1))"; done
timeout 120 python tools/gpu/pcie_probe.py 2>&1 | tail -1
nvidia-smi topo -m 2>&1 | head -8
