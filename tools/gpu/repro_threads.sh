mkdir -p gpurun_out
for i in 1 2 3; do
  TORCH_SHOW_CPP_STACKTRACES=1 timeout 900 python -X faulthandler -m pytest tests/test_gpu_properties.py tests/test_gpu_parity.py tests/test_gpu_threads.py -m gpu -q -x -s -p no:cacheprovider > gpurun_out/repro_$i.log 2>&1
  echo "run $i rc=$?"; grep -n "terminate\|what()\|CUDA error\|rror:\|corrupt\|free()\|double free\|Assert\|assert" gpurun_out/repro_$i.log | head -8; tail -n 2 gpurun_out/repro_$i.log | cut -c 1-200
done
