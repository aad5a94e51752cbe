# the GPU suite several times over (flakiness check); "threads" as first argument appends
# tools/gpu/check_threads.py to every run (SBF_SERIALISE_CALLS=1 in the environment: with the
# diagnostic process-wide call lock)
mkdir -p gpurun_out
extra=""; [ "$1" = "threads" ] && extra="tools/gpu/check_threads.py"
for i in ${RUNS:-1 2 3}; do timeout 1500 python -X faulthandler -m pytest tests $extra -m gpu -q -x -s -p no:cacheprovider > gpurun_out/rep_$i.log 2>&1; echo "run $i rc=$? $(tail -n 1 gpurun_out/rep_$i.log | cut -c 1-120)"; grep -n "terminate\|what()\|CUDA error\|corrupt\|free()\|double free" gpurun_out/rep_$i.log | head -5; done
