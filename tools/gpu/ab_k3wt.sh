# A/B of the K3 sweep (sbf_filter: K3 + divide) across library builds given as arguments
mkdir -p gpurun_out
SBF_VARIANT=${SBF_VARIANT:-0} timeout 300 python tools/gpu/k3wt.py "$@" > gpurun_out/k3wt.log 2>&1; echo "rc=$?"; cat gpurun_out/k3wt.log
