mkdir -p gpurun_out
for args in "${@:-16384 12}"; do
  timeout 900 python tools/gpu/bigimage.py $args > gpurun_out/big.log 2>&1; echo "[$SBF_LIB $args] rc=$?"; grep -v Warn gpurun_out/big.log | tail -6
done
