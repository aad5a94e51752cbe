#!/bin/bash
# compile one K3 sweep instantiation with -Xptxas -v: tools/nvcc1.sh <r> [passes] [extra flags]
cd /root/repo/paper_1203_5128_b200/csrc
r=$1; p=${2:-3}; shift; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xptxas -v -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I ../../include -I . -DSBF_R=$r -DSBF_P=$p "$@" -c sbf_sweep_inst.cu -o /tmp/sweep_r${r}_p$p.o 2>&1 | grep -E "error|registers|spill" 
