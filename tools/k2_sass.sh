#!/bin/bash
# Compile the working tree to a cubin and print K2's (k_residual<N,0>) static
# loop schedule: tools/k2_sass.sh [N=5] [extra nvcc flags...]
n=${1:-5}; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=/tmp/sass; mkdir -p $out
nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -cubin -Xptxas -v "$@" \
  "$root/paper_2312_07725_b200/csrc/nsfr_gpu.cu" -o $out/wt.cubin 2> $out/ptxas.log || { tail -20 $out/ptxas.log; exit 1; }
fn="_ZN9nsfr_b20010k_residualILi${n}ELi0EEEvNS_9ResParamsENS_6ResOpsIXT_EEEi"
grep -A2 "Compiling entry function '$fn'" $out/ptxas.log | tail -2
cuobjdump -sass -fun "$fn" $out/wt.cubin > $out/k2_wt.sass
python "$root/tools/sass_loops.py" $out/k2_wt.sass
