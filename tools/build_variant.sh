#!/bin/bash
# Build libnsfr_b200.so from a git revision (or the working tree with "WT")
# plus optional extra nvcc flags into tools/libnsfr_<name>.so (A/B timing).
#   tools/build_variant.sh NAME REV [NVCC FLAGS...]
set -e
name=$1; rev=$2; shift 2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
if [ "$rev" = "WT" ]; then
  cp -r "$root/paper_2312_07725_b200/csrc" "$root/include" "$tmp/"
else
  (cd "$root" && git archive "$rev" paper_2312_07725_b200/csrc include) | tar -x -C "$tmp"
  mv "$tmp/paper_2312_07725_b200/csrc" "$tmp/csrc"
fi
sed -i 's#../../include/#../include/#' "$tmp/csrc/nsfr_gpu.cu"
nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared "$@" \
  "$tmp/csrc/nsfr_gpu.cu" "$tmp/csrc/tables.cpp" -lnccl -o "$root/tools/libnsfr_$name.so"
rm -rf "$tmp"
echo "$root/tools/libnsfr_$name.so"
