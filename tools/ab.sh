#!/bin/bash
# A/B timing of library variants (tools/libnsfr_<name>.so), interleaved twice.
#   tools/ab.sh "SIZES" name1 name2 ...
sizes=$1; shift
for rep in 1 2; do
  for v in "$@"; do
    NSFR_B200_LIB=tools/libnsfr_$v.so python tools/perf_probe.py $sizes
  done
done
