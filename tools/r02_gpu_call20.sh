#!/bin/bash
O=gpurun_out; mkdir -p $O
for rep in 1 2; do for v in sym cur fc1; do NSFR_B200_LIB=tools/libnsfr_$v.so python tools/k1_probe.py 4x96 5x64 3x96; done; done > $O/k1_probe.jsonl 2> $O/k1_probe.err
cat $O/k1_probe.jsonl; tail -3 $O/k1_probe.err
tools/ab.sh "4x128 5x64" cur fc1 > $O/ab_fc1.jsonl 2> $O/ab_fc1.err; cat $O/ab_fc1.jsonl
