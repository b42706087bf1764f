#!/bin/bash
O=gpurun_out; mkdir -p $O
for rep in 1 2; do for w in 0.25 0 0.5 1; do NSFR_PF_WAVES=$w python tools/perf_probe.py 4x128 3x96 5x64 | sed "s/\"lib\": \"default\"/\"lib\": \"pf_$w\"/"; done; done > $O/ab_pf.jsonl 2> $O/ab_pf.err
cat $O/ab_pf.jsonl; tail -2 $O/ab_pf.err
