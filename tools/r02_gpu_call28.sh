#!/bin/bash
O=gpurun_out; mkdir -p $O
for rep in 1 2; do for w in 0 0.25 0.5; do NSFR_PF_WAVES=$w python tools/perf_probe.py 6x40 | sed "s/\"lib\": \"default\"/\"lib\": \"pf_$w\"/"; NSFR_PROBE_C=1e-6 NSFR_PF_WAVES=$w python tools/perf_probe.py 6x40 | sed "s/\"lib\": \"default\"/\"lib\": \"pfc_$w\"/"; done; done > $O/ab_pf7.jsonl 2> $O/ab_pf7.err
cat $O/ab_pf7.jsonl; tail -2 $O/ab_pf7.err
