#!/bin/bash
for rep in 1 2; do for f in cta warp; do echo "form=$f"; NSFR_K3_FORM=$f python tools/perf_probe.py 4x128 4x96 5x64 3x96 6x40; done; done > gpurun_out/ab_k3w.log 2>&1
NSFR_K3_FORM=cta python tools/debug_compare.py > gpurun_out/k3_cta.json 2>&1
NSFR_K3_FORM=warp python tools/debug_compare.py > gpurun_out/k3_warp.json 2>&1
cmp gpurun_out/k3_cta.json gpurun_out/k3_warp.json && echo SAME > gpurun_out/k3_cmp.txt || echo DIFF > gpurun_out/k3_cmp.txt
