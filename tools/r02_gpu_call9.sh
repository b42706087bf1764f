#!/bin/bash
# A/B base (HEAD) vs fused face lift, then the GPU tests with the fused in-tree library
O=gpurun_out; mkdir -p $O
tools/ab.sh "4x128 4x96 5x64 3x96 6x40" base fuse > $O/ab_fuse.jsonl 2> $O/ab_fuse.err
cat $O/ab_fuse.jsonl
NSFR_PARITY_REPORT=$O/parity_report_fuse.md timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_fuse.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest_gpu_fuse.log
