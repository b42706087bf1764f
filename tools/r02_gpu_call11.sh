#!/bin/bash
O=gpurun_out; mkdir -p $O
tools/ab.sh "4x128 6x40" fdiv k3m k3e1 > $O/ab_k3.jsonl 2> $O/ab_k3.err
cat $O/ab_k3.jsonl
NSFR_B200_LIB=tools/libnsfr_k3m.so timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/pytest_k3m.log 2>&1; tail -3 $O/pytest_k3m.log
