#!/bin/bash
O=gpurun_out; mkdir -p $O
tools/ab.sh "4x128 3x96 5x64 6x40" mapf sym > $O/ab_sym.jsonl 2> $O/ab_sym.err
cat $O/ab_sym.jsonl; tail -3 $O/ab_sym.err
NSFR_B200_LIB=tools/libnsfr_sym.so NSFR_PARITY_REPORT=$O/parity_report_sym.md timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_sym.log 2>&1; tail -3 $O/pytest_sym.log
