#!/bin/bash
O=gpurun_out; mkdir -p $O
tools/ab.sh "4x128 3x96 5x64" onef onelog > $O/ab_onelog.jsonl 2> $O/ab_onelog.err
cat $O/ab_onelog.jsonl; tail -3 $O/ab_onelog.err
NSFR_B200_LIB=tools/libnsfr_onef.so NSFR_PARITY_REPORT=$O/parity_report_onef.md timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/pytest_p_onef.log 2>&1; tail -2 $O/pytest_p_onef.log
NSFR_B200_LIB=tools/libnsfr_onelog.so NSFR_PARITY_REPORT=$O/parity_report_onelog.md timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_onelog.log 2>&1; tail -2 $O/pytest_onelog.log
