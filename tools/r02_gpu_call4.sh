#!/bin/bash
O=gpurun_out
bash tools/debug_checks.sh
export NSFR_PARITY_REPORT=$O/r02c_parity.jsonl; rm -f $NSFR_PARITY_REPORT
timeout 2400 python -m pytest tests -m gpu -q -k "not trajectory" -p no:cacheprovider > $O/r02c_gpu_tests.log 2>&1
echo "pytest rc=$?" >> $O/r02c_gpu_tests.log
unset NSFR_PARITY_REPORT
timeout 900 python bench.py --steps 10 --warmup 3 > $O/r02c_bench.json 2> $O/r02c_bench.err
