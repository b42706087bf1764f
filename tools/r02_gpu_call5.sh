#!/bin/bash
O=gpurun_out
export NSFR_PARITY_REPORT=$O/r02d_parity.jsonl; rm -f $NSFR_PARITY_REPORT
timeout 2400 python -m pytest tests -m gpu -q -k "not trajectory" -p no:cacheprovider > $O/r02d_gpu_tests.log 2>&1
echo "pytest rc=$?" >> $O/r02d_gpu_tests.log
unset NSFR_PARITY_REPORT
timeout 1200 python tools/config_table.py 20 > $O/r02d_config_table.log 2>&1
timeout 1200 python bench.py --steps 100 --warmup 3 > $O/r02d_bench100.json 2> $O/r02d_bench100.err
