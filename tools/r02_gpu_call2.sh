#!/bin/bash
O=gpurun_out
export NSFR_PARITY_REPORT=$O/r02b_parity.jsonl; rm -f $NSFR_PARITY_REPORT
timeout 2400 python -m pytest tests -m gpu -q -k "not trajectory" -p no:cacheprovider > $O/r02b_gpu_tests.log 2>&1
echo "pytest rc=$?" >> $O/r02b_gpu_tests.log
unset NSFR_PARITY_REPORT
timeout 900 python bench.py --steps 5 --warmup 3 > $O/r02b_bench.json 2> $O/r02b_bench.err
echo "bench rc=$?" >> $O/r02b_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/r02b_bench_ref.json 2> $O/r02b_bench_ref.err
