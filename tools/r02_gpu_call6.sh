#!/bin/bash
O=gpurun_out
mkdir -p $O
export NSFR_PARITY_REPORT=$O/r02e_parity.jsonl; rm -f $NSFR_PARITY_REPORT
timeout 2400 python -m pytest tests -m gpu -q -k "not trajectory" -p no:cacheprovider > $O/r02e_gpu_tests.log 2>&1
echo "pytest rc=$?" >> $O/r02e_gpu_tests.log
unset NSFR_PARITY_REPORT
timeout 900 python bench.py --steps 10 --warmup 3 > $O/r02e_bench.json 2> $O/r02e_bench.err
python -c "import __graft_entry__ as g; g.smoke()" > $O/r02e_smoke.log 2>&1
tail -3 $O/r02e_gpu_tests.log; cat $O/r02e_bench.json; cat $O/r02e_smoke.log
