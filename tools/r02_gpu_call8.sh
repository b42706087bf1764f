#!/bin/bash
# re-entry validation: GPU tests, bench (default and reference arm), full profile round
O=gpurun_out; mkdir -p $O
NSFR_PARITY_REPORT=$O/parity_report.md timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
python __graft_entry__.py --smoke > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; cat $O/bench.json
tools/profile_round.sh > $O/prof.log 2>&1; tail -12 $O/prof.log
