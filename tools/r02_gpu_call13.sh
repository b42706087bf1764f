#!/bin/bash
# checkpoint validation of the fused-face / mapped build: tests, smoke, bench, profiles, debug-checks build, config table
O=gpurun_out; mkdir -p $O
NSFR_PARITY_REPORT=$O/parity_report.md timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
python __graft_entry__.py --smoke > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; cat $O/bench.json
tools/profile_round.sh > $O/prof.log 2>&1; tail -4 $O/prof.log
tools/debug_checks.sh; cat $O/debug_verdict.txt; tail -2 $O/debug_tests.log
timeout 1500 python tools/config_table.py > $O/config_table.md 2> $O/config_table.err; tail -12 $O/config_table.md
