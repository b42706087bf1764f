#!/bin/bash
# final validation of the round: tests, smoke, bench (10 and 100 steps, reference arm), profiles, debug-checks build, config table
O=gpurun_out; mkdir -p $O
NSFR_PARITY_REPORT=$O/parity_report.md timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
python __graft_entry__.py --smoke > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; cut -c1-400 $O/bench.json
python bench.py --steps 100 --warmup 3 --no-cpu-baseline > $O/bench_100.json 2> $O/bench_100.err; echo "bench100 rc=$?"; cut -c1-300 $O/bench_100.json
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"; cut -c1-300 $O/bench_reference.json
tools/profile_round.sh > $O/prof.log 2>&1; tail -4 $O/prof.log
tools/debug_checks.sh; cat $O/debug_verdict.txt; tail -2 $O/debug_tests.log
timeout 1500 python tools/config_table.py > $O/config_table.md 2> $O/config_table.err; tail -8 $O/config_table.md | cut -c1-200
