#!/bin/bash
# round-2 GPU call 1: parity suite (with per-case report), compute-sanitizer tools
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/r02a_env.txt; free -g >> $O/r02a_env.txt; nproc >> $O/r02a_env.txt
export NSFR_PARITY_REPORT=$O/r02a_parity.jsonl; rm -f $NSFR_PARITY_REPORT
timeout 2400 python -m pytest tests -m gpu -q -k "not trajectory" -p no:cacheprovider > $O/r02a_gpu_tests.log 2>&1
echo "pytest rc=$?" >> $O/r02a_gpu_tests.log
unset NSFR_PARITY_REPORT
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py > $O/r02a_sanitize_$tool.log 2>&1
  echo "rc=$?" >> $O/r02a_sanitize_$tool.log
done
