#!/bin/bash
O=gpurun_out; mkdir -p $O
for rep in 1 2; do for v in 0 1 2 0.5; do NSFR_UPD_PERSIST=$v python tools/perf_probe.py 4x128 4x64 | sed "s/\"lib\": \"default\"/\"lib\": \"persist_$v\"/"; done; done > $O/ab_persist.jsonl 2> $O/ab_persist.err
cat $O/ab_persist.jsonl; tail -3 $O/ab_persist.err
NSFR_UPD_PERSIST=1 timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_persist.log 2>&1; tail -3 $O/pytest_persist.log
