#!/bin/bash
O=gpurun_out; mkdir -p $O
NSFR_PROBE_C=1e-6 tools/ab.sh "6x40" cur t7_256 t7_128 > $O/ab_t7c.jsonl 2> $O/ab_t7c.err; cat $O/ab_t7c.jsonl; tail -2 $O/ab_t7c.err
