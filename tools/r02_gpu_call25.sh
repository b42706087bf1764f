#!/bin/bash
O=gpurun_out; mkdir -p $O
tools/ab.sh "5x64 6x40" cur t6_96 t6_192 t6_224 t7_128 t7_256 > $O/ab_t67.jsonl 2> $O/ab_t67.err; cat $O/ab_t67.jsonl; tail -2 $O/ab_t67.err
