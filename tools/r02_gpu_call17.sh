#!/bin/bash
O=gpurun_out; mkdir -p $O
tools/ab.sh "4x128 3x96 5x64" sym one onef > $O/ab_one.jsonl 2> $O/ab_one.err
cat $O/ab_one.jsonl; tail -3 $O/ab_one.err
