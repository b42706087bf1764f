#!/bin/bash
O=gpurun_out; mkdir -p $O
tools/ab.sh "3x96 5x64 6x40 4x64" fdiv map mapf > $O/ab_map.jsonl 2> $O/ab_map.err
cat $O/ab_map.jsonl; tail -3 $O/ab_map.err
