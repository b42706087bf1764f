#!/bin/bash
O=gpurun_out; mkdir -p $O
tools/ab.sh "4x128 4x64" cur r136 > $O/ab_r136.jsonl 2> $O/ab_r136.err; cat $O/ab_r136.jsonl; tail -2 $O/ab_r136.err
