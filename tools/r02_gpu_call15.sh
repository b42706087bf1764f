#!/bin/bash
O=gpurun_out; mkdir -p $O
tools/ab.sh "4x128 4x64" mapf k3t320 k3f2 > $O/ab_k3t.jsonl 2> $O/ab_k3t.err
cat $O/ab_k3t.jsonl; tail -3 $O/ab_k3t.err
