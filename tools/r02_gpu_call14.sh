#!/bin/bash
O=gpurun_out; mkdir -p $O
tools/ab.sh "4x128 4x64" mapf k3r48 k3r48l > $O/ab_k3r.jsonl 2> $O/ab_k3r.err
cat $O/ab_k3r.jsonl; tail -3 $O/ab_k3r.err
