#!/bin/bash
O=gpurun_out; mkdir -p $O
tools/ab.sh "3x96 5x64 4x64" h1 h2 > $O/ab_h2.jsonl 2> $O/ab_h2.err; cat $O/ab_h2.jsonl; tail -2 $O/ab_h2.err
