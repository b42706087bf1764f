#!/bin/bash
O=gpurun_out; mkdir -p $O
tools/ab.sh "4x128 3x96" cur map2 > $O/ab_map2.jsonl 2> $O/ab_map2.err; cat $O/ab_map2.jsonl; tail -2 $O/ab_map2.err
