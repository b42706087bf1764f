#!/bin/bash
O=gpurun_out; mkdir -p $O
tools/ab.sh "4x128 5x64 3x96 6x40" fuse fdiv > $O/ab_fdiv.jsonl 2> $O/ab_fdiv.err
cat $O/ab_fdiv.jsonl
NO_LAUNCH_LIST=1 tools/profile_round.sh k_residual k_update > $O/prof_fdiv.log 2>&1; tail -3 $O/prof_fdiv.log
