#!/bin/bash
# A/B of library variants + one full ncu capture of K2 with the working-tree library
O=gpurun_out; mkdir -p $O
SIZES=${SIZES:-"4x128 4x96 5x64 3x96"}
tools/ab.sh "$SIZES" $VARIANTS > $O/ab_$TAG.jsonl 2> $O/ab_$TAG.err
cat $O/ab_$TAG.jsonl
if [ -n "$NCU" ]; then
  NO_LAUNCH_LIST=1 tools/profile_round.sh k_residual > $O/prof_$TAG.log 2>&1
  tail -3 $O/prof_$TAG.log
fi
