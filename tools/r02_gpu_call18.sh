#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_onef.log 2>&1; tail -3 $O/pytest_onef.log
NO_LAUNCH_LIST=1 tools/profile_round.sh k_update > $O/prof_onef.log 2>&1; tail -3 $O/prof_onef.log
