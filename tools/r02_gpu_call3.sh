#!/bin/bash
# debug-check build vs release (sanitizer substitute), then the round profile
bash tools/debug_checks.sh
bash tools/profile_round.sh k_residual k_update k_project k_convert_lines > gpurun_out/prof_round.log 2>&1
