#!/bin/bash
# Sanitizer substitute (compute-sanitizer is closed on this pool): build the
# -DNSFR_DEBUG_CHECKS variant (csrc/debug_checks.cuh), check it reproduces the
# release build bitwise on every kernel family, and run the GPU parity tests
# against it. Writes gpurun_out/debug_*.
set -u
O=gpurun_out
python tools/debug_compare.py > $O/debug_release.json 2> $O/debug_release.err; rc1=$?
NSFR_B200_LIB=tools/libnsfr_dbg.so python tools/debug_compare.py > $O/debug_checked.json 2> $O/debug_checked.err; rc2=$?
n=$(grep -c '"rhs"' $O/debug_release.json)
if [ $rc1 -ne 0 ] || [ $rc2 -ne 0 ] || [ "$n" -lt 10 ]; then echo "FAILED rc=$rc1/$rc2 configs=$n" > $O/debug_verdict.txt;
elif cmp -s $O/debug_release.json $O/debug_checked.json; then echo "BITWISE EQUAL ($n configurations)" > $O/debug_verdict.txt;
else echo "DIFFER" > $O/debug_verdict.txt; diff $O/debug_release.json $O/debug_checked.json >> $O/debug_verdict.txt; fi
NSFR_B200_LIB=tools/libnsfr_dbg.so timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider \
  -k "not trajectory and not config3_p4 and not config2" > $O/debug_tests.log 2>&1
echo "pytest rc=$?" >> $O/debug_tests.log
