#!/bin/bash
# Round profiling on the GPU box, leaving only small summaries under
# gpurun_out/prof (the .ncu-rep files stay in /tmp: gpurun returns <= 64 MiB):
#   1. bench.py exits 0 without ncu
#   2. the ncu launch list of the same command (gpu__time_duration.sum)
#   3. one `ncu --set full` capture per hot kernel -> markdown summary,
#      per-line FP64/other instruction split, DRAM traffic JSON (K2/K3)
# usage: [NO_LAUNCH_LIST=1] tools/profile_round.sh [kernel-regex ...]
OUT=gpurun_out/prof
mkdir -p $OUT
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > $OUT/bench_plain.log 2>&1 || { echo "bench failed"; exit 1; }
if [ -z "$NO_LAUNCH_LIST" ]; then
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_raw.csv $CMD > $OUT/ncu_ll.log 2>&1
  echo "launch list rc=$?"
fi
KERNELS=${@:-k_residual k_update k_convert_lines k_project}
for k in $KERNELS; do
  skip=4
  [ "$k" = "k_project" ] && skip=0
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -s $skip -c 1 \
    -o /tmp/full_$k -f $CMD > $OUT/ncu_$k.log 2>&1
  echo "$k rc=$?"
  python tools/ncu_report.py /tmp/full_$k.ncu-rep "ncu --set full: $k at the bench workload" \
    "ncu --set full --import-source on --clock-control none -k regex:$k -s $skip -c 1 $CMD" \
    $OUT/$k.md > /dev/null 2>&1
  python tools/ncu_ops_by_line.py /tmp/full_$k.ncu-rep 40 > $OUT/${k}_ops_by_line.txt 2>&1
  python tools/ncu_opcode_hist.py /tmp/full_$k.ncu-rep 40 > $OUT/${k}_opcodes.txt 2>&1
  [ "$k" = "k_residual" ] && cp /tmp/full_$k.ncu-rep $OUT/ 2>/dev/null
  for r in barrier wait short_sb long_sb mio lg; do
    python tools/ncu_stall_by_line.py /tmp/full_$k.ncu-rep $r 10; done > $OUT/${k}_stalls_by_line.txt 2>&1
  case $k in
    k_residual|k_update) python tools/ncu_traffic.py /tmp/full_$k.ncu-rep 2097152 $OUT/${k}_traffic.json $k > /dev/null 2>&1 ;;
  esac
done
ls -la $OUT
