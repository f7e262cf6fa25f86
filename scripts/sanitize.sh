#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on the production unit
# kernel with the big-launch shapes, R0 + 1, partial-row planning and late
# splitting forced (scripts/sanitize_case.py).  Logs: gpurun_out/san_*.txt
export SIMBA_BIG_LAUNCH=1 SIMBA_SPLIT_MIN=4096
for tool in memcheck racecheck synccheck; do
  for c in "k2 9" "k4 8"; do
    set -- $c
    SIMBA_R0_UP=$2 timeout 1200 compute-sanitizer --tool $tool --kernel-name kns=unit_kernel \
      python scripts/sanitize_case.py $1 > gpurun_out/san_${tool}_$1.txt 2>&1
    echo "$tool $1 rc=$? $(tail -2 gpurun_out/san_${tool}_$1.txt | tr '\n' ' ')"
  done
done
# the adaptive-table path (example 0 dense: its table and density, the other
# example's table added in place, the examples reordered; 64-bit words), then
# level-guided searches -- every kernel of the context, not only unit_kernel
unset SIMBA_BIG_LAUNCH SIMBA_SPLIT_MIN
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool python scripts/sanitize_case.py adapt > gpurun_out/san_${tool}_adapt.txt 2>&1
  echo "$tool adapt rc=$? $(tail -2 gpurun_out/san_${tool}_adapt.txt | tr '\n' ' ')"
done
