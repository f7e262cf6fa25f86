#!/bin/bash
# finer queue size classes (libsimba_c8.so = -DSIMBA_SIZE_CLASSES=8): full GPU suite, 16 dense stress runs, sweep A/B
SIMBA_LIB=paper_2605_08243_b200/_lib/libsimba_c8.so timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
ok=0; bad=0
for i in $(seq 1 16); do
  if [ $((i % 2)) = 0 ]; then export SIMBA_SPLIT_MIN=2048; else unset SIMBA_SPLIT_MIN; fi
  out=$(SIMBA_LIB=paper_2605_08243_b200/_lib/libsimba_c8.so timeout 30 python scripts/hang_case.py 1 12 2>&1 | tail -1)
  case "$out" in ok*1451548*) ok=$((ok+1));; *) bad=$((bad+1)); echo "run $i: ${out:0:300}";; esac
done
unset SIMBA_SPLIT_MIN
echo "dense stress ok=$ok bad=$bad"
bash scripts/fused_ab.sh sg4 c8
bash scripts/shards8_ab.sh sg4 c8
