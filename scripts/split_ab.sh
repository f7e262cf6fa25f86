#!/bin/bash
# fused C5 sweep device time vs the late-splitting threshold (SIMBA_SPLIT_MIN), 3 interleaved rounds
for r in 1 2 3; do for m in 65536 131072 262144 524288 1048576; do
  echo -n "split_min $m r$r: "; SIMBA_SPLIT_MIN=$m bash scripts/fused_ab.sh cur 2>&1 | head -1 | sed 's/^cur r1: //'
done; done
