#!/bin/bash
# 8-way shard times under SIMBA_R0_UP / SIMBA_GUIDE overrides (claim length vs row length)
for cfg in "0 0" "13 1" "13 2" "13 4" "0 2" "0 4"; do
  set -- $cfg; echo "== R0_UP=$1 GUIDE=$2"
  env $( [ $1 != 0 ] && echo SIMBA_R0_UP=$1 ) $( [ $2 != 0 ] && echo SIMBA_GUIDE=$2 ) bash scripts/shards8_ab.sh new | tail -1
done
