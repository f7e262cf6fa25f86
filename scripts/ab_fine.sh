#!/bin/bash
# A/B of partial-row planning (SIMBA_FINE_ROW) and the R0+1 claim condition
# (SIMBA_R0_ROWS) on the full C5 sweep and its 8-way shards.
for cfg in "SIMBA_FINE_ROW=0" "" "SIMBA_R0_ROWS=4" "SIMBA_R0_ROWS=1" "SIMBA_FINE_ROW=0 SIMBA_R0_ROWS=1"; do
  echo "== $cfg"
  env $cfg python scripts/probe_shapes.py 0:0
done
