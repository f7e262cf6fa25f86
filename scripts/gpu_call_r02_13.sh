for i in 1 2; do for cfg in "SIMBA_R0_ROWS=16" "SIMBA_R0_ROWS=8" "SIMBA_R0_ROWS=4" "SIMBA_R0_ROWS=2" "SIMBA_R0_ROWS=4 SIMBA_SPLIT_MIN=131072"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_shapes.py 0:0
done; done
