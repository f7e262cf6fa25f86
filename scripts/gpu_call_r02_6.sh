# A/B: L2 persisting window on the value table; claim guide 2 vs 4 (big launches)
for i in 1 2; do
for cfg in "SIMBA_L2_PERSIST=1" "SIMBA_L2_PERSIST=0" "SIMBA_GUIDE=2" "SIMBA_GUIDE=2 SIMBA_L2_PERSIST=0"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_shapes.py 0:0
done
done
