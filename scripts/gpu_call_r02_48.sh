for i in 1 2; do for cfg in "X=1" "SIMBA_DPW_LATE=12" "SIMBA_DPW_LATE=16"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_shapes.py 0:0; env $cfg timeout 300 python scripts/probe_shards.py 8
done; done
