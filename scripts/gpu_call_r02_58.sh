for i in 1 2; do for cfg in "SIMBA_SHARED_CAP=1" "SIMBA_SHARED_CAP=0"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_shapes.py 0:0; env $cfg timeout 300 python scripts/probe_shards.py 2
done; done
