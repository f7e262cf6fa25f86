for i in 1 2; do for cfg in "SIMBA_SUPER_PER_SHARD=16" "SIMBA_SUPER_PER_SHARD=4" "SIMBA_SUPER_PER_SHARD=1" "SIMBA_SUPER_PER_SHARD=64"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_shapes.py 0:0
done; done
