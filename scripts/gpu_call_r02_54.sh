timeout 600 python scripts/probe_shapes.py 0:0
for i in 1 2; do for cfg in "SIMBA_FUSED_SHARDS=0" "SIMBA_FUSED_SHARDS=1"; do for N in 2 4; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_shards.py $N
done; done; done
