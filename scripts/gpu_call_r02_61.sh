for i in 1 2; do for cfg in "X=1" "SIMBA_SPLIT_MIN=524288" "SIMBA_SPLIT_MIN=262144"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_shapes.py 0:0; env $cfg timeout 300 python scripts/probe_shards.py 2; env $cfg timeout 300 python scripts/probe_variance.py 20
done; done
