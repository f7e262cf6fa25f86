for i in 1 2; do for cfg in "X=1" "SIMBA_DPW_LATE=0" "SIMBA_DPW_LATE=12" "SIMBA_DPW_RT=16 SIMBA_DPW_LATE=0"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 30
done; done
for cfg in "X=1" "SIMBA_SHARD_PG=0" "SIMBA_SHARD_DPW=16"; do echo "== $cfg"; env $cfg timeout 300 python scripts/probe_shards.py 8; done
