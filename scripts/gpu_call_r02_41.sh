for i in 1 2; do for cfg in "X=1" "SIMBA_SHARD_PG=0" "SIMBA_SHARD_PG=2" "SIMBA_SHARD_DPW=32" "SIMBA_SHARD_DPW=16" "SIMBA_SHARD_DPW=32 SIMBA_SHARD_PG=0" "SIMBA_GUIDE=8"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_shards.py 8
done; done
