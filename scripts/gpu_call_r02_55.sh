for i in 1 2; do
for cfg in "SIMBA_FUSED_SHARDS=1" "SIMBA_FUSED_SHARDS=1 SIMBA_BIG_LAUNCH=20000000000"; do echo "== $cfg N4"; env $cfg timeout 300 python scripts/probe_shards.py 4; done
for cfg in "SIMBA_FUSED_SHARDS=1" "SIMBA_FUSED_SHARDS=1 SIMBA_BIG_LAUNCH=10000000000"; do echo "== $cfg N8"; env $cfg timeout 300 python scripts/probe_shards.py 8; done
done
