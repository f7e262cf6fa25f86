# all levels fused: which part of the level guidance costs at size 13
for g in 0 7 1 3 5 6; do
  echo "== SIMBA_FUSE_CANDS=2^40 SIMBA_LEVEL_GUIDE=$g"; SIMBA_FUSE_CANDS=1099511627776 SIMBA_LEVEL_GUIDE=$g timeout 300 python scripts/probe_tts.py
done > gpurun_out/c74.log 2>&1
