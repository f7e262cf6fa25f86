# all levels fused + level-guided claims: claim guide and descriptors per warp
export SIMBA_FUSE_CANDS=1099511627776 SIMBA_LEVEL_GUIDE=1
for cfg in "X=1" "SIMBA_GUIDE=4" "SIMBA_GUIDE=8" "SIMBA_DPW_RT=12" "SIMBA_DPW_RT=8" "SIMBA_LEVEL_GUIDE=5" "SIMBA_GUIDE=4 SIMBA_DPW_RT=12"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_tts.py
done > gpurun_out/c76.log 2>&1
