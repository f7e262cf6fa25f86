# level-guided fused searches: fusion threshold x guidance (probe_tts: best of 3 per target after the first)
for f in 67108864 2147483648 17179869184 1099511627776; do for g in 0 1; do
  echo "== SIMBA_FUSE_CANDS=$f SIMBA_LEVEL_GUIDE=$g"; SIMBA_FUSE_CANDS=$f SIMBA_LEVEL_GUIDE=$g timeout 300 python scripts/probe_tts.py
done; done > gpurun_out/c72.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c72_gpu.log 2>&1
