# synthesize level fusion: 2^26 (levels 1..9 | 10 | 11 | 12 | 13) vs 2^31 (1..11 | 12 | 13) vs 2^34 (1..12 | 13)
for f in 67108864 2147483648 17179869184 67108864 2147483648 17179869184; do
  echo "== SIMBA_FUSE_CANDS=$f"; SIMBA_FUSE_CANDS=$f timeout 300 python scripts/probe_tts.py
done > gpurun_out/c71.log 2>&1
