# tiles above a recorded hit skipped at execution; fusion x level guidance again
for cfg in "67108864 0" "2147483648 0" "17179869184 0" "1099511627776 0" "1099511627776 1" "1099511627776 5"; do set -- $cfg
  echo "== SIMBA_FUSE_CANDS=$1 SIMBA_LEVEL_GUIDE=$2"; SIMBA_FUSE_CANDS=$1 SIMBA_LEVEL_GUIDE=$2 timeout 300 python scripts/probe_tts.py
done > gpurun_out/c75.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c75_gpu.log 2>&1
