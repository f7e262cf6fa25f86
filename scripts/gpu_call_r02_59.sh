for i in 1 2; do for cfg in "X=1" "SIMBA_DPW_LATE=8" "SIMBA_DPW_LATE=16" "SIMBA_DPW_LATE=24"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 30
done; done
