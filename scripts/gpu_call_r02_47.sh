for i in 1 2; do for cfg in "X=1" "SIMBA_DPW_LATE=8" "SIMBA_DPW_LATE=10" "SIMBA_DPW_LATE=6"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 30
done; done
