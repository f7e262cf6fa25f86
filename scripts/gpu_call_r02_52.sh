for i in 1 2; do for cfg in "X=1" "SIMBA_GUIDE=1" "SIMBA_GUIDE=3" "SIMBA_GUIDE=4" "SIMBA_DPW_LATE=16"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 30
done; done
