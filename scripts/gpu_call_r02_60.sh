for i in 1 2; do for cfg in "X=1" "SIMBA_R0_UP=11" "SIMBA_R0_UP=13" "SIMBA_GUIDE=3" "SIMBA_SPLIT_MIN=524288"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 30
done; done
