for cfg in "X=1" "SIMBA_SPLIT_MIN=131072" "SIMBA_SPLIT_MIN=2097152" "X=1"; do echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 40; done
