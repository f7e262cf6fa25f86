for cfg in "X=1" "SIMBA_L2_PERSIST=0" "SIMBA_EX0_DENSE=1e9" "SIMBA_L2_PERSIST=0 SIMBA_EX0_DENSE=1e9"; do echo "== $cfg"; env $cfg timeout 120 python scripts/probe_ctx.py; done
