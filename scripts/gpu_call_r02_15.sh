for cfg in "SIMBA_L2_PERSIST=1" "SIMBA_L2_PERSIST=0" "SIMBA_EX0_DENSE=2"; do echo "== $cfg"; env $cfg timeout 120 python scripts/probe_e2e.py; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:unit_kernel -c 1 -o gpurun_out/c15_unit python scripts/probe_fused_once.py > gpurun_out/c15_ncu.log 2>&1; tail -2 gpurun_out/c15_ncu.log
