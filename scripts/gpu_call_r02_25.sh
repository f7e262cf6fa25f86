timeout 1200 python -m pytest tests/test_production_paths.py tests/test_gpu_parity.py tests/test_xbest.py -q -x > gpurun_out/c25_tests.log 2>&1; tail -3 gpurun_out/c25_tests.log
for cfg in "SIMBA_STEAL=1" "SIMBA_STEAL=0" "SIMBA_STEAL=1" "SIMBA_STEAL=0"; do echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 40; env $cfg timeout 300 python scripts/probe_shapes.py 0:0; done
