timeout 1500 python -m pytest tests/test_production_paths.py tests/test_gpu_parity.py tests/test_xbest.py -q -x > gpurun_out/c57_tests.log 2>&1; tail -2 gpurun_out/c57_tests.log
for i in 1 2; do for cfg in "SIMBA_SHARED_CAP=1" "SIMBA_SHARED_CAP=0"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 30; env $cfg timeout 300 python scripts/probe_shapes.py 0:0
done; done
