timeout 1200 python -m pytest tests/test_production_paths.py tests/test_gpu_parity.py -q -x > gpurun_out/c38_tests.log 2>&1; tail -2 gpurun_out/c38_tests.log
for i in 1 2; do for cfg in "X=1" "SIMBA_DPW_RT=24" "SIMBA_DPW_RT=20"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 30; env $cfg timeout 300 python scripts/probe_shapes.py 0:0
done; done
