timeout 1200 python -m pytest tests/test_production_paths.py tests/test_gpu_parity.py tests/test_xbest.py -q -x > gpurun_out/c27_tests.log 2>&1; tail -3 gpurun_out/c27_tests.log
for i in 1 2; do for cfg in "SIMBA_STEAL=1" "SIMBA_STEAL=0" "SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/libsimba_head.so"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 40; env $cfg timeout 300 python scripts/probe_shapes.py 0:0
done; done
