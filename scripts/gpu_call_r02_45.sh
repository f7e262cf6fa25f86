timeout 1200 python -m pytest tests/test_production_paths.py tests/test_gpu_parity.py tests/test_xbest.py -q -x > gpurun_out/c45_tests.log 2>&1; tail -2 gpurun_out/c45_tests.log
for i in 1 2; do for lib in libsimba.so libsimba_head.so; do
  echo "== $lib"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_variance.py 30; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_shapes.py 0:0
done; done
