timeout 1200 python -m pytest tests/test_production_paths.py tests/test_gpu_parity.py -q -x > gpurun_out/c12_tests.log 2>&1; tail -2 gpurun_out/c12_tests.log
echo "== stats"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/libsimba_stats.so timeout 300 python scripts/probe_shard_stats.py 2>&1 | grep -v "   cyc\|   w_"
for i in 1 2 3; do for lib in libsimba.so libsimba_abs1.so; do
  echo "== $lib"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_shapes.py 0:0
done; done
