timeout 1200 python -m pytest tests/test_production_paths.py tests/test_gpu_parity.py tests/test_xbest.py -q -x > gpurun_out/c35_tests.log 2>&1; tail -2 gpurun_out/c35_tests.log
for i in 1 2; do for cfg in "SIMBA_SMEM_QUEUE=1" "SIMBA_SMEM_QUEUE=0"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 30; env $cfg timeout 300 python scripts/probe_shapes.py 0:0
done; done
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:unit_kernel -c 1 python scripts/probe_fused_once.py 2>&1 | grep -E "dram|duration"
