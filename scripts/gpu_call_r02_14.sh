timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c14_gpu.log 2>&1; tail -3 gpurun_out/c14_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c14_smoke.log 2>&1; tail -2 gpurun_out/c14_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/c14_bench.log 2>&1; tail -c 2500 gpurun_out/c14_bench.log
