timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c19_gpu.log 2>&1; tail -3 gpurun_out/c19_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c19_smoke.log 2>&1; tail -2 gpurun_out/c19_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/c19_bench.log 2>&1; tail -c 600 gpurun_out/c19_bench.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:unit_kernel -c 1 -o gpurun_out/c19_unit python scripts/probe_fused_once.py > gpurun_out/c19_ncu.log 2>&1; tail -1 gpurun_out/c19_ncu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c19_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-tts --e2e-steps 1 > /dev/null 2>&1; wc -l gpurun_out/c19_launches.csv
