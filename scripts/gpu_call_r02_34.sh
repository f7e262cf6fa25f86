sha256sum paper_2605_08243_b200/_lib/libsimba.so
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c34_gpu.log 2>&1; tail -3 gpurun_out/c34_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c34_smoke.log 2>&1; tail -2 gpurun_out/c34_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/c34_bench.log 2>&1; tail -c 400 gpurun_out/c34_bench.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:unit_kernel -c 1 -o gpurun_out/c34_unit python scripts/probe_fused_once.py > gpurun_out/c34_ncu.log 2>&1; tail -1 gpurun_out/c34_ncu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c34_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-tts --e2e-steps 1 > /dev/null 2>&1; wc -l gpurun_out/c34_launches.csv
timeout 900 python scripts/configs.py > gpurun_out/c34_configs.json 2> /dev/null; head -c 300 gpurun_out/c34_configs.json
