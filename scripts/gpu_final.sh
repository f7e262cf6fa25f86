# round-2 final validation: tests, smoke, bench, ncu of the bench launch, launch list, configs, multi-rank protocol
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/fin_gpu.log 2>&1; tail -3 gpurun_out/fin_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; tail -2 gpurun_out/fin_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/fin_bench.log 2>&1; tail -c 300 gpurun_out/fin_bench.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:unit_kernel -c 1 -o gpurun_out/fin_unit python scripts/probe_fused_once.py > gpurun_out/fin_ncu.log 2>&1; tail -1 gpurun_out/fin_ncu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-tts --e2e-steps 1 > /dev/null 2>&1; wc -l gpurun_out/fin_launches.csv
timeout 900 python scripts/configs.py > gpurun_out/fin_configs.json 2> /dev/null; head -c 200 gpurun_out/fin_configs.json
export SIMBA_BENCH_BACKEND=gloo SIMBA_BENCH_DEVICE=0
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/fin_bench2.log 2>&1; tail -c 300 gpurun_out/fin_bench2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 8 --steps 3 --warmup 3 --no-cpu > gpurun_out/fin_bench8.log 2>&1; tail -c 300 gpurun_out/fin_bench8.log
