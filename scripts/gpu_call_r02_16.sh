export SIMBA_BENCH_BACKEND=gloo SIMBA_BENCH_DEVICE=0
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/c16_bench2.log 2>&1; tail -c 1500 gpurun_out/c16_bench2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 8 --steps 3 --warmup 3 --no-cpu > gpurun_out/c16_bench8.log 2>&1; tail -c 1500 gpurun_out/c16_bench8.log
