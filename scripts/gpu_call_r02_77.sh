# new synthesize defaults (all levels fused, level-guided, search dpw 12, exec skip): parity, TTS, bench, configs
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c77_gpu.log 2>&1
timeout 300 python scripts/probe_tts.py > gpurun_out/c77_probe.log 2>&1
for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/c77_bench$i.log 2>&1; done
timeout 900 python scripts/configs.py > gpurun_out/c77_configs.json 2> /dev/null
