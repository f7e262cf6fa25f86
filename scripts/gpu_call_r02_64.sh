# TTS outliers: full bench process (after the sweep + e2e) vs eager module loading
for i in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/c64_b$i.log 2>&1; done
CUDA_MODULE_LOADING=EAGER timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/c64_eager.log 2>&1
timeout 600 python scripts/probe_tts.py > gpurun_out/c64_probe.log 2>&1
