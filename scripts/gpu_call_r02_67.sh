# pooled streams: parity + context-creation phases + TTS (x2 bench processes)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c67_gpu.log 2>&1
SIMBA_TRACE_CTX=1 timeout 300 python scripts/probe_tts.py s11_k4_i10 s12_k4_i08 s12_k4_i09 s13_k4_i03 s13_k4_i04 > gpurun_out/c67_trace.log 2>&1
timeout 300 python scripts/probe_tts.py > gpurun_out/c67_probe.log 2>&1
for i in 1 2 3; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/c67_bench$i.log 2>&1; done
