# in-place adaptive E: parity + context-creation phases + TTS
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c66_gpu.log 2>&1
SIMBA_TRACE_CTX=1 timeout 300 python scripts/probe_tts.py s11_k4_i10 s12_k4_i08 s12_k4_i09 s13_k4_i03 > gpurun_out/c66_trace.log 2>&1
timeout 300 python scripts/probe_tts.py > gpurun_out/c66_probe.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/c66_bench.log 2>&1
