# context-creation phase times (SIMBA_TRACE_CTX=1)
SIMBA_TRACE_CTX=1 timeout 300 python scripts/probe_tts.py s11_k4_i10 s12_k4_i08 s12_k4_i09 s13_k4_i03 > gpurun_out/c65.log 2>&1
