timeout 1200 python -m pytest tests/test_production_paths.py tests/test_gpu_parity.py tests/test_vfb.py tests/test_cli.py -q -x > gpurun_out/c17_tests.log 2>&1; tail -2 gpurun_out/c17_tests.log
timeout 120 python scripts/probe_e2e.py
SIMBA_VT_DECODE=1 timeout 120 python scripts/probe_e2e.py
timeout 300 python scripts/probe_tts.py s11_k4_i02 s11_k4_i06 s12_k4_i09 s12_k4_i08
