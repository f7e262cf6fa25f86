SIMBA_LIB=build/libsimba_cta.so timeout 300 python scripts/probe_small_launch.py 1..9 10..10 11..11 > gpurun_out/c69.log 2>&1
