SIMBA_LIB=build/libsimba_stats.so timeout 300 python scripts/probe_small_stats.py 1..9 9..9 10..10 11..11 12..12 > gpurun_out/c70.log 2>&1
