timeout 300 python scripts/probe_launch_lat.py s11_k4_i10 s11_k4_i02 s12_k4_i09 > gpurun_out/c68.log 2>&1
