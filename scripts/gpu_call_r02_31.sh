timeout 900 python scripts/configs.py > gpurun_out/c31_configs.json 2> gpurun_out/c31_configs.err; tail -c 3000 gpurun_out/c31_configs.json; tail -3 gpurun_out/c31_configs.err
