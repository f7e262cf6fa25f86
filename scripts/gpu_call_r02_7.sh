sha256sum paper_2605_08243_b200/_lib/libsimba.so > gpurun_out/c7_libsha.txt
timeout 300 python scripts/probe_shapes.py 0:0
timeout 300 python scripts/probe_int_peak.py
timeout 300 ncu --clock-control none -k regex:int_pipe_kernel --metrics sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,gpu__time_duration.sum python scripts/probe_int_peak.py > gpurun_out/c7_ncu_peak.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:unit_kernel -c 1 -o gpurun_out/c7_unit python scripts/probe_fused_once.py > gpurun_out/c7_ncu.log 2>&1; tail -2 gpurun_out/c7_ncu.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c7_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-tts --e2e-steps 1 > gpurun_out/c7_bench_under_ncu.log 2>&1; tail -2 gpurun_out/c7_launches.csv
