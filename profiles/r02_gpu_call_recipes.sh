# The gpurun command files of round 2's A/B and probe calls, in call order
# (each ran as 'bash <file>' on one B200; its results are the profiles/r02_*.txt
# records named in DESIGN.md).  Kept here as provenance; scripts/gpu_final.sh is
# the final-validation recipe.

# ---- gpu_call_r02_4.sh
timeout 900 python -m pytest tests/test_xbest.py tests/test_production_paths.py -q > gpurun_out/c4_tests.log 2>&1; tail -3 gpurun_out/c4_tests.log
echo "== shapes default"; timeout 300 python scripts/probe_shapes.py 0:0 0:8
echo "== shapes row1 depth 1"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/libsimba_row1d1.so timeout 300 python scripts/probe_shapes.py 0:0
echo "== tts"; timeout 600 python scripts/probe_tts.py s12_k4_i08 s12_k4_i37 s12_k4_i09 s13_k4_i04 s13_k4_i03 s11_k4_i02
echo "== stats"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/libsimba_stats.so timeout 300 python scripts/probe_shard_stats.py
echo "== sanitize"; timeout 1500 bash scripts/sanitize.sh

# ---- gpu_call_r02_5.sh
# A/B: RF-tile column prefetch; shard claim guide / R0+1 row condition
for lib in libsimba.so libsimba_nopf.so libsimba.so libsimba_nopf.so; do
  echo "== $lib"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_shapes.py 0:0
done
for cfg in "SIMBA_GUIDE=1" "SIMBA_GUIDE=2" "SIMBA_GUIDE=2 SIMBA_R0_ROWS=8" "SIMBA_GUIDE=1 SIMBA_FINE_ROW=0"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_shapes.py 0:0
done

# ---- gpu_call_r02_6.sh
# A/B: L2 persisting window on the value table; claim guide 2 vs 4 (big launches)
for i in 1 2; do
for cfg in "SIMBA_L2_PERSIST=1" "SIMBA_L2_PERSIST=0" "SIMBA_GUIDE=2" "SIMBA_GUIDE=2 SIMBA_L2_PERSIST=0"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_shapes.py 0:0
done
done

# ---- gpu_call_r02_7.sh
sha256sum paper_2605_08243_b200/_lib/libsimba.so > gpurun_out/c7_libsha.txt
timeout 300 python scripts/probe_shapes.py 0:0
timeout 300 python scripts/probe_int_peak.py
timeout 300 ncu --clock-control none -k regex:int_pipe_kernel --metrics sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,gpu__time_duration.sum python scripts/probe_int_peak.py > gpurun_out/c7_ncu_peak.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:unit_kernel -c 1 -o gpurun_out/c7_unit python scripts/probe_fused_once.py > gpurun_out/c7_ncu.log 2>&1; tail -2 gpurun_out/c7_ncu.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c7_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-tts --e2e-steps 1 > gpurun_out/c7_bench_under_ncu.log 2>&1; tail -2 gpurun_out/c7_launches.csv

# ---- gpu_call_r02_8.sh
timeout 1200 python -m pytest tests/test_production_paths.py tests/test_gpu_parity.py tests/test_fold.py -q -x > gpurun_out/c8_tests.log 2>&1; tail -2 gpurun_out/c8_tests.log
for i in 1 2; do for lib in libsimba.so libsimba_noaff.so; do
  echo "== $lib"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_shapes.py 0:0
done; done

# ---- gpu_call_r02_9.sh
timeout 1200 python -m pytest tests/test_production_paths.py tests/test_gpu_parity.py -q -x > gpurun_out/c9_tests.log 2>&1; tail -2 gpurun_out/c9_tests.log
for i in 1 2; do for lib in libsimba.so libsimba_nocfpf.so; do
  echo "== $lib"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_shapes.py 0:0
done; done

# ---- gpu_call_r02_10.sh
echo "== stats"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/libsimba_stats.so timeout 300 python scripts/probe_shard_stats.py
for i in 1 2; do for lib in libsimba.so libsimba_dpw32.so libsimba_desc19.so; do
  echo "== $lib"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_shapes.py 0:0
done; done

# ---- gpu_call_r02_11.sh
timeout 1200 python -m pytest tests/test_production_paths.py tests/test_gpu_parity.py -q -x > gpurun_out/c11_tests.log 2>&1; tail -2 gpurun_out/c11_tests.log
echo "== stats"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/libsimba_stats.so timeout 300 python scripts/probe_shard_stats.py 2>&1 | grep -v "   cyc\|   ph_\|   w_"
for i in 1 2 3; do for cfg in "SIMBA_ABSORB=1" "SIMBA_ABSORB=0"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_shapes.py 0:0
done; done

# ---- gpu_call_r02_12.sh
timeout 1200 python -m pytest tests/test_production_paths.py tests/test_gpu_parity.py -q -x > gpurun_out/c12_tests.log 2>&1; tail -2 gpurun_out/c12_tests.log
echo "== stats"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/libsimba_stats.so timeout 300 python scripts/probe_shard_stats.py 2>&1 | grep -v "   cyc\|   w_"
for i in 1 2 3; do for lib in libsimba.so libsimba_abs1.so; do
  echo "== $lib"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_shapes.py 0:0
done; done

# ---- gpu_call_r02_13.sh
for i in 1 2; do for cfg in "SIMBA_R0_ROWS=16" "SIMBA_R0_ROWS=8" "SIMBA_R0_ROWS=4" "SIMBA_R0_ROWS=2" "SIMBA_R0_ROWS=4 SIMBA_SPLIT_MIN=131072"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_shapes.py 0:0
done; done

# ---- gpu_call_r02_14.sh
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c14_gpu.log 2>&1; tail -3 gpurun_out/c14_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c14_smoke.log 2>&1; tail -2 gpurun_out/c14_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/c14_bench.log 2>&1; tail -c 2500 gpurun_out/c14_bench.log

# ---- gpu_call_r02_15.sh
for cfg in "SIMBA_L2_PERSIST=1" "SIMBA_L2_PERSIST=0" "SIMBA_EX0_DENSE=2"; do echo "== $cfg"; env $cfg timeout 120 python scripts/probe_e2e.py; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:unit_kernel -c 1 -o gpurun_out/c15_unit python scripts/probe_fused_once.py > gpurun_out/c15_ncu.log 2>&1; tail -2 gpurun_out/c15_ncu.log

# ---- gpu_call_r02_16.sh
export SIMBA_BENCH_BACKEND=gloo SIMBA_BENCH_DEVICE=0
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/c16_bench2.log 2>&1; tail -c 1500 gpurun_out/c16_bench2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 8 --steps 3 --warmup 3 --no-cpu > gpurun_out/c16_bench8.log 2>&1; tail -c 1500 gpurun_out/c16_bench8.log

# ---- gpu_call_r02_17.sh
timeout 1200 python -m pytest tests/test_production_paths.py tests/test_gpu_parity.py tests/test_vfb.py tests/test_cli.py -q -x > gpurun_out/c17_tests.log 2>&1; tail -2 gpurun_out/c17_tests.log
timeout 120 python scripts/probe_e2e.py
SIMBA_VT_DECODE=1 timeout 120 python scripts/probe_e2e.py
timeout 300 python scripts/probe_tts.py s11_k4_i02 s11_k4_i06 s12_k4_i09 s12_k4_i08

# ---- gpu_call_r02_18.sh
timeout 1200 python -m pytest tests/test_production_paths.py tests/test_gpu_parity.py -q -x > gpurun_out/c18_tests.log 2>&1; tail -2 gpurun_out/c18_tests.log
for i in 1 2 3; do for lib in libsimba.so libsimba_rows4.so; do
  echo "== $lib"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_shapes.py 0:0
done; done

# ---- gpu_call_r02_19.sh
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c19_gpu.log 2>&1; tail -3 gpurun_out/c19_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c19_smoke.log 2>&1; tail -2 gpurun_out/c19_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/c19_bench.log 2>&1; tail -c 600 gpurun_out/c19_bench.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:unit_kernel -c 1 -o gpurun_out/c19_unit python scripts/probe_fused_once.py > gpurun_out/c19_ncu.log 2>&1; tail -1 gpurun_out/c19_ncu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c19_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-tts --e2e-steps 1 > /dev/null 2>&1; wc -l gpurun_out/c19_launches.csv

# ---- gpu_call_r02_20.sh
for cfg in "X=1" "SIMBA_SPLIT_MIN=131072" "SIMBA_SPLIT_MIN=2097152" "X=1"; do echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 40; done

# ---- gpu_call_r02_21.sh
for cfg in "SIMBA_SPLIT_MIN=32768" "SIMBA_SPLIT_MIN=65536" "SIMBA_SPLIT_MIN=131072" "SIMBA_SPLIT_MIN=262144" "SIMBA_SPLIT_MIN=524288"; do echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 40; done
for lib in libsimba_pg2.so libsimba_pg8.so; do echo "== $lib"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_variance.py 40; done
for lib in libsimba_pg2.so libsimba_pg8.so; do echo "== $lib split 131072"; SIMBA_SPLIT_MIN=131072 SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_variance.py 40; done

# ---- gpu_call_r02_22.sh
for cfg in "SIMBA_TAIL_DEN=0" "SIMBA_TAIL_DEN=16" "SIMBA_TAIL_DEN=8" "SIMBA_TAIL_DEN=32" "SIMBA_TAIL_DEN=16 SIMBA_TAIL_GUIDE=1" "SIMBA_TAIL_DEN=16 SIMBA_TAIL_GUIDE=4" "SIMBA_TAIL_DEN=0"; do echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 40; done

# ---- gpu_call_r02_23.sh
# per-CTA timelines of 6 launches of the full sweep (one launch per process)
for i in 1 2 3 4 5 6; do
  SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/libsimba_cta.so timeout 120 python scripts/probe_cta_times.py 1 0 > gpurun_out/c23_cta_$i.txt 2>&1
  grep KERNEL_MS gpurun_out/c23_cta_$i.txt; python scripts/cta_times.py gpurun_out/c23_cta_$i.txt
done

# ---- gpu_call_r02_24.sh
for cfg in "SIMBA_TAIL_GUIDE=0" "SIMBA_TAIL_GUIDE=1" "SIMBA_TAIL_GUIDE=2" "SIMBA_TAIL_GUIDE=4" "SIMBA_TAIL_GUIDE=0" "SIMBA_TAIL_GUIDE=1" "SIMBA_TAIL_GUIDE=2"; do echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 40; done

# ---- gpu_call_r02_25.sh
timeout 1200 python -m pytest tests/test_production_paths.py tests/test_gpu_parity.py tests/test_xbest.py -q -x > gpurun_out/c25_tests.log 2>&1; tail -3 gpurun_out/c25_tests.log
for cfg in "SIMBA_STEAL=1" "SIMBA_STEAL=0" "SIMBA_STEAL=1" "SIMBA_STEAL=0"; do echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 40; env $cfg timeout 300 python scripts/probe_shapes.py 0:0; done

# ---- gpu_call_r02_26.sh
for i in 1 2; do for lib in libsimba_head.so libsimba_nocall.so libsimba.so; do
  echo "== $lib"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_variance.py 40; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_shapes.py 0:0
done; done

# ---- gpu_call_r02_27.sh
timeout 1200 python -m pytest tests/test_production_paths.py tests/test_gpu_parity.py tests/test_xbest.py -q -x > gpurun_out/c27_tests.log 2>&1; tail -3 gpurun_out/c27_tests.log
for i in 1 2; do for cfg in "SIMBA_STEAL=1" "SIMBA_STEAL=0" "SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/libsimba_head.so"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 40; env $cfg timeout 300 python scripts/probe_shapes.py 0:0
done; done

# ---- gpu_call_r02_29.sh
for lib in libsimba_v1.so libsimba_v2.so libsimba_v3.so libsimba_head.so; do for st in 1 0; do
  echo "== $lib STEAL=$st"; SIMBA_STEAL=$st SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_variance.py 20; SIMBA_STEAL=$st SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_shapes.py 0:0
done; done

# ---- gpu_call_r02_30.sh
for i in 1 2; do for cfg in "SIMBA_SUPER_PER_SHARD=16" "SIMBA_SUPER_PER_SHARD=4" "SIMBA_SUPER_PER_SHARD=1" "SIMBA_SUPER_PER_SHARD=64"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_shapes.py 0:0
done; done

# ---- gpu_call_r02_31.sh
timeout 900 python scripts/configs.py > gpurun_out/c31_configs.json 2> gpurun_out/c31_configs.err; tail -c 3000 gpurun_out/c31_configs.json; tail -3 gpurun_out/c31_configs.err

# ---- gpu_call_r02_32.sh
for cfg in "X=1" "SIMBA_L2_PERSIST=0" "SIMBA_EX0_DENSE=1e9" "SIMBA_L2_PERSIST=0 SIMBA_EX0_DENSE=1e9"; do echo "== $cfg"; env $cfg timeout 120 python scripts/probe_ctx.py; done

# ---- gpu_call_r02_34.sh
sha256sum paper_2605_08243_b200/_lib/libsimba.so
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c34_gpu.log 2>&1; tail -3 gpurun_out/c34_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c34_smoke.log 2>&1; tail -2 gpurun_out/c34_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/c34_bench.log 2>&1; tail -c 400 gpurun_out/c34_bench.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:unit_kernel -c 1 -o gpurun_out/c34_unit python scripts/probe_fused_once.py > gpurun_out/c34_ncu.log 2>&1; tail -1 gpurun_out/c34_ncu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c34_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-tts --e2e-steps 1 > /dev/null 2>&1; wc -l gpurun_out/c34_launches.csv
timeout 900 python scripts/configs.py > gpurun_out/c34_configs.json 2> /dev/null; head -c 300 gpurun_out/c34_configs.json

# ---- gpu_call_r02_35.sh
timeout 1200 python -m pytest tests/test_production_paths.py tests/test_gpu_parity.py tests/test_xbest.py -q -x > gpurun_out/c35_tests.log 2>&1; tail -2 gpurun_out/c35_tests.log
for i in 1 2; do for cfg in "SIMBA_SMEM_QUEUE=1" "SIMBA_SMEM_QUEUE=0"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 30; env $cfg timeout 300 python scripts/probe_shapes.py 0:0
done; done
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:unit_kernel -c 1 python scripts/probe_fused_once.py 2>&1 | grep -E "dram|duration"

# ---- gpu_call_r02_36.sh
for i in 1 2; do for lib in libsimba.so libsimba_t384.so; do
  echo "== $lib"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_variance.py 30; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_shapes.py 0:0
done; done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv

# ---- gpu_call_r02_37.sh
for i in 1 2; do for lib in libsimba.so libsimba_dpw16.so libsimba_dpw12.so; do
  echo "== $lib"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_variance.py 30; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_shapes.py 0:0
done; done

# ---- gpu_call_r02_38.sh
timeout 1200 python -m pytest tests/test_production_paths.py tests/test_gpu_parity.py -q -x > gpurun_out/c38_tests.log 2>&1; tail -2 gpurun_out/c38_tests.log
for i in 1 2; do for cfg in "X=1" "SIMBA_DPW_RT=24" "SIMBA_DPW_RT=20"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 30; env $cfg timeout 300 python scripts/probe_shapes.py 0:0
done; done

# ---- gpu_call_r02_41.sh
for i in 1 2; do for cfg in "X=1" "SIMBA_SHARD_PG=0" "SIMBA_SHARD_PG=2" "SIMBA_SHARD_DPW=32" "SIMBA_SHARD_DPW=16" "SIMBA_SHARD_DPW=32 SIMBA_SHARD_PG=0" "SIMBA_GUIDE=8"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_shards.py 8
done; done

# ---- gpu_call_r02_42.sh
timeout 900 python -m pytest tests/test_production_paths.py -q -x 2>&1 | tail -1
for i in 1 2; do for lib in libsimba.so libsimba_gd0.so libsimba_gd1.so; do
  echo "== $lib"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_variance.py 30; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_shapes.py 0:0
done; done

# ---- gpu_call_r02_43.sh
for i in 1 2; do for cfg in "X=1" "SIMBA_DPW_RT=24 SIMBA_DPW_LATE=16" "SIMBA_DPW_RT=24 SIMBA_DPW_LATE=12" "SIMBA_DPW_RT=16 SIMBA_DPW_LATE=12" "SIMBA_DPW_RT=24 SIMBA_DPW_LATE=8"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 30
done; done

# ---- gpu_call_r02_44.sh
timeout 900 python -m pytest tests/test_production_paths.py -q -x 2>&1 | tail -1
for i in 1 2; do for cfg in "X=1" "SIMBA_DPW_LATE=16" "SIMBA_DPW_LATE=12"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_shapes.py 0:0; env $cfg timeout 300 python scripts/probe_shards.py 8
done; done

# ---- gpu_call_r02_45.sh
timeout 1200 python -m pytest tests/test_production_paths.py tests/test_gpu_parity.py tests/test_xbest.py -q -x > gpurun_out/c45_tests.log 2>&1; tail -2 gpurun_out/c45_tests.log
for i in 1 2; do for lib in libsimba.so libsimba_head.so; do
  echo "== $lib"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_variance.py 30; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_shapes.py 0:0
done; done

# ---- gpu_call_r02_46.sh
for i in 1 2; do for cfg in "X=1" "SIMBA_DPW_LATE=0" "SIMBA_DPW_LATE=12" "SIMBA_DPW_RT=16 SIMBA_DPW_LATE=0"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 30
done; done
for cfg in "X=1" "SIMBA_SHARD_PG=0" "SIMBA_SHARD_DPW=16"; do echo "== $cfg"; env $cfg timeout 300 python scripts/probe_shards.py 8; done

# ---- gpu_call_r02_47.sh
for i in 1 2; do for cfg in "X=1" "SIMBA_DPW_LATE=8" "SIMBA_DPW_LATE=10" "SIMBA_DPW_LATE=6"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 30
done; done

# ---- gpu_call_r02_48.sh
for i in 1 2; do for cfg in "X=1" "SIMBA_DPW_LATE=12" "SIMBA_DPW_LATE=16"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_shapes.py 0:0; env $cfg timeout 300 python scripts/probe_shards.py 8
done; done

# ---- gpu_call_r02_49.sh
for i in 1 2; do for lib in libsimba.so libsimba_desc17.so libsimba_split16.so; do
  echo "== $lib"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_variance.py 30; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_shapes.py 0:0
done; done

# ---- gpu_call_r02_50.sh
for i in 1 2; do for lib in libsimba.so libsimba_desc19.so; do
  echo "== $lib"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_variance.py 30; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_shapes.py 0:0
done; done

# ---- gpu_call_r02_51.sh
timeout 900 python -m pytest tests/test_production_paths.py -q -x 2>&1 | tail -1
for i in 1 2; do for lib in libsimba.so libsimba_fd0.so libsimba_fd2.so; do
  echo "== $lib"; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_variance.py 30; SIMBA_LIB=$PWD/paper_2605_08243_b200/_lib/$lib timeout 300 python scripts/probe_shapes.py 0:0
done; done

# ---- gpu_call_r02_52.sh
for i in 1 2; do for cfg in "X=1" "SIMBA_GUIDE=1" "SIMBA_GUIDE=3" "SIMBA_GUIDE=4" "SIMBA_DPW_LATE=16"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 30
done; done

# ---- gpu_call_r02_54.sh
timeout 600 python scripts/probe_shapes.py 0:0
for i in 1 2; do for cfg in "SIMBA_FUSED_SHARDS=0" "SIMBA_FUSED_SHARDS=1"; do for N in 2 4; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_shards.py $N
done; done; done

# ---- gpu_call_r02_55.sh
for i in 1 2; do
for cfg in "SIMBA_FUSED_SHARDS=1" "SIMBA_FUSED_SHARDS=1 SIMBA_BIG_LAUNCH=20000000000"; do echo "== $cfg N4"; env $cfg timeout 300 python scripts/probe_shards.py 4; done
for cfg in "SIMBA_FUSED_SHARDS=1" "SIMBA_FUSED_SHARDS=1 SIMBA_BIG_LAUNCH=10000000000"; do echo "== $cfg N8"; env $cfg timeout 300 python scripts/probe_shards.py 8; done
done

# ---- gpu_call_r02_57.sh
timeout 1500 python -m pytest tests/test_production_paths.py tests/test_gpu_parity.py tests/test_xbest.py -q -x > gpurun_out/c57_tests.log 2>&1; tail -2 gpurun_out/c57_tests.log
for i in 1 2; do for cfg in "SIMBA_SHARED_CAP=1" "SIMBA_SHARED_CAP=0"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 30; env $cfg timeout 300 python scripts/probe_shapes.py 0:0
done; done

# ---- gpu_call_r02_58.sh
for i in 1 2; do for cfg in "SIMBA_SHARED_CAP=1" "SIMBA_SHARED_CAP=0"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_shapes.py 0:0; env $cfg timeout 300 python scripts/probe_shards.py 2
done; done

# ---- gpu_call_r02_59.sh
for i in 1 2; do for cfg in "X=1" "SIMBA_DPW_LATE=8" "SIMBA_DPW_LATE=16" "SIMBA_DPW_LATE=24"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 30
done; done

# ---- gpu_call_r02_60.sh
for i in 1 2; do for cfg in "X=1" "SIMBA_R0_UP=11" "SIMBA_R0_UP=13" "SIMBA_GUIDE=3" "SIMBA_SPLIT_MIN=524288"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_variance.py 30
done; done

# ---- gpu_call_r02_61.sh
for i in 1 2; do for cfg in "X=1" "SIMBA_SPLIT_MIN=524288" "SIMBA_SPLIT_MIN=262144"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_shapes.py 0:0; env $cfg timeout 300 python scripts/probe_shards.py 2; env $cfg timeout 300 python scripts/probe_variance.py 20
done; done

# ---- gpu_call_r02_62.sh
for cfg in "X=1" "SIMBA_SPLIT_MIN=131072" "SIMBA_SHARED_CAP=0" "SIMBA_EX0_DENSE=1e9"; do echo "== $cfg"; env $cfg timeout 300 python scripts/probe_tts.py s12_k4_i08 s11_k4_i14 s11_k4_i10 s12_k4_i37; done

# ---- gpu_call_r02_63.sh
for cfg in "X=1" "SIMBA_L2_PERSIST=0"; do echo "== $cfg"; env $cfg timeout 300 python scripts/probe_tts.py s12_k4_i08 s11_k4_i10; done

# ---- gpu_call_r02_64.sh
# TTS outliers: full bench process (after the sweep + e2e) vs eager module loading
for i in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/c64_b$i.log 2>&1; done
CUDA_MODULE_LOADING=EAGER timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/c64_eager.log 2>&1
timeout 600 python scripts/probe_tts.py > gpurun_out/c64_probe.log 2>&1

# ---- gpu_call_r02_65.sh
# context-creation phase times (SIMBA_TRACE_CTX=1)
SIMBA_TRACE_CTX=1 timeout 300 python scripts/probe_tts.py s11_k4_i10 s12_k4_i08 s12_k4_i09 s13_k4_i03 > gpurun_out/c65.log 2>&1

# ---- gpu_call_r02_66.sh
# in-place adaptive E: parity + context-creation phases + TTS
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c66_gpu.log 2>&1
SIMBA_TRACE_CTX=1 timeout 300 python scripts/probe_tts.py s11_k4_i10 s12_k4_i08 s12_k4_i09 s13_k4_i03 > gpurun_out/c66_trace.log 2>&1
timeout 300 python scripts/probe_tts.py > gpurun_out/c66_probe.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/c66_bench.log 2>&1

# ---- gpu_call_r02_67.sh
# pooled streams: parity + context-creation phases + TTS (x2 bench processes)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c67_gpu.log 2>&1
SIMBA_TRACE_CTX=1 timeout 300 python scripts/probe_tts.py s11_k4_i10 s12_k4_i08 s12_k4_i09 s13_k4_i03 s13_k4_i04 > gpurun_out/c67_trace.log 2>&1
timeout 300 python scripts/probe_tts.py > gpurun_out/c67_probe.log 2>&1
for i in 1 2 3; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/c67_bench$i.log 2>&1; done

# ---- gpu_call_r02_68.sh
timeout 300 python scripts/probe_launch_lat.py s11_k4_i10 s11_k4_i02 s12_k4_i09 > gpurun_out/c68.log 2>&1

# ---- gpu_call_r02_69.sh
SIMBA_LIB=build/libsimba_cta.so timeout 300 python scripts/probe_small_launch.py 1..9 10..10 11..11 > gpurun_out/c69.log 2>&1

# ---- gpu_call_r02_70.sh
SIMBA_LIB=build/libsimba_stats.so timeout 300 python scripts/probe_small_stats.py 1..9 9..9 10..10 11..11 12..12 > gpurun_out/c70.log 2>&1

# ---- gpu_call_r02_71.sh
# synthesize level fusion: 2^26 (levels 1..9 | 10 | 11 | 12 | 13) vs 2^31 (1..11 | 12 | 13) vs 2^34 (1..12 | 13)
for f in 67108864 2147483648 17179869184 67108864 2147483648 17179869184; do
  echo "== SIMBA_FUSE_CANDS=$f"; SIMBA_FUSE_CANDS=$f timeout 300 python scripts/probe_tts.py
done > gpurun_out/c71.log 2>&1

# ---- gpu_call_r02_72.sh
# level-guided fused searches: fusion threshold x guidance (probe_tts: best of 3 per target after the first)
for f in 67108864 2147483648 17179869184 1099511627776; do for g in 0 1; do
  echo "== SIMBA_FUSE_CANDS=$f SIMBA_LEVEL_GUIDE=$g"; SIMBA_FUSE_CANDS=$f SIMBA_LEVEL_GUIDE=$g timeout 300 python scripts/probe_tts.py
done; done > gpurun_out/c72.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c72_gpu.log 2>&1

# ---- gpu_call_r02_73.sh
# level-guided fused searches (fixed build): fusion threshold x guidance
for f in 2147483648 17179869184 1099511627776; do for g in 0 1; do
  echo "== SIMBA_FUSE_CANDS=$f SIMBA_LEVEL_GUIDE=$g"; SIMBA_FUSE_CANDS=$f SIMBA_LEVEL_GUIDE=$g timeout 300 python scripts/probe_tts.py
done; done > gpurun_out/c73.log 2>&1
SIMBA_FUSE_CANDS=1099511627776 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c73_gpu.log 2>&1

# ---- gpu_call_r02_74.sh
# all levels fused: which part of the level guidance costs at size 13
for g in 0 7 1 3 5 6; do
  echo "== SIMBA_FUSE_CANDS=2^40 SIMBA_LEVEL_GUIDE=$g"; SIMBA_FUSE_CANDS=1099511627776 SIMBA_LEVEL_GUIDE=$g timeout 300 python scripts/probe_tts.py
done > gpurun_out/c74.log 2>&1

# ---- gpu_call_r02_75.sh
# tiles above a recorded hit skipped at execution; fusion x level guidance again
for cfg in "67108864 0" "2147483648 0" "17179869184 0" "1099511627776 0" "1099511627776 1" "1099511627776 5"; do set -- $cfg
  echo "== SIMBA_FUSE_CANDS=$1 SIMBA_LEVEL_GUIDE=$2"; SIMBA_FUSE_CANDS=$1 SIMBA_LEVEL_GUIDE=$2 timeout 300 python scripts/probe_tts.py
done > gpurun_out/c75.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c75_gpu.log 2>&1

# ---- gpu_call_r02_76.sh
# all levels fused + level-guided claims: claim guide and descriptors per warp
export SIMBA_FUSE_CANDS=1099511627776 SIMBA_LEVEL_GUIDE=1
for cfg in "X=1" "SIMBA_GUIDE=4" "SIMBA_GUIDE=8" "SIMBA_DPW_RT=12" "SIMBA_DPW_RT=8" "SIMBA_LEVEL_GUIDE=5" "SIMBA_GUIDE=4 SIMBA_DPW_RT=12"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/probe_tts.py
done > gpurun_out/c76.log 2>&1

# ---- gpu_call_r02_77.sh
# new synthesize defaults (all levels fused, level-guided, search dpw 12, exec skip): parity, TTS, bench, configs
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c77_gpu.log 2>&1
timeout 300 python scripts/probe_tts.py > gpurun_out/c77_probe.log 2>&1
for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/c77_bench$i.log 2>&1; done
timeout 900 python scripts/configs.py > gpurun_out/c77_configs.json 2> /dev/null

# ---- gpu_call_r02_78.sh
# ncu of a level-12 launch and of 1/8 shard of the sweep (where small launches lose rate)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:unit_kernel -c 1 -o gpurun_out/l12 python scripts/probe_once.py 12 12 > gpurun_out/l12_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:unit_kernel -c 1 -o gpurun_out/sh8 python scripts/probe_once.py 1 13 1 8 > gpurun_out/sh8_ncu.log 2>&1
