#!/bin/bash
# Copy the final-validation outputs (scripts/gpu_final.sh, in gpurun_out/) into profiles/:
# the ncu summary of the bench launch tagged with this build's source hash, the launch
# list, the bench lines, the configs report and the GPU test log.
set -e
cd "$(dirname "$0")/.."
python scripts/ncu_summary.py gpurun_out/fin_unit.ncu-rep /tmp/fin.json "r02 final build: bench-step fused launch (C5 sizes 1..13), unit_kernel<u32,1>" 111946005116 > /dev/null
python - <<'PY'
import json, bench
d = json.load(open('/tmp/fin.json'))
d['report'] = 'gpurun_out/fin_unit.ncu-rep (scratch; this is its summary)'
d['libsimba_sha16'] = bench.lib_sha16()
for f in ('profiles/ncu_unit_kernel.json', 'profiles/r02_ncu_unit_kernel_final_build.json'):
    json.dump(d, open(f, 'w'), indent=1)
m = d['metrics']
print(d['libsimba_sha16'], d['dram_bytes_per_launch'], {k: m[k][0] for k in m if any(s in k for s in ['time', 'inst_executed.sum', 'issue_active', 'pipe_alu'])})
print(d['stall_share'])
PY
python scripts/launch_summary.py gpurun_out/fin_launches.csv profiles/r02_launches_bench.json "ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 2 --warmup 1 --no-cpu --no-tts --e2e-steps 1" | tail -6
cp gpurun_out/fin_bench.log profiles/r02_bench_final.log
cp gpurun_out/fin_bench2.log profiles/r02_bench_2rank_gloo_1gpu.log
cp gpurun_out/fin_bench8.log profiles/r02_bench_8rank_gloo_1gpu.log
cp gpurun_out/fin_configs.json profiles/r02_configs_c1_c5_rtid.json
cp gpurun_out/fin_gpu.log profiles/r02_gpu_tests_final.log
python - <<'PY'
import json
for f in ['profiles/r02_bench_final.log', 'profiles/r02_bench_2rank_gloo_1gpu.log', 'profiles/r02_bench_8rank_gloo_1gpu.log']:
    l = [x for x in open(f) if x.startswith('{')][-1]
    d = json.loads(l)
    t = d['time_to_solve']
    hw = d['roofline']['hw']
    print(f, f"{d['value']:.4g}", round(d['ms_per_step'], 2), f"{d['e2e']['value']:.4g}", round(hw['test_op_frac'], 3),
          round(hw['issue_frac'] or 0, 3), hw['profile_matches_build'], d['clocks'],
          {k: (v['median_ms'], v['max_ms']) for k, v in t['by_size'].items()})
PY
