#!/bin/bash
# configs.py summary per libsimba variant: scripts/configs_ab.sh name ...
for v in "$@"; do
  SIMBA_LIB=paper_2605_08243_b200/_lib/libsimba_$v.so timeout 900 python scripts/configs.py > gpurun_out/configs_$v.json 2> gpurun_out/configs_$v.err
  python3 - "$v" <<'PY'
import json, sys
v = sys.argv[1]
d = json.load(open(f"gpurun_out/configs_{v}.json"))
out = [v]
for k in ("C1", "C2", "C3", "C4"):
    out.append(f"{k} {d[k]['all_match_reference']} med {d[k]['time_to_solve_ms']['median']:.3f} max {d[k]['time_to_solve_ms']['max']:.2f}")
for k in ("count_C3_unsat777", "count_C4_stress_i0", "count_dense_k3_w64_stress"):
    out.append(f"{k} {d[k]['cand_per_s']:.3g}")
out.append("tts " + str([t["ms"] for t in d["C5_time_to_solve"]]))
print(" | ".join(out))
PY
done
