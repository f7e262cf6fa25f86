#!/bin/bash
# fused C5 sweep (bench step) device time per libsimba variant, 3 interleaved rounds
for r in 1 2 3; do for v in "$@"; do
  echo -n "$v r$r: "
  SIMBA_LIB=paper_2605_08243_b200/_lib/libsimba_$v.so timeout 120 python -c "
import sys; sys.path.insert(0, '.')
import bench, paper_2605_08243_b200 as S
from paper_2605_08243_b200.engine import DeviceContext
spec = S.Specification(k=4, w=32, pairs=bench.unsat_pairs())
with DeviceContext(spec, 13) as ctx:
    for _ in range(3): ctx.run_levels(1, 13)
    ms = sorted(ctx.run_levels(1, 13)[0].kernel_ms for _ in range(5))
    print(f'min {ms[0]:.3f} med {ms[2]:.3f}')
"
done; done
