#!/bin/bash
# 8-way shard device times of the fused sweep per libsimba variant (and SIMBA_R0_UP=13 forced on the base)
for v in "$@"; do echo "== $v"; SIMBA_LIB=paper_2605_08243_b200/_lib/libsimba_$v.so timeout 120 python -c "
import sys; sys.path.insert(0, '.')
import bench, paper_2605_08243_b200 as S
from paper_2605_08243_b200.engine import DeviceContext
spec = S.Specification(k=4, w=32, pairs=bench.unsat_pairs())
with DeviceContext(spec, 13) as ctx:
    for _ in range(2): ctx.run_levels(1, 13)
    full = min(ctx.run_levels(1, 13)[0].kernel_ms for _ in range(3))
    ms = [min(ctx.run_levels(1, 13, shard=i, nshards=8)[0].kernel_ms for _ in range(2)) for i in range(8)]
    print(f'full {full:.3f} N=8 max {max(ms):.3f} mean {sum(ms)/8:.3f} ceiling {full/max(ms):.2f}', [round(m,2) for m in ms])
"; done
