"""Fused C5 sweep device time vs the late-splitting threshold (SIMBA_SPLIT_MIN is
read at context creation), interleaved rounds, plus the 8-way shard max.  Diagnostics."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
import paper_2605_08243_b200 as S
from paper_2605_08243_b200.engine import DeviceContext

spec = S.Specification(k=4, w=32, pairs=bench.unsat_pairs())
vals = [1 << 16, 1 << 17, 1 << 18, 1 << 19, 1 << 20, 1 << 22]
res = {v: [] for v in vals}
sh = {v: [] for v in vals}
for rnd in range(3):
    for v in vals:
        os.environ["SIMBA_SPLIT_MIN"] = str(v)
        with DeviceContext(spec, 13) as ctx:
            for _ in range(2):
                ctx.run_levels(1, 13)
            res[v].append(min(ctx.run_levels(1, 13)[0].kernel_ms for _ in range(3)))
            if rnd == 0:
                sh[v] = max(ctx.run_levels(1, 13, shard=i, nshards=8)[0].kernel_ms for i in range(8))
for v in vals:
    print(f"split_min 2^{v.bit_length() - 1}: sweep {[round(x, 3) for x in res[v]]} 8-shard max {sh[v]:.3f}", flush=True)
