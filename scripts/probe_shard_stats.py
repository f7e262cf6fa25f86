"""Path / phase statistics (libsimba built with -DSIMBA_STATS) of the fused C5
sweep against one 8-way shard of it: where a shard launch loses rate.  Diagnostics."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
import paper_2605_08243_b200 as S
from paper_2605_08243_b200.engine import DeviceContext

spec = S.Specification(k=4, w=32, pairs=bench.unsat_pairs())
for label, kw in (("full", {}), ("shard 1/8", {"shard": 1, "nshards": 8}), ("shard 7/8", {"shard": 7, "nshards": 8})):
    with DeviceContext(spec, 13) as ctx:
        ctx.run_levels(1, 13, **kw)
        a = ctx.path_stats()
        r = ctx.run_levels(1, 13, **kw)[0]
        b = ctx.path_stats()
    d = {k: (b[k][0] - a[k][0], b[k][1] - a[k][1]) for k in b}
    print(f"== {label}: {r.kernel_ms:.3f} ms visited {r.visited:.3e} units {r.units}")
    for k, v in d.items():
        if v[0] or v[1]:
            print(f"   {k:14s} {v[0]:>14d} {v[1]:>18d}")
