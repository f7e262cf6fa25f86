"""Full C5 sweep (sizes 1..13 fused, count mode) and its 8-way shards for
context options (rg, r0) given as arguments, e.g. `probe_shapes.py 0:0 0:8`
(r0:rg, 0 = auto).  Diagnostics for DESIGN.md 6."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
import paper_2605_08243_b200 as S
from paper_2605_08243_b200.engine import DeviceContext

spec = S.Specification(k=4, w=32, pairs=bench.unsat_pairs())
tab = S.build(4, 13)
for arg in sys.argv[1:] or ["0:0"]:
    r0, rg = (int(x) for x in arg.split(":"))
    with DeviceContext(spec, 13, r0=r0, rg=rg) as ctx:
        for _ in range(2):
            ctx.run_levels(1, 13)
        full = min(ctx.run_levels(1, 13)[0].kernel_ms for _ in range(5))
        _, lv = ctx.run_levels(1, 13)
        assert [v for *_, v in lv] == [tab.total(s) for s in range(1, 14)]
        ms = [min(ctx.run_levels(1, 13, shard=i, nshards=8)[0].kernel_ms for _ in range(2)) for i in range(8)]
        s13 = min(ctx.count(13).kernel_ms for _ in range(3))
        print(f"{ctx.info()} full {full:.3f} ms ({tab.cumulative_total(13) / full / 1e9:.3f}e12 cand/s) "
              f"size13 {s13:.3f} ms; 8 shards max {max(ms):.3f} ms -> ceiling {full / max(ms):.2f}x", flush=True)
