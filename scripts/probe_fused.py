"""Fused multi-level launch vs per-level launches, and its shards (diagnostics)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
import paper_2605_08243_b200 as S
from paper_2605_08243_b200.engine import DeviceContext

spec = S.Specification(k=4, w=32, pairs=bench.unsat_pairs())
tab = S.build(4, 13)
with DeviceContext(spec, 13) as ctx:
    for it in range(2):
        per = sum(ctx.count(s).kernel_ms for s in range(1, 14))
        r, lv = ctx.run_levels(1, 13, "count")
        ok = [v for *_, v in lv] == [tab.total(s) for s in range(1, 14)]
        print(f"per-level launches {per:.2f} ms; fused {r.kernel_ms:.2f} ms visited ok {ok}", flush=True)
    for N in (2, 4, 8):
        ms = [ctx.run_levels(1, 13, "count", shard=i, nshards=N)[0].kernel_ms for i in range(N)]
        print(f"fused N={N} shards {[round(m, 2) for m in ms]} max/mean {max(ms) * N / sum(ms):.3f} "
              f"speedup {r.kernel_ms / max(ms):.2f}", flush=True)
