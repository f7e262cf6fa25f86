"""Per-shard device time of the C5 size-13 count split over N shards on one
GPU (load balance of the multi-GPU partition; diagnostics)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
import paper_2605_08243_b200 as S
from paper_2605_08243_b200.engine import DeviceContext

spec = S.Specification(k=4, w=32, pairs=bench.unsat_pairs())
T = S.build(4, 13).total(13)
with DeviceContext(spec, 13) as ctx:
    ctx.count(13)
    for N in (2, 4, 8):
        ms = [ctx.run(13, 0, T, mode="count", shard=i, nshards=N).kernel_ms for i in range(N)]
        vis = [ctx.run(13, 0, T, mode="count", shard=i, nshards=N).visited for i in range(N)]
        print(f"N={N} shard ms {[round(m, 2) for m in ms]} max/mean {max(ms) / (sum(ms) / N):.3f} "
              f"ideal speedup {sum(ms) / max(ms):.2f} visited ok {sum(vis) == T}", flush=True)
    # contiguous eighths (no round robin) and the full level for comparison
    full = ctx.count(13).kernel_ms
    parts = [ctx.count(13, i * T // 8, (i + 1) * T // 8).kernel_ms for i in range(8)]
    print(f"full {full:.2f} ms; contiguous eighths {[round(m, 2) for m in parts]} sum {sum(parts):.2f}", flush=True)
    parts = [ctx.count(12, i * S.build(4, 13).total(12) // 8, (i + 1) * S.build(4, 13).total(12) // 8).kernel_ms
             for i in range(8)]
    print(f"size 12 full {ctx.count(12).kernel_ms:.2f} ms; contiguous eighths sum {sum(parts):.2f}", flush=True)
