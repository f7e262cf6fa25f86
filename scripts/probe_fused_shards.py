"""Per-shard device time of the bench step (C5 sizes 1..13 fused, count mode)
split over N shards on one GPU: the multi-GPU partition's balance and its
strong-scaling ceiling (full time / max shard time).  Diagnostics."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
import paper_2605_08243_b200 as S
from paper_2605_08243_b200.engine import DeviceContext

spec = S.Specification(k=4, w=32, pairs=bench.unsat_pairs())
with DeviceContext(spec, 13) as ctx:
    for _ in range(2):
        ctx.run_levels(1, 13)
    full = min(ctx.run_levels(1, 13)[0].kernel_ms for _ in range(3))
    print(f"full {full:.3f} ms", flush=True)
    for N in (2, 4, 8):
        ms = [min(ctx.run_levels(1, 13, shard=i, nshards=N)[0].kernel_ms for _ in range(2)) for i in range(N)]
        print(f"N={N} shard ms {[round(m, 3) for m in ms]} max/mean {max(ms) / (sum(ms) / N):.3f} "
              f"speedup ceiling {full / max(ms):.2f} ({full / max(ms) / N:.1%})", flush=True)
