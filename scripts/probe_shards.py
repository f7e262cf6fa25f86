"""8-way shards of the fused C5 sweep, each timed alone on one GPU (the
multi-GPU partition's slowest shard), min of 3 per shard.  Env knobs apply."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2605_08243_b200 as S  # noqa: E402
from paper_2605_08243_b200.engine import DeviceContext  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
spec = S.Specification(k=4, w=32, pairs=bench.unsat_pairs())
with DeviceContext(spec, 13) as ctx:
    ctx.run_levels(1, 13)
    ms = [min(ctx.run_levels(1, 13, shard=i, nshards=N)[0].kernel_ms for _ in range(3)) for i in range(N)]
print(f"N={N} shards ms {[round(m, 3) for m in ms]} max {max(ms):.3f} mean {sum(ms) / N:.3f}", flush=True)
