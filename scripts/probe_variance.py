"""Launch-to-launch spread of the bench step (fused C5 sweep, one context,
N launches): sorted device times.  Env knobs apply (SIMBA_SPLIT_MIN, ...)."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2605_08243_b200 as S  # noqa: E402
from paper_2605_08243_b200.engine import DeviceContext  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
spec = S.Specification(k=4, w=32, pairs=bench.unsat_pairs())
with DeviceContext(spec, 13) as ctx:
    for _ in range(3):
        ctx.run_levels(1, 13)
    ms = sorted(ctx.run_levels(1, 13)[0].kernel_ms for _ in range(n))
print(f"n={n} min {ms[0]:.2f} median {statistics.median(ms):.2f} mean {statistics.mean(ms):.2f} "
      f"max {ms[-1]:.2f} ms; deciles {[round(ms[int(i * (n - 1) / 10)], 2) for i in range(11)]}", flush=True)
