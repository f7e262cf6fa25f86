"""Level-guided fused searches without hits (the C5 unsat spec) against
unguided fused counts and single-level launches: what the guidance costs on
the levels below a size-13 answer.  Diagnostics."""
import statistics
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2605_08243_b200 as S  # noqa: E402
from paper_2605_08243_b200.engine import DeviceContext  # noqa: E402

spec = S.Specification(k=4, w=32, pairs=bench.unsat_pairs())
with DeviceContext(spec, 13) as ctx:
    ctx.run_levels(1, 12, mode="count")
    for lo, hi in [(1, 11), (1, 12), (12, 12), (11, 12), (1, 13)]:
        row = []
        for mode in ("count", "search"):
            ms = [ctx.run_levels(lo, hi, mode=mode)[0].kernel_ms for _ in range(5)]
            row.append(f"{mode} {statistics.median(ms):7.3f} ms")
        print(f"levels {lo:2d}..{hi:2d}: " + " | ".join(row), flush=True)
