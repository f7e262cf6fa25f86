"""CTA timelines (library built with -DSIMBA_CTA_TIMES) of the fused sweep
levels 1..13 as a count and as a level-guided search without hits."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2605_08243_b200 as S  # noqa: E402
from paper_2605_08243_b200.engine import DeviceContext  # noqa: E402

spec = S.Specification(k=4, w=32, pairs=bench.unsat_pairs())
with DeviceContext(spec, 13) as ctx:
    for mode in ("count", "search", "count", "search"):
        print(f"=== {mode}", flush=True)
        r, _ = ctx.run_levels(1, 13, mode=mode)
        print(f"KERNEL_MS {r.kernel_ms} units {r.units}", flush=True)
