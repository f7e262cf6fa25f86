"""One fused C5 sweep launch (levels 1..13) for ncu captures."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
import paper_2605_08243_b200 as S
from paper_2605_08243_b200.engine import DeviceContext

spec = S.Specification(k=4, w=32, pairs=bench.unsat_pairs())
with DeviceContext(spec, 13) as ctx:
    r, lv = ctx.run_levels(1, 13, "count")
    print(f"fused sweep {r.kernel_ms:.2f} ms, {sum(v for *_, v in lv)} candidates", flush=True)
