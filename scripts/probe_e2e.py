"""Where the end-to-end step time goes (diagnostics): context creation
(table upload, value tables, example-0 density, L2 window), the fused sweep
(device vs wall), close.  Env knobs (SIMBA_L2_PERSIST, SIMBA_EX0_DENSE) apply."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2605_08243_b200 as S  # noqa: E402
from paper_2605_08243_b200 import parallel  # noqa: E402
from paper_2605_08243_b200.engine import DeviceContext  # noqa: E402

spec = S.Specification(k=4, w=32, pairs=bench.unsat_pairs())
for it in range(6):
    t0 = time.perf_counter()
    ctx = DeviceContext(spec, 13)
    t1 = time.perf_counter()
    r, _ = ctx.run_levels(1, 13, "count")
    t2 = time.perf_counter()
    ctx.close()
    t3 = time.perf_counter()
    print(f"create {1e3 * (t1 - t0):.2f} ms  sweep {1e3 * (t2 - t1):.2f} ms (device {r.kernel_ms:.2f})  "
          f"close {1e3 * (t3 - t2):.2f} ms", flush=True)
