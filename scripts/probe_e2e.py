"""Where the end-to-end step time goes (diagnostics): context creation,
per-size scans (device vs wall), close."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
import paper_2605_08243_b200 as S
from paper_2605_08243_b200 import parallel
from paper_2605_08243_b200.engine import DeviceContext

spec = S.Specification(k=4, w=32, pairs=bench.unsat_pairs())
table = S.build(4, 13)
totals = [table.total(s) for s in range(1, 14)]
for it in range(4):
    t0 = time.perf_counter()
    ctx = DeviceContext(spec, 13)
    t1 = time.perf_counter()
    scan = parallel.device_scan(ctx)
    per = []
    for s, t in enumerate(totals, start=1):
        a = time.perf_counter()
        r = scan(s, 0, t, "count", 0, 1, 0)
        per.append((s, round((time.perf_counter() - a) * 1e3, 3), round(r.kernel_ms, 3)))
    t2 = time.perf_counter()
    ctx.close()
    t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.2f} ms  scans {1e3*(t2-t1):.2f} ms  close {1e3*(t3-t2):.2f} ms", flush=True)
    if it == 3:
        print(per)
