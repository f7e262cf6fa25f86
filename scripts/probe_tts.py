"""Time-to-solve suite, each target several times: wall ms, device ms and
launches of simba_synthesize (diagnostics for outliers)."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2605_08243_b200 as S  # noqa: E402
from paper_2605_08243_b200.engine import DeviceContext  # noqa: E402

ids = set(sys.argv[1:])
S.synthesize(S.Specification(k=4, w=32, pairs=bench.unsat_pairs()), S.build(4, 5), S.EngineConfig(size_bound=5))
for target, spec, rec in bench.c5_targets(S):
    if ids and rec["id"] not in ids:
        continue
    row = []
    for _ in range(3):
        t0 = time.perf_counter()
        with DeviceContext(spec, 13) as ctx:
            t1 = time.perf_counter()
            o = ctx.synthesize_raw(13)
        t2 = time.perf_counter()
        row.append(f"{(t2 - t0) * 1e3:.2f}ms(ctx {(t1 - t0) * 1e3:.2f}, dev {o.kernel_ms:.2f}, {o.launches} launches, "
                   f"size {o.size} rank {o.rank})")
    print(rec["id"], " | ".join(row), flush=True)
