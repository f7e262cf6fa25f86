"""Per-launch device time of small searches (time-to-solve diagnostics):
synthesize's launch groups run alone in count and search mode, per target."""
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2605_08243_b200 as S  # noqa: E402
from paper_2605_08243_b200.engine import DeviceContext  # noqa: E402

ids = set(sys.argv[1:]) or {"s11_k4_i10", "s12_k4_i09"}
unsat = S.Specification(k=4, w=32, pairs=bench.unsat_pairs())
targets = [("unsat", unsat)] + [(rec["id"], spec) for _, spec, rec in bench.c5_targets(S) if rec["id"] in ids]
groups = [(1, 1), (1, 9), (10, 10), (11, 11), (12, 12)]
for name, spec in targets:
    with DeviceContext(spec, 13) as ctx:
        ctx.run_levels(1, 9, mode="count")
        for lo, hi in groups:
            row = []
            for mode in ("count", "search"):
                ms = []
                for _ in range(5):
                    r, lv = ctx.run_levels(lo, hi, mode=mode)
                    ms.append(r.kernel_ms)
                vis = sum(v for *_, v in lv)
                row.append(f"{mode} {statistics.median(ms) * 1e3:8.1f} us vis {vis:.3e} "
                           f"({vis / (statistics.median(ms) * 1e-3) / 1e12:.2f}e12/s)")
            print(f"{name:12s} levels {lo:2d}..{hi:2d}: " + " | ".join(row), flush=True)
