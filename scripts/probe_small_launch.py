"""CTA timelines of small launches (libsimba built with -DSIMBA_CTA_TIMES;
SIMBA_LIB points at it): levels lo..hi of the C5 unsat spec, count mode."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2605_08243_b200 as S  # noqa: E402
from paper_2605_08243_b200.engine import DeviceContext  # noqa: E402

spec = S.Specification(k=4, w=32, pairs=bench.unsat_pairs())
with DeviceContext(spec, 13) as ctx:
    for arg in sys.argv[1:]:
        lo, hi = map(int, arg.split(".."))
        ctx.run_levels(lo, hi)
        print(f"=== levels {lo}..{hi}", flush=True)
        r, _ = ctx.run_levels(lo, hi)
        print(f"KERNEL_MS {r.kernel_ms} units {r.units}", flush=True)
