"""Path / phase statistics (libsimba built with -DSIMBA_STATS) of small
launches (levels lo..hi of the C5 unsat spec): where small levels lose rate."""
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
        a = ctx.path_stats()
        r = ctx.run_levels(lo, hi)[0]
        b = ctx.path_stats()
        d = {k: (b[k][0] - a[k][0], b[k][1] - a[k][1]) for k in b}
        print(f"== levels {lo}..{hi}: {r.kernel_ms:.3f} ms visited {r.visited:.3e} units {r.units}")
        for k, v in d.items():
            if v[0] or v[1]:
                print(f"   {k:14s} {v[0]:>14d} {v[1]:>18d}")
