"""One launch of levels lo..hi of the C5 unsat spec (optionally shard i of N),
count mode, for ncu captures.  usage: probe_once.py lo hi [shard nshards]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2605_08243_b200 as S  # noqa: E402
from paper_2605_08243_b200.engine import DeviceContext  # noqa: E402

lo, hi = int(sys.argv[1]), int(sys.argv[2])
kw = {"shard": int(sys.argv[3]), "nshards": int(sys.argv[4])} if len(sys.argv) > 4 else {}
spec = S.Specification(k=4, w=32, pairs=bench.unsat_pairs())
with DeviceContext(spec, 13) as ctx:
    r, lv = ctx.run_levels(lo, hi, "count", **kw)
    print(f"levels {lo}..{hi} {kw}: {r.kernel_ms:.3f} ms, {sum(v for *_, v in lv)} candidates, units {r.units}", flush=True)
