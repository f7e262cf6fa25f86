"""Sharded searches of consecutive time-to-solve targets in one process (each
shard launched in turn, optionally with one shared minimum reset between
targets), against the oracle answers: the multi-rank protocol without the
processes.  usage: probe_shard_seq.py N [xbest]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2605_08243_b200 as S  # noqa: E402
from paper_2605_08243_b200.engine import DeviceContext, SharedMinimum  # noqa: E402

N = int(sys.argv[1])
use_x = len(sys.argv) > 2
shared = SharedMinimum(0) if use_x else None
bad = 0
for target, spec, rec in bench.c5_targets(S):
    if shared:
        shared.reset()
    best = None
    with DeviceContext(spec, 13) as ctx:
        info = ctx.info()
        if shared:
            ctx.set_shared_minimum(shared)
        for i in range(N):
            r, _ = ctx.run_levels(1, 13, mode="search", shard=i, nshards=N)
            if r.best_rank is not None and (best is None or (r.size, r.best_rank) < best):
                best = (r.size, r.best_rank)
        if shared:
            ctx.set_shared_minimum(None)
    want = (rec["oracle"]["size"], rec["oracle"]["rank"])
    ok = best == want
    bad += not ok
    print(rec["id"], "E", info["table_examples"], "ok" if ok else f"WRONG {best} != {want}", flush=True)
print("wrong:", bad)
