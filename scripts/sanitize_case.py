"""Hit-dense production-path case for compute-sanitizer runs:
k=2 w=3 (about one example-0 hit in 8 candidates) or k=4 w=32 x0+x1, count and
search, with the big-launch shapes, R0 + 1 from level 8, partial-row R0
planning and late splitting forced on a launch small enough for the
sanitizers; results checked against the CPU oracle.

usage: SIMBA_BIG_LAUNCH=1 SIMBA_R0_UP=8 SIMBA_SPLIT_MIN=4096 \
       compute-sanitizer --tool racecheck python scripts/sanitize_case.py [k2|k4]"""
import random
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import oracle as O  # noqa: E402
import paper_2605_08243_b200 as S  # noqa: E402
from paper_2605_08243_b200.engine import DeviceContext  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "k2"
if case == "adapt":
    # a dense example 0 (all inputs equal) in a search of >= 2^30 candidates:
    # example 0's table and density, the per-example table added in place, the
    # examples reordered (64-bit words), then level-guided searches, one launch
    # and 3 shards, against the oracle's answer
    from paper_2605_08243_b200 import codec, expr
    rng = random.Random(2001)  # minimal answer at size 7
    e = codec.sample_uniform(7, S.build(3, 7), rng)
    v = rng.getrandbits(64) | (1 << 63)
    xs = [(v, v, v)]
    while len(xs) < 3:
        x = tuple(rng.getrandbits(64) for _ in range(3))
        if x not in xs:
            xs.append(x)
    pairs = [(x, expr.evaluate(e, x, 64)) for x in xs]
    tab = O.OracleTable(3, 9)
    first = None
    for s in range(1, 10):
        _, _, fr, _ = O.scan_range(tab, 3, 64, pairs, s, 0, tab.total(s), 0, tab.total(s), threads=O.cpu_count())
        if fr is not None:
            first = (s, fr)
            break
    with DeviceContext(S.Specification(k=3, w=64, pairs=tuple(pairs)), 12) as ctx:
        print("ctx", ctx.info(), flush=True)
        assert ctx.info()["table_examples"] == 2
        r, _ = ctx.run_levels(1, 12, mode="search")
        assert (r.size, r.best_rank) == first, (r, first)
        best = min((x.size, x.best_rank) for x in (ctx.run_levels(1, 12, mode="search", shard=i, nshards=3)[0]
                                                 for i in range(3)) if x.best_rank is not None)
        assert best == first, (best, first)
    print(f"sanitize case ok: adaptive tables, answer {first}", flush=True)
    sys.exit(0)
if case == "k2":  # k=2 w=3 n=4, sizes 1..10 (8.2e6 candidates); rg=8 makes R0 + 1 = 8 available
    k, w, n, size, rg, f = 2, 3, 4, 10, 8, (lambda x: x[0] * x[1] + x[0])
else:  # k=4 w=32 n=10, target x0 + x1, sizes 1..9 (2e7 candidates); R0 + 1 = 7 = RG
    k, w, n, size, rg, f = 4, 32, 10, 9, 0, (lambda x: x[0] + x[1])
rng = random.Random(4242)
pairs, seen = [], set()
while len(pairs) < n:
    x = tuple(rng.getrandbits(w) for _ in range(k))
    if x not in seen:
        seen.add(x)
        pairs.append((x, f(x) & ((1 << w) - 1)))
tab = O.OracleTable(k, size)
want = []
for s in range(1, size + 1):
    _, c, fr, _ = O.scan_range(tab, k, w, pairs, s, 0, tab.total(s), 0, tab.total(s), threads=O.cpu_count())
    want.append((s, c, fr, tab.total(s)))
with DeviceContext(S.Specification(k=k, w=w, pairs=tuple(pairs)), size, rg=rg) as ctx:
    print("ctx", ctx.info(), flush=True)
    _, lv = ctx.run_levels(1, size, mode="count")
    assert [tuple(x) for x in lv] == want, (lv, want)
    r, _ = ctx.run_levels(1, size, mode="search")
    first = next((s, f) for s, c, f, _ in want if c)
    assert (r.size, r.best_rank) == first, (r, first)
    for i in range(3):
        ctx.run_levels(1, size, mode="count", shard=i, nshards=3)
print(f"sanitize case ok: sizes 1..{size}, {sum(c for _, c, _, _ in want)} satisfying candidates", flush=True)
