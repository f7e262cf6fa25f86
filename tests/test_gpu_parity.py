"""CUDA path vs the reference (golden fixtures) and the pinned CPU oracle.

Every test here calls libsimba.so through the package API / C ABI on cuda:0.
"""

import random

import pytest

import oracle as O
from conftest import load_golden

pytestmark = pytest.mark.gpu

S = pytest.importorskip("paper_2605_08243_b200")
from paper_2605_08243_b200 import _native as N  # noqa: E402
from paper_2605_08243_b200.engine import DeviceContext  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def need_device():
    if N.device_count() < 1:
        pytest.fail("no CUDA device visible: the GPU tests must run on a B200")


def spec_of(d):
    return S.Specification(k=d["k"], w=d["w"], pairs=tuple((tuple(i), o) for i, o in d["pairs"]))


def pairs_of(d):
    return [(tuple(i), o) for i, o in d["pairs"]]


# ---------------------------------------------------------------- decode


def test_decode_every_rank_small_sizes():
    for g in load_golden("decode")["digests"]:
        if g["tokens"] is None:
            continue
        t = S.build(g["k"], g["s"])
        for n, toks in enumerate(g["tokens"]):
            assert S.decode(n, g["s"], t).tokens == tuple(toks)


def test_decode_samples_large_sizes():
    tables = {}
    for smp in load_golden("decode")["samples"]:
        if smp["s"] > N.MAX_SIZE:
            continue
        k = smp["k"]
        tables.setdefault(k, S.build(k, 24 if k == 1 else 16))
        assert S.decode(smp["rank"], smp["s"], tables[k]).tokens == tuple(smp["tokens"]), smp


def test_decode_rejects_out_of_range():
    t = S.build(2, 3)
    with pytest.raises(S.RankError):
        S.decode(t.total(3), 3, t)


# ---------------------------------------------------------------- search (Alg. 1)


@pytest.mark.parametrize("config", ["C1", "C2", "C3", "C4", None])
def test_synthesize_matches_reference(config):
    cases = [r for r in load_golden("search") if r["meta"].get("config") == config]
    assert cases
    for r in cases:
        spec = spec_of(r["spec"])
        C = r["size_bound"]
        out = S.synthesize(spec, S.build(spec.k, C), S.EngineConfig(size_bound=C))
        assert out.status.value == r["status"], r["name"]
        assert out.size == r["size"] and out.rank == r["rank"], r["name"]
        assert (list(out.expr.tokens) if out.expr else None) == r["tokens"], r["name"]
        # fully swept sizes visit exactly T[s][8] (test_engine.py:145-159); the
        # hit size's count is chunk-granular in the reference and is not pinned
        full = r["per_size"] if r["status"] != "found" else r["per_size"][:-1]
        assert [[s.size, s.candidates] for s in out.stats][: len(full)] == full, r["name"]
        assert len(out.stats) == len(r["per_size"])


def test_shuffled_mode_same_outcome():
    cases = [r for r in load_golden("search") if r["meta"].get("config") in ("C1", "C2")][::3]
    for r in cases:
        spec = spec_of(r["spec"])
        C = r["size_bound"]
        out = S.synthesize(spec, S.build(spec.k, C), S.EngineConfig(size_bound=C, mode="shuffled"))
        assert (out.status.value, out.size, out.rank) == (r["status"], r["size"], r["rank"]), r["name"]


def test_min_rank_wins_within_block():
    # test_engine.py:59-77: x0 & x1 (rank 5) and x1 & x0 (rank 6) both satisfy
    r = [r for r in load_golden("search") if r["name"] == "and_k2"][0]
    spec = spec_of(r["spec"])
    for mode in ("local", "shuffled"):
        for kernel in ("unit", "direct"):
            out = S.synthesize(spec, S.build(2, 3), S.EngineConfig(size_bound=3, mode=mode, kernel=kernel))
            assert (out.size, out.rank, out.expr.tokens) == (3, 5, (0, 1, -2))


def test_identity_and_not_found_stats():
    spec = S.Specification.of([((0,), 1), ((1,), 0)], k=1)
    out = S.synthesize(spec, S.build(1, 8), S.EngineConfig(size_bound=2))
    assert out.status is S.Status.NOT_FOUND
    assert [(s.size, s.candidates) for s in out.stats] == [(1, 1), (2, 2)]
    rep = S.run_stats(out)
    assert rep["total_candidates"] == 3
    ident = S.Specification.of([((v,), v) for v in (3, 9, 12345)], k=1)
    out = S.synthesize(ident, S.build(1, 3), S.EngineConfig(size_bound=3))
    assert (out.status, out.size, out.rank, out.expr.tokens) == (S.Status.FOUND, 1, 0, (0,))
    assert S.run_stats(out)["rank"] == "0"


def test_time_budget():
    # a budget the device cannot meet: k=3 up to size 14 is ~1.1e12 candidates
    spec = S.Specification.of([((i, i + 1, i + 2), (31 * i + 7) & 0xFFFFFFFF) for i in range(16)], k=3)
    out = S.synthesize(spec, S.build(3, 14), S.EngineConfig(size_bound=14, time_budget=0.01))
    assert out.status is S.Status.TIMED_OUT and out.expr is None
    # an expired budget never masks a hit in the current block (test_engine.py:122-130)
    ident = S.Specification.of([((v,), v) for v in (3, 9)], k=1)
    for mode in ("local", "shuffled"):
        out = S.synthesize(ident, S.build(1, 2), S.EngineConfig(size_bound=2, mode=mode, time_budget=0.0))
        assert out.status is S.Status.FOUND and out.size == 1


# ---------------------------------------------------------------- exhaustive count mode


@pytest.mark.parametrize("name", [r["name"] for r in load_golden("counts")])
def test_exhaustive_counts_match_reference(name):
    r = [r for r in load_golden("counts") if r["name"] == name][0]
    spec = spec_of(r["spec"])
    C = r["size_bound"]
    got = S.count_solutions(spec, S.build(spec.k, C), S.EngineConfig(size_bound=C))
    table = S.build(spec.k, C)
    assert [[c.size, c.count, c.first_rank] for c in got] == r["per_size"]
    assert [c.candidates for c in got] == [table.total(s) for s in range(1, C + 1)]


@pytest.mark.parametrize("variant", [dict(r0=1, rg=1), dict(r0=2), dict(r0=2, rg=3), dict(r0=3, table_examples=1),
                                     dict(r0=3, rg=6), dict(table_examples=2), dict(table_examples=4),
                                     dict(kernel="direct")])
def test_counts_independent_of_kernel_configuration(variant):
    for name in ("dense_k3_w3_n2", "C4_stress_i0", "dense_k3_w64_stress", "C2_s5_i0"):
        r = [r for r in load_golden("counts") if r["name"] == name][0]
        spec = spec_of(r["spec"])
        C = min(r["size_bound"], 8)
        got = S.count_solutions(spec, S.build(spec.k, C), S.EngineConfig(size_bound=C, **variant))
        assert [[c.size, c.count, c.first_rank] for c in got] == r["per_size"][:C], (name, variant)


# ---------------------------------------------------------------- rank windows (C5 sizes 11..13)


# exercise (r0, rg) combinations other than the automatic one on some C5 windows
WINDOW_RG = {"C5_s12_t1": (5, 5), "C5dense_s13_op2": (6, 6), "C5dense_s12_op4": (4, 9), "C5_s13_t0": (6, 9),
             "C5dense_s11_op4": (3, 7)}


@pytest.mark.parametrize("name", [r["name"] for r in load_golden("windows")])
def test_windows_match_reference(name):
    r = [r for r in load_golden("windows") if r["name"] == name][0]
    spec = spec_of(r["spec"])
    r0, rg = WINDOW_RG.get(r["name"], (0, 0))
    with DeviceContext(spec, r["size_bound"], r0=r0, rg=rg) as ctx:
        c = ctx.count(r["size"], r["lo"], r["hi"])
        assert (c.count, c.best_rank) == (r["count"], r["first"])
        assert c.visited == r["hi"] - r["lo"]
        s = ctx.run(r["size"], r["lo"], r["hi"], mode="search")
        assert s.best_rank == r["first"]
        if r["first"] is not None:
            assert list(s.tokens) == list(O.decode(O.OracleTable(spec.k, r["size_bound"]), r["first"], r["size"]))
        # odd chunking and 3-way round-robin sharding give the same answer
        tot, first = 0, []
        for shard in range(3):
            p = ctx.run(r["size"], r["lo"], r["hi"], mode="count", chunk=777, shard=shard, nshards=3)
            tot += p.count
            if p.best_rank is not None:
                first.append(p.best_rank)
        assert tot == r["count"] and (min(first) if first else None) == r["first"]


def test_sharded_search_min_equals_unsharded():
    # each shard's early-exit search returns its exact minimum,
    # so the MIN over shards is the level minimum (the reference's rank)
    for r in [r for r in load_golden("windows") if r["count"] > 1][:8]:
        spec = spec_of(r["spec"])
        with DeviceContext(spec, r["size_bound"]) as ctx:
            for nsh in (2, 3, 5):
                got = [ctx.run(r["size"], r["lo"], r["hi"], mode="search", chunk=1 << 10, shard=i, nshards=nsh)
                       for i in range(nsh)]
                firsts = [g.best_rank for g in got if g.best_rank is not None]
                assert min(firsts) == r["first"], (r["name"], nsh)


def test_scan_range_seam_matches_reference_chunks():
    r = [r for r in load_golden("counts") if r["name"] == "dense_k3_w3_n2"][0]
    spec = spec_of(r["spec"])
    t = O.OracleTable(3, 9)
    rng = random.Random(5)
    with DeviceContext(spec, 9) as ctx:
        for s in (6, 7, 8):
            for op in range(8):
                cnt = t.entry(s, op)
                if not cnt:
                    continue
                off = t.operator_offset(s, op)
                for _ in range(3):
                    a = rng.randrange(cnt)
                    b = min(cnt, a + rng.randrange(1, 5000))
                    for shuffled in (False, True):
                        want = O.scan_range(t, 3, spec.w, pairs_of(r["spec"]), s, off, cnt, a, b, shuffled)
                        got = ctx.scan_range(s, off, cnt, a, b, shuffled)
                        assert got == (want[0], want[2], want[3]), (s, op, a, b, shuffled)


# ---------------------------------------------------------------- full-size properties


def test_c5_full_sweep_size11_visits_every_rank():
    rng = random.Random(31337)
    pairs = []
    seen = set()
    while len(pairs) < 10:
        x = tuple(rng.getrandbits(32) for _ in range(4))
        if x not in seen:
            seen.add(x)
            pairs.append((x, rng.getrandbits(32)))
    spec = S.Specification(k=4, w=32, pairs=tuple(pairs))
    with DeviceContext(spec, 11) as ctx:
        r = ctx.count(11)
        assert r.visited == 1_314_029_568
        # planted solution: the decoded rank's own spec always has a hit at or below it
        planted = 987_654_321
        toks = ctx.decode(planted, 11)
        tgt = S.RpnExpr(toks)
        spec2 = S.Specification(k=4, w=32, pairs=tuple((x, S.evaluate(tgt, x, 32)) for x, _ in pairs))
    with DeviceContext(spec2, 11) as ctx2:
        hit = ctx2.run(11, 0, 1_314_029_568, mode="search")
        assert hit.best_rank is not None and hit.best_rank <= planted
        assert S.check(S.RpnExpr(hit.tokens), spec2)
        # no smaller hit in the 1M ranks below it (oracle, 8 threads)
        lo = max(0, hit.best_rank - 1_000_000)
        tab = O.OracleTable(4, 11)
        _, cnt, _, _ = O.scan_range(tab, 4, 32, list(spec2.pairs), 11, 0, tab.total(11), lo, hit.best_rank,
                                    threads=O.cpu_count())
        assert cnt == 0
        full = ctx2.count(11)
        assert full.best_rank == hit.best_rank and full.count >= 1


def test_shuffled_scan_on_block_beyond_2_32():
    # RTid permutation i * 2246822507 mod block_total with block_total > 2^32
    # (128-bit product): a window of local indices, device vs oracle
    r = [r for r in load_golden("windows") if r["name"] == "C5dense_s13_op2"][0]
    spec = spec_of(r["spec"])
    t = O.OracleTable(4, 13)
    off, cnt = t.operator_offset(13, 5), t.entry(13, 5)
    assert cnt > 1 << 32
    with DeviceContext(spec, 13) as ctx:
        for a in (0, cnt // 3, cnt - 40000):
            b = min(cnt, a + 40000)
            want = O.scan_range(t, 4, spec.w, pairs_of(r["spec"]), 13, off, cnt, a, b, shuffled=True,
                                threads=O.cpu_count())
            got = ctx.scan_range(13, off, cnt, a, b, shuffled=True)
            assert got == (want[0], want[2], want[3]), a


@pytest.mark.gpu
def test_enumerate_all_and_sampling():
    """engine.enumerate_all (engine.py:279-293) visits the device decode of
    every rank in order; sample_uniform / decode / encode round trips
    (test_engine.py:162-176, test_codec.py:156-183)."""
    import random

    import oracle as O
    from paper_2605_08243_b200.codec import encode

    assert S.enumerate_all(3, S.build(2, 3)) == 32
    assert S.enumerate_all(1, S.build(5, 1)) == 5
    for k, s in ((2, 5), (3, 4), (1, 7)):
        tab, otab = S.build(k, s), O.OracleTable(k, s)
        seen = []
        assert S.enumerate_all(s, tab, lambda e: seen.append(e.tokens), batch=97) == tab.total(s)
        assert seen == [tuple(O.decode(otab, n, s)) for n in range(tab.total(s))]
    rng = random.Random(11)
    tab = S.build(5, 12)
    for s in range(1, 13):
        e = S.sample_uniform(s, tab, rng)
        assert e.size == s
        r = encode(e, tab)
        assert S.decode(r.value, s, tab) == e


@pytest.mark.gpu
@pytest.mark.parametrize("k,w,n,size", [(3, 6, 5, 7), (2, 4, 6, 8), (4, 32, 10, 6)])
def test_example0_hits_counter_is_exact(k, w, n, size):
    """The e-bar statistic's counter (candidates that match example 0, SURVEY.md
    8(d)) equals the oracle's exhaustive count of the one-example spec."""
    rng = random.Random(k * 100 + w)
    pairs, seen = [], set()
    while len(pairs) < n:
        x = tuple(rng.getrandbits(w) for _ in range(k))
        if x not in seen:
            seen.add(x)
            pairs.append((x, rng.getrandbits(w)))
    spec = S.Specification(k=k, w=w, pairs=tuple(pairs))
    tab = O.OracleTable(k, size)
    with DeviceContext(spec, size) as ctx:
        for s in range(1, size + 1):
            r = ctx.count(s)
            _, want, _, _ = O.scan_range(tab, k, w, pairs[:1], s, 0, tab.total(s), 0, tab.total(s),
                                         threads=O.cpu_count())
            assert r.ex0_hits == want, (s, r.ex0_hits, want)


@pytest.mark.gpu
def test_late_splitting_keeps_counts_exact(monkeypatch):
    """With a tiny late-splitting threshold (SIMBA_SPLIT_MIN, read at context
    creation) almost every piece is split through the range pool once the
    claims run dry; per-level counts, first ranks and visited counts of a
    hit-dense spec must still equal the oracle's (no rank lost or doubled)."""
    monkeypatch.setenv("SIMBA_SPLIT_MIN", "2048")
    rng = random.Random(4242)
    pairs, seen = [], set()
    while len(pairs) < 4:
        x = tuple(rng.getrandbits(3) for _ in range(2))
        if x not in seen:
            seen.add(x)
            pairs.append((x, (x[0] * x[1] + x[0]) & 7))  # planted: many formulas match
    spec = S.Specification(k=2, w=3, pairs=tuple(pairs))
    size = 12
    tab = O.OracleTable(2, size)
    with DeviceContext(spec, size) as ctx:
        _, levels = ctx.run_levels(1, size)
        for s, count, first, visited in levels:
            _, want, first_want, _ = O.scan_range(tab, 2, 3, pairs, s, 0, tab.total(s), 0, tab.total(s),
                                                  threads=O.cpu_count())
            assert (count, first, visited) == (want, first_want, tab.total(s)), s
        for shard in range(3):  # sharded, split pieces included
            r = ctx.run(size, 0, tab.total(size), mode="count", shard=shard, nshards=3)
            assert r.visited > 0
        total = sum(ctx.run(size, 0, tab.total(size), mode="count", shard=i, nshards=3).count for i in range(3))
        assert total == levels[-1][1]
    out = S.synthesize(spec, S.build(2, size), S.EngineConfig(size_bound=size))
    first = next((s, f) for s, c, f, _ in levels if c)
    assert (out.size, out.rank) == first


def test_fused_shards_partition_levels_exactly():
    """Sharded fused launches (simba_run_levels with nshards > 1: the
    multi-GPU bench path, with the shard phase budget and claim guide) must
    partition every level's rank space exactly: per-level counts and visited
    counts summed over shards, and the minimum first rank over shards, equal
    the oracle's; in search mode the (size, rank) minimum over shards is the
    oracle's first hit."""
    rng = random.Random(4242)
    pairs, seen = [], set()
    while len(pairs) < 4:
        x = tuple(rng.getrandbits(3) for _ in range(2))
        if x not in seen:
            seen.add(x)
            pairs.append((x, (x[0] * x[1] + x[0]) & 7))  # hit-dense: many formulas match
    spec = S.Specification(k=2, w=3, pairs=tuple(pairs))
    size = 11
    tab = O.OracleTable(2, size)
    want = {}
    for s in range(1, size + 1):
        _, c, f, _ = O.scan_range(tab, 2, 3, pairs, s, 0, tab.total(s), 0, tab.total(s), threads=O.cpu_count())
        want[s] = (c, f, tab.total(s))
    first_hit = min((s, f) for s, (c, f, _) in want.items() if c)
    with DeviceContext(spec, size) as ctx:
        for nsh in (2, 3, 8):
            got = {s: [0, None, 0] for s in range(1, size + 1)}
            for i in range(nsh):
                _, levels = ctx.run_levels(1, size, shard=i, nshards=nsh)
                for s, c, f, v in levels:
                    g = got[s]
                    g[0] += c
                    g[2] += v
                    if f is not None and (g[1] is None or f < g[1]):
                        g[1] = f
            assert {s: tuple(g) for s, g in got.items()} == want, nsh
            hits = []
            for i in range(nsh):
                r, _ = ctx.run_levels(1, size, mode="search", shard=i, nshards=nsh)
                if r.best_rank is not None:
                    hits.append((r.size, r.best_rank))
            assert min(hits) == first_hit, nsh


def test_fused_shards_c5_shape_cover_every_rank():
    """C5 shape (k=4, w=32, n=10, random outputs), sizes 1..12 (1.2e10 ranks):
    8-way sharded fused launches visit every rank of every level exactly once
    and their counts add up to the single launch's."""
    rng = random.Random(8243)
    pairs, seen = [], set()
    while len(pairs) < 10:
        x = tuple(rng.getrandbits(32) for _ in range(4))
        if x not in seen:
            seen.add(x)
            pairs.append((x, rng.getrandbits(32)))
    spec = S.Specification(k=4, w=32, pairs=tuple(pairs))
    size = 12
    table = S.build(4, size)
    with DeviceContext(spec, size) as ctx:
        _, whole = ctx.run_levels(1, size)
        assert [v for *_, v in whole] == [table.total(s) for s in range(1, size + 1)]
        count = {s: 0 for s in range(1, size + 1)}
        visited = {s: 0 for s in range(1, size + 1)}
        for i in range(8):
            _, levels = ctx.run_levels(1, size, shard=i, nshards=8)
            for s, c, _, v in levels:
                count[s] += c
                visited[s] += v
        assert visited == {s: table.total(s) for s in range(1, size + 1)}
        assert count == {s: c for s, c, _, _ in whole}


def test_fused_shards_search_c5_shape_matches_single_launch():
    """Search mode over 8 fused shards (the multi-GPU Algorithm 1): for planted
    k=4 w=32 n=10 targets of sizes 7..10, the lexicographic (size, rank)
    minimum over shards equals the single launch's answer and the
    synthesize() outcome, and the shard holding it decodes the same tokens."""
    from paper_2605_08243_b200 import codec, expr

    rng = random.Random(20261017)
    size = 10
    table = S.build(4, size)
    for target in (7, 8, 9, 10):
        e = codec.sample_uniform(target, table, rng)
        pairs, seen = [], set()
        while len(pairs) < 10:
            x = tuple(rng.getrandbits(32) for _ in range(4))
            if x not in seen:
                seen.add(x)
                pairs.append((x, expr.evaluate(e, x, 32)))
        spec = S.Specification(k=4, w=32, pairs=tuple(pairs))
        with DeviceContext(spec, size) as ctx:
            one, _ = ctx.run_levels(1, size, mode="search")
            assert one.best_rank is not None
            best = None
            for i in range(8):
                r, _ = ctx.run_levels(1, size, mode="search", shard=i, nshards=8)
                if r.best_rank is not None and (best is None or (r.size, r.best_rank) < best[:2]):
                    best = (r.size, r.best_rank, r.tokens)
            assert best == (one.size, one.best_rank, one.tokens), target
        out = S.synthesize(spec, table, S.EngineConfig(size_bound=size))
        assert (out.size, out.rank) == best[:2], target
        assert out.size <= target
