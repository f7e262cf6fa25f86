"""The production tile paths against the oracle on specs WITH hits.

The bench's C5 sweep runs through launch shapes that only switch on for
large launches: R0 + 1 column rows on the largest levels,
2^18-candidate descriptors and claim guide 4 from 4e10 candidates per shard.
Here they are (a) forced on hit-dense k = 2..4 specs small enough for the
oracle at test time (SIMBA_R0_UP: the level from which R0 + 1 is used;
SIMBA_BIG_LAUNCH: the big-launch threshold in candidates per shard), and
(b) reached naturally by the full C5 sweep of planted specs whose per-level
counts and first ranks over sizes 1..13 (1.12e11 candidates) the
multithreaded oracle computed once (tests/golden/c5.json,
make_c5_golden.py).  Reference: Alg. 1 engine.py:190-276; the count oracle
enumerate_all + check, engine.py:279-293, expr.py:201-218.
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


def dense_spec(k, w, n, seed, f):
    rng = random.Random(seed)
    pairs, seen = [], set()
    while len(pairs) < n:
        x = tuple(rng.getrandbits(w) for _ in range(k))
        if x not in seen:
            seen.add(x)
            pairs.append((x, f(x) & ((1 << w) - 1)))
    return {"k": k, "w": w, "pairs": [[list(x), y] for x, y in pairs]}


# (spec, size bound, level from which R0 + 1 is forced)
DENSE = {
    "k2_w3": (dense_spec(2, 3, 4, 4242, lambda x: x[0] * x[1] + x[0]), 12, 9),
    "k3_w4": (dense_spec(3, 4, 5, 77, lambda x: (x[0] ^ x[1]) + x[2]), 11, 8),
    "k4_w32_x0px1": (dense_spec(4, 32, 10, 11, lambda x: x[0] + x[1]), 10, 8),
    "k4_w8": (dense_spec(4, 8, 6, 5, lambda x: (x[0] & x[1]) - x[3]), 10, 8),
}

_oracle_cache = {}


def oracle_levels(name):
    if name not in _oracle_cache:
        sp, C, _ = DENSE[name]
        tab = O.OracleTable(sp["k"], C)
        pairs = [(tuple(i), o) for i, o in sp["pairs"]]
        out = []
        for s in range(1, C + 1):
            _, c, f, _ = O.scan_range(tab, sp["k"], sp["w"], pairs, s, 0, tab.total(s), 0, tab.total(s),
                                      threads=O.cpu_count())
            out.append((s, c, f, tab.total(s)))
        _oracle_cache[name] = out
    return _oracle_cache[name]


SHAPES = {
    "default": {},
    "r0up": {"r0up": True},
    "big": {"SIMBA_BIG_LAUNCH": "1"},
    "r0up_big": {"r0up": True, "SIMBA_BIG_LAUNCH": "1"},
    "r0up_big_split": {"r0up": True, "SIMBA_BIG_LAUNCH": "1", "SIMBA_SPLIT_MIN": "4096"},
}


@pytest.mark.parametrize("shape", list(SHAPES))
@pytest.mark.parametrize("name", list(DENSE))
def test_forced_launch_shapes_match_oracle(name, shape, monkeypatch):
    sp, C, r0up = DENSE[name]
    for key, val in SHAPES[shape].items():
        if key == "r0up":
            monkeypatch.setenv("SIMBA_R0_UP", str(r0up))
        else:
            monkeypatch.setenv(key, val)
    want = oracle_levels(name)
    assert any(c for _, c, _, _ in want), "spec must have hits"
    first_hit = next((s, f) for s, c, f, _ in want if c)
    spec = spec_of(sp)
    with DeviceContext(spec, C) as ctx:
        info = ctx.info()
        if "r0up" in SHAPES[shape]:
            assert info["r0"] + 1 <= info["rg"], info  # the forced shape is really available
        r, levels = ctx.run_levels(1, C, mode="count")
        assert [tuple(x) for x in levels] == want, (name, shape)
        assert r.count == sum(c for _, c, _, _ in want)
        # search: the lexicographic minimum (size, rank) and its tokens
        r, _ = ctx.run_levels(1, C, mode="search")
        assert (r.size, r.best_rank) == first_hit
        # the whole top level alone (single-level launch shapes)
        top = ctx.count(C)
        assert (top.count, top.best_rank, top.visited) == want[-1][1:]
        # 3-way shards of the fused count add up exactly
        tot = {s: [0, None, 0] for s in range(1, C + 1)}
        for i in range(3):
            _, lv = ctx.run_levels(1, C, mode="count", shard=i, nshards=3)
            for s, c, f, v in lv:
                t = tot[s]
                t[0] += c
                t[2] += v
                if f is not None and (t[1] is None or f < t[1]):
                    t[1] = f
        assert [(s, *t) for s, t in sorted(tot.items())] == [tuple(x) for x in want]
    out = S.synthesize(spec, S.build(sp["k"], C), S.EngineConfig(size_bound=C))
    assert (out.size, out.rank) == first_hit


def test_dense_k2_w3_size12_stress_repeated():
    """The hit-dense k=2 w=3 case of the round-1 order-dependent fault
    (DESIGN.md 6): repeated full sweeps of sizes 1..12 (3.6e8 candidates,
    about one example-0 hit per 8 candidates) stay exact."""
    want = oracle_levels("k2_w3")
    sp, C, _ = DENSE["k2_w3"]
    with DeviceContext(spec_of(sp), C) as ctx:
        for _ in range(5):
            _, levels = ctx.run_levels(1, C, mode="count")
            assert [tuple(x) for x in levels] == want


# ------------------------------------------------------------ full C5 sweeps


def c5_golden():
    try:
        return load_golden("c5")
    except FileNotFoundError:
        pytest.skip("tests/golden/c5.json not generated")


@pytest.mark.timeout(600)
def test_c5_planted_full_sweep_levels_1_to_13():
    """Unsharded production launch of all 13 levels (the bench step's shape:
    R0 + 1 on levels 12-13, big descriptors, late splitting) on planted specs
    with hits: per-level counts and first ranks equal the oracle's full
    1.12e11-candidate sweep; so do the single size-13 launch and synthesize."""
    g = c5_golden()
    table = S.build(4, 13)
    for p in g["planted"]:
        spec = spec_of(p["spec"])
        want = [(x["size"], x["count"], x["first"], x["candidates"]) for x in p["levels"]]
        with DeviceContext(spec, 13) as ctx:
            r, levels = ctx.run_levels(1, 13, mode="count")
            assert [tuple(x) for x in levels] == want, p["name"]
            top = ctx.count(13)
            assert (top.count, top.best_rank, top.visited) == want[-1][1:], p["name"]
            # 8 shards (the multi-GPU partition) add up to the same
            tot_c = [0] * 13
            for i in range(8):
                _, lv = ctx.run_levels(1, 13, mode="count", shard=i, nshards=8)
                for s, c, _, _ in lv:
                    tot_c[s - 1] += c
            assert tot_c == [c for _, c, _, _ in want], p["name"]
        first = next((s, f) for s, c, f, _ in want if c)
        out = S.synthesize(spec, table, S.EngineConfig(size_bound=13))
        assert (out.size, out.rank) == first, p["name"]


@pytest.mark.timeout(600)
def test_c5_time_to_solve_suite_matches_oracle():
    """The 30 time-to-solve targets (ten per size 11, 12, 13 whose minimal
    size is that size): synthesize returns the oracle's (size, rank, tokens)."""
    g = c5_golden()
    table = S.build(4, 13)
    n = 0
    for size, recs in g["tts"].items():
        for rec in recs:
            out = S.synthesize(spec_of(rec["spec"]), table, S.EngineConfig(size_bound=13))
            o = rec["oracle"]
            assert (out.size, out.rank, list(out.expr.tokens)) == (o["size"], o["rank"], o["tokens"]), rec["id"]
            assert out.size == int(size)
            n += 1
    assert n == sum(len(v) for v in g["tts"].values()) > 0


@pytest.mark.parametrize("name", ["k3_w4", "k4_w32_x0px1"])
def test_value_tables_bottom_up_equal_per_entry_decode(name, monkeypatch):
    """The value tables are built bottom-up (one operator per entry over the
    levels below); SIMBA_VT_DECODE=1 builds them by the reference-exact
    per-entry decode + eval instead.  Both give the oracle's counts."""
    sp, C, _ = DENSE[name]
    want = oracle_levels(name)
    for mode in ("0", "1"):
        monkeypatch.setenv("SIMBA_VT_DECODE", mode)
        with DeviceContext(spec_of(sp), C) as ctx:
            _, levels = ctx.run_levels(1, C, mode="count")
        assert [tuple(x) for x in levels] == want, mode


@pytest.mark.parametrize("mode", ["local", "shuffled"])
def test_budget_never_reports_a_non_minimal_hit(mode):
    """Under a time budget a run dropped by the budget records its lowest rank;
    a hit above a dropped run is not reported (the reference, scanning chunks
    in order, would have timed out before it, engine.py:251-258), and in
    shuffled order a cut-short block reports no hit.  So every FOUND equals
    the oracle's minimum, whatever the budget -- checked over budgets from
    0 to well past the search time on a spec with hits at many ranks."""
    sp, C, _ = DENSE["k4_w32_x0px1"]
    want = oracle_levels("k4_w32_x0px1")
    first = next((s, f) for s, c, f, _ in want if c)
    # a spec whose first hit sits deep in a large level: the pieces below it
    # are what a budget can drop
    spec = spec_of(sp)
    table = S.build(4, C)
    seen = set()
    for budget in (0.0, 1e-5, 3e-5, 1e-4, 3e-4, 1e-3, 1.0):
        for _ in range(3):
            out = S.synthesize(spec, table, S.EngineConfig(size_bound=C, mode=mode, time_budget=budget))
            seen.add(out.status)
            if out.status is S.Status.FOUND:
                assert (out.size, out.rank) == first, (budget, mode)
            else:
                assert out.status is S.Status.TIMED_OUT and out.expr is None
    assert S.Status.FOUND in seen


# ------------------------------------------- per-example tables chosen at creation


def _collapsed_spec(k, w, n, seed, target_size):
    """Example 0 has all inputs equal (v, v, ..., v) -- most expressions
    collapse onto a few values there, so example 0 is dense at its output --
    the others are random; labelled by a uniform expression of target_size."""
    from paper_2605_08243_b200 import codec, expr

    rng = random.Random(seed)
    e = codec.sample_uniform(target_size, S.build(k, target_size), rng)
    v = rng.getrandbits(w) | (1 << (w - 1))
    xs = [tuple([v] * k)]
    while len(xs) < n:
        x = tuple(rng.getrandbits(w) for _ in range(k))
        if x not in xs:
            xs.append(x)
    return S.Specification(k=k, w=w, pairs=tuple((x, expr.evaluate(e, x, w)) for x in xs))


@pytest.mark.parametrize("k,w,n,emax", [(3, 64, 3, 2), (3, 32, 5, 4)])
def test_dense_example_zero_gets_tables_in_place_and_is_reordered(k, w, n, emax, monkeypatch):
    """Searches of >= 2^30 candidates (k=3, sizes 1..12) measure example 0's
    density after building its table; a dense example 0 makes the same
    context add the other examples' tables (E = emax: n = 3 -> 2, n = 5 -> 4)
    and swap the sparsest tabled example into place (their rows of the staged
    examples and their table slices; 64-bit words too).  The answer is the
    oracle's, as with tables for example 0 only (SIMBA_EX0_DENSE=2: never
    dense)."""
    spec = _collapsed_spec(k, w, n, 2001, 7)  # minimal answer at size 7 (seed 1003: size 2)
    tab = O.OracleTable(k, 9)
    want = None
    for s in range(1, 10):
        _, _, first, _ = O.scan_range(tab, k, w, [tuple(p) for p in spec.pairs], s, 0, tab.total(s), 0, tab.total(s),
                                      threads=O.cpu_count())
        if first is not None:
            want = (s, first)
            break
    assert want is not None
    table = S.build(k, 12)
    with DeviceContext(spec, 12) as ctx:
        assert ctx.info()["table_examples"] == emax
        r, _ = ctx.run_levels(1, 12, mode="search")
        assert (r.size, r.best_rank) == want
    out = S.synthesize(spec, table, S.EngineConfig(size_bound=12))
    assert (out.size, out.rank) == want
    monkeypatch.setenv("SIMBA_EX0_DENSE", "2")
    with DeviceContext(spec, 12) as ctx:
        assert ctx.info()["table_examples"] == 1
        r, _ = ctx.run_levels(1, 12, mode="search")
        assert (r.size, r.best_rank) == want
