"""The VFB cache-based baseline (reference baseline.py).

CPU part: the oracle restatement (oracle/vfb_oracle.py) against the golden
records of the unmodified reference run_baseline (tests/golden/vfb.json), and
the host-side report logic against the reference's own known answers
(test_baseline.py).  GPU part: the device enumeration (csrc/vfb_impl.cuh)
against the same goldens -- status, size, RPN tokens, oom_at and every
per-size row -- with the default batch and with small batches (many batches
and tiles per size), on random specs against the oracle, and the reference's
behavioural tests.
"""

import json
import os
import random

import pytest

import paper_2605_08243_b200 as S
from conftest import ROOT
from paper_2605_08243_b200 import baseline as B

GOLD = json.loads((ROOT / "tests" / "golden" / "vfb.json").read_text())


def _spec(case):
    return S.Specification(k=case["k"], w=case["w"], pairs=tuple((tuple(x), y) for x, y in case["pairs"]))


def _spec_from_target(text, k, n=16, seed=0, w=32):
    tgt = S.parse_infix(text, k)
    rng = random.Random(seed)
    pairs, seen = [], set()
    while len(pairs) < n:
        x = tuple(rng.getrandbits(w) for _ in range(k))
        if x not in seen:
            seen.add(x)
            pairs.append((x, S.evaluate(tgt, x, w)))
    return S.Specification(k=k, w=w, pairs=tuple(pairs))


# ---------------------------------------------------------------- CPU

@pytest.mark.parametrize("i", [i for i, c in enumerate(GOLD) if sum(r[3] for r in c["rows"]) < 150_000])
def test_oracle_matches_reference_golden(i):
    import vfb_oracle as V

    c = GOLD[i]
    got = V.vfb(c["k"], c["w"], [(tuple(x), y) for x, y in c["pairs"]], c["size_bound"], c["memory_budget"])
    assert got["status"] == c["status"]
    assert got["size"] == c["size"]
    assert (list(got["tokens"]) if got["tokens"] else None) == c["tokens"]
    assert got["oom_at"] == c["oom_at"]
    assert [list(r) for r in got["rows"]] == c["rows"]


def test_entry_bytes_and_format_mem():
    assert B.entry_bytes(16, 32) == 64
    assert B.modeled_bytes(756_167, 16, 32) == 48_394_688
    assert B.format_mem(999_999) == "<1 MB"
    assert B.format_mem(48_394_688) == "48.4 MB"
    assert B.format_mem(B.modeled_bytes(32_523_385, 16, 32)) == "2.1 GB"
    assert B.format_mem(B.modeled_bytes(21_222, 16, 32)) == "1.4 MB"


def test_project_oom_size_published_threshold():
    # published five-variable cache growth (test_baseline.py:18-29): OOM at size 11
    rows = [(2, 15), (3, 99), (4, 166), (5, 1749), (6, 6874), (7, 115_080), (8, 504_522),
            (9, 5_547_921), (10, 32_523_385)]
    assert B.project_oom_size(rows, 16, 32, 2_500_000_000) == 11
    assert B.project_oom_size([(2, 10), (3, 100)], 16, 32, 64 * 50) == 3
    assert B.project_oom_size([], 16, 32, 100) is None
    assert B.project_oom_size([(2, 10)], 16, 32, 10**12) is None


def test_cache_report_layout():
    rows = (B.CacheSizeRow(1, 2, 2, 2, 128, 1.0), B.CacheSizeRow(2, 4, 6, 4, 384, 2.0),
            B.CacheSizeRow(3, 2, 8, 20, 512, 3.0))
    st = B.CacheStats(k=2, n=16, w=32, rows=rows, oom_at=3, expr_tokens_total=16)
    text = B.cache_report(st)
    head = text.splitlines()[0]
    for col in ("Size", "#MBA", "#VFB cache", "VFB mem", "% cached", "hardware-dependent"):
        assert col in head
    assert "OOM" in text.splitlines()[-1]
    assert "100.0%" in text.splitlines()[2]  # size 2: 6 of 6 expressions cached
    csv = B.cache_report(st, fmt="csv").splitlines()
    assert csv[0].startswith("Size,#MBA,#VFB cache")
    assert csv[1] == "1,2,2,<1 MB,100.0%,0.0"
    assert B.cache_report(B.CacheStats(k=2, n=16, w=32, rows=())) == ""


def test_run_baseline_argument_checks():
    spec = S.Specification.of([((1, 2), 3)], k=2)
    with pytest.raises(ValueError):
        B.run_baseline(spec, 0)


# ---------------------------------------------------------------- GPU

def _check_against(c, outcome, stats):
    assert outcome.status.value == c["status"]
    assert outcome.size == c["size"]
    assert (list(outcome.expr.tokens) if outcome.expr is not None else None) == c["tokens"]
    assert stats.oom_at == c["oom_at"]
    assert [[r.size, r.stored, r.stored_cum, r.candidates] for r in stats.rows] == c["rows"]
    if "expr_tokens_total" in c:
        assert stats.expr_tokens_total == c["expr_tokens_total"]
    assert [(s.size, s.candidates) for s in outcome.stats] == [(r[0], r[3]) for r in c["rows"]]


@pytest.mark.gpu
@pytest.mark.parametrize("batch", [None, "1000", "2049"])
def test_device_matches_reference_golden(batch, monkeypatch):
    if batch:
        monkeypatch.setenv("SIMBA_VFB_BATCH", batch)
    for c in GOLD:
        outcome, stats = B.run_baseline(_spec(c), c["size_bound"], memory_budget=c["memory_budget"])
        _check_against(c, outcome, stats)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(8))
def test_device_matches_oracle_random(seed, monkeypatch):
    import vfb_oracle as V

    rng = random.Random(500 + seed)
    k = rng.choice([1, 2, 3])
    w = rng.choice([1, 2, 4, 7, 8, 16, 31, 32, 33, 64])
    n = rng.choice([1, 2, 3, 6, 12])
    pairs, seen = [], set()
    while len(pairs) < min(n, 1 << (k * w)):
        x = tuple(rng.getrandbits(w) for _ in range(k))
        if x not in seen:
            seen.add(x)
            pairs.append((x, rng.getrandbits(w)))
    spec = S.Specification(k=k, w=w, pairs=tuple(pairs))
    bound = {1: 7, 2: 6, 3: 5}[k]
    budget = rng.choice([2_500_000_000, 40 * B.entry_bytes(len(pairs), w), 0])
    monkeypatch.setenv("SIMBA_VFB_BATCH", str(rng.choice([64, 999, 1 << 20])))
    want = V.vfb(k, w, pairs, bound, budget)
    outcome, stats = B.run_baseline(spec, bound, memory_budget=budget)
    _check_against(dict(want, tokens=list(want["tokens"]) if want["tokens"] else None,
                        rows=[list(r) for r in want["rows"]]), outcome, stats)


@pytest.mark.gpu
def test_reference_behaviours():
    # test_baseline.py:46-134, restated
    for k in (3, 5, 8):
        spec = _spec_from_target(" + ".join(f"x{i}" for i in range(k)), k, seed=k)
        _, st = B.run_baseline(spec, 2)
        assert st.rows[-1].stored_cum == 3 * k and st.rows[-1].candidates == 2 * k and st.oom_at is None
    spec = S.Specification.of([((i,), (i * 77) & 0xFFFFFFFF) for i in range(2, 18)], k=1)
    _, st = B.run_baseline(spec, 3)
    assert [r.candidates for r in st.rows] == [1, 2, 10] and [r.stored for r in st.rows] == [1, 2, 5]
    spec = _spec_from_target("x2 + (x0 & x0)", 4, seed=3)
    out, st = B.run_baseline(spec, 5)
    assert out.status is S.Status.FOUND and out.size == 3 and S.check(out.expr, spec) and st.rows[-1].size == 3
    table = S.build(2, 5)
    rng = random.Random(31)
    for text in ("x0", "~(x0 ^ x1)", "x0 * x0", "(x1 - x0) & x1"):
        spec = _spec_from_target(text, 2, seed=rng.randrange(1 << 30))
        eng = S.synthesize(spec, table, S.EngineConfig(size_bound=5))
        base, _ = B.run_baseline(spec, 5)
        assert eng.status is base.status is S.Status.FOUND and eng.size == base.size
    spec = _spec_from_target("x0 + x1", 2, seed=9)
    out, st = B.run_baseline(spec, 6, memory_budget=B.entry_bytes(16, 32) * 5)
    assert out.status is S.Status.OOM_ABORTED and st.oom_at == 2 and st.rows[-1].stored_cum <= 5
    spec = _spec_from_target("~(x0)", 1, seed=2)
    out, st = B.run_baseline(spec, 2, memory_budget=B.entry_bytes(16, 32))
    assert out.status is S.Status.FOUND and out.size == 2 and st.oom_at is None
    spec = _spec_from_target("(x0 * x1) ^ (x2 + x0)", 3, seed=5)
    out, _ = B.run_baseline(spec, 12, time_budget=0.02)
    assert out.status in (S.Status.TIMED_OUT, S.Status.FOUND)
    spec = _spec_from_target("~(x0 * x1)", 2, seed=12)
    _, st = B.run_baseline(spec, 5)
    for r in st.rows:
        assert r.stored <= r.candidates and r.modeled_bytes == r.stored_cum * 64
    text = B.cache_report(st)
    assert "#VFB cache" in text.splitlines()[0]


@pytest.mark.gpu
def test_device_memory_is_not_the_modeled_budget():
    """A budget far above the device is fine while the entries actually
    stored fit; the modeled budget alone decides OOM."""
    spec = _spec_from_target("(x0 * x1) ^ (x2 + x0)", 3, seed=5, n=10)
    out, st = B.run_baseline(spec, 6, memory_budget=10**15)
    assert st.oom_at is None and out.status in (S.Status.FOUND, S.Status.NOT_FOUND)
