"""Host-side logic on CPU: the drop-in API surface, validation errors, the
128-bit count table against the reference's golden cells, and the C ABI
(every symbol include/simba.h declares is exported; no device calls here)."""

import re
from pathlib import Path

import pytest

import paper_2605_08243_b200 as S
from conftest import ROOT, load_golden
from paper_2605_08243_b200 import _native as N
from paper_2605_08243_b200.expr import MalformedRpnError, RpnExpr, evaluate, parse_infix, to_infix


def test_header_symbols_exported():
    header = (ROOT / "include" / "simba.h").read_text()
    declared = set(re.findall(r"\b(simba_[a-z0-9_]+)\s*\(", header))
    assert declared >= {"simba_scan_range", "simba_run", "simba_synthesize", "simba_table_build"}
    for name in declared:
        assert hasattr(N.lib, name), name
    assert declared == set(N.SIGNATURES), declared ^ set(N.SIGNATURES)


def test_no_device_means_loud_failure():
    if N.device_count() > 0:
        pytest.skip("a device is present")
    spec = S.Specification.of([((1, 2), 3)], k=2)
    with pytest.raises(N.DeviceError):
        S.synthesize(spec, S.build(2, 3), S.EngineConfig(size_bound=3))


def test_tables_match_reference_cells():
    for t in load_golden("tables")["tables"]:
        tab = S.build(t["k"], t["max_size"])
        assert [list(r) for r in tab.rows] == t["rows"]
        assert list(tab.cumulative) == t["cumulative"]


def test_published_mba_cells():
    # test_acceptance.py:27-40 (criterion 1), a sample of the 60 cells
    cells = {(3, 9): 6_298_419, (4, 12): 12_299_156_092, (5, 10): 438_822_815, (8, 9): 383_703_544,
             (6, 11): 11_272_896_474, (7, 10): 2_053_008_573}
    for (k, s), v in cells.items():
        assert S.build(k, s).cumulative_total(s) == v


def test_capacity_error_like_reference():
    cap = load_golden("tables")["capacity_error"]
    with pytest.raises(S.CountCapacityError) as exc:
        S.build(cap["k"], cap["max_size"])
    assert (exc.value.s, exc.value.op) == (cap["s"], cap["op"])


def test_table_queries():
    t = S.build(2, 3)
    assert t.operator_offset(3, S.Op.AND) == 4 and t.operator_offset(3, S.Op.NEG) == 16
    with pytest.raises(ValueError):
        t.operator_offset(1, S.Op.NOT)
    with pytest.raises(ValueError):
        t.total(4)
    with pytest.raises(ValueError):
        S.build(0, 3)


def test_specification_validation():
    with pytest.raises(ValueError):
        S.Specification.of([], k=1)
    with pytest.raises(ValueError):
        S.Specification.of([((1, 2), 0)], k=1)
    with pytest.raises(ValueError):
        S.Specification.of([((1,), 0), ((1,), 1)], k=1)
    with pytest.raises(ValueError):
        S.Specification.of([((1 << 32,), 0)], k=1)
    with pytest.raises(ValueError):
        S.Specification.of([((1,), 0)], k=1, w=99)


def test_engine_config_validation():
    for kw in (dict(size_bound=0), dict(size_bound=1, chunk=0), dict(size_bound=1, mode="scrambled"),
               dict(size_bound=1, workers=0), dict(size_bound=1, kernel="triton")):
        with pytest.raises(ValueError):
            S.EngineConfig(**kw)


def test_synthesize_argument_checks_before_device():
    spec = S.Specification.of([((1,), 1)], k=1)
    with pytest.raises(ValueError):
        S.synthesize(spec, S.build(2, 3), S.EngineConfig(size_bound=2))
    with pytest.raises(ValueError):
        S.synthesize(spec, S.build(1, 3), S.EngineConfig(size_bound=4))


def test_expr_semantics_and_text():
    for e in load_golden("eval")[:200]:
        assert evaluate(RpnExpr(tuple(e["tokens"])), tuple(e["inputs"]), e["w"]) == e["value"]
    add_mba = parse_infix("(x0 ^ x1) + ((x0 & x1) + (x0 & x1))", 2)
    assert to_infix(parse_infix(to_infix(add_mba), 2)) == to_infix(add_mba)
    assert to_infix(RpnExpr((0, 1, -6))) == "(x0 + x1)"
    assert to_infix(RpnExpr((0, 1, -2, -1))) == "~(x0 & x1)"
    with pytest.raises(MalformedRpnError):
        RpnExpr((0, 1))


def test_run_stats_format():
    st = (S.SizeStats(1, 1, 0.5), S.SizeStats(2, 2, 0.5))
    rep = S.run_stats(S.SynthesisOutcome(S.Status.NOT_FOUND, stats=st))
    assert rep["status"] == "not_found" and rep["total_candidates"] == 3
    assert [(r["size"], r["candidates"]) for r in rep["per_size"]] == [(1, 1), (2, 2)]
    rep = S.run_stats(S.SynthesisOutcome(S.Status.FOUND, RpnExpr((0,)), 1, 0, st[:1]))
    assert rep["rank"] == "0" and rep["expr"] == "x0"


def test_gm_reciprocals_exact():
    # the Granlund-Montgomery divisors used by div_T (simba_device.cuh), checked
    # on the host with the same formula for every T[s] of the C5 table
    def magic(d, N):
        l = 0
        while (1 << l) < d:
            l += 1
        m = ((((1 << l) - d) << N) // d) + 1
        return m, min(l, 1), max(l - 1, 0)

    import random
    rng = random.Random(3)
    t = S.build(4, 22)
    for s in range(1, 23):
        d = t.total(s)
        for N_ in (32, 64):
            if d >= 1 << N_:
                continue
            m, s1, s2 = magic(d, N_)
            for _ in range(300):
                n = rng.randrange(1 << N_)
                hi = (n * m) >> N_
                assert (hi + ((n - hi) >> s1)) >> s2 == n // d


def test_context_argument_errors_before_device():
    # checks of simba_ctx_create that run before any device work
    spec = S.Specification.of([((1,) * 10, 0)], k=10)
    with pytest.raises(ValueError, match="2\\^64"):
        S.DeviceContext(spec, 24)  # T[s][8] >= 2^64 for k=10 well below size 24
    with pytest.raises(ValueError):
        S.DeviceContext(S.Specification.of([((1,), 0)], k=1), 25)  # beyond SIMBA_MAX_SIZE
    big_k = S.Specification.of([((0,) * 65, 0)], k=65)
    with pytest.raises(ValueError):
        S.DeviceContext(big_k, 3)


def test_encode_examples_and_errors():
    """codec.encode (codec.py:147-207): reference known answers
    (test_codec.py:52-70)."""
    from paper_2605_08243_b200.codec import CanonicalityError, Rank, encode

    t2 = S.build(2, 5)
    assert encode(parse_infix("(x0 & x1)", 2), t2) == Rank(5, 3)
    assert encode(parse_infix("(x1 & x0)", 2), t2) == Rank(6, 3)
    t3 = S.build(3, 5)
    with pytest.raises(CanonicalityError):
        encode(RpnExpr((0, 1, -2, 2, -2)), t3)  # (x0 & x1) & x2: left size 3 > right size 1
    ok = RpnExpr((0, 1, -2, 2, -7))  # (x0 & x1) - x2: SUB takes any split
    assert encode(ok, t3).size == 5
    with pytest.raises(ValueError):
        encode(RpnExpr((0, 1, -2)), S.build(1, 3))


def test_encode_inverts_the_oracle_decode():
    """Every rank at small (k, s), and sampled ranks at size 10, through the
    CPU oracle's decode (oracle/simba_oracle.c, pinned to the reference)."""
    import random

    import oracle as O
    from paper_2605_08243_b200.codec import encode

    for k, smax in ((1, 7), (2, 6), (3, 5)):
        tab, otab = S.build(k, smax), O.OracleTable(k, smax)
        for s in range(1, smax + 1):
            for n in range(tab.total(s)):
                assert encode(RpnExpr(O.decode(otab, n, s)), tab) == (n, s)
    rng = random.Random(7)
    tab, otab = S.build(4, 10), O.OracleTable(4, 10)
    for _ in range(300):
        n = rng.randrange(tab.total(10))
        assert encode(RpnExpr(O.decode(otab, n, 10)), tab) == (n, 10)


def test_observational_behavior():
    spec = S.Specification.of([((3, 5), 8), ((7, 9), 16)], k=2)
    assert S.observational_behavior(parse_infix("x0 + x1", 2), spec) == (8, 16)


def test_cli_encode(capsys):
    from paper_2605_08243_b200.cli import main

    assert main(["encode", "--k", "2", "--expr", "(x0 & x1)"]) == 0
    assert capsys.readouterr().out.split() == ["3", "5"]
