"""Benchmark-suite harness (suite.py) against the reference's bench module.

Fixtures: tests/golden/suite.json, written by tests/golden/make_suite_golden.py
from the unmodified reference (generate_suite / write_suite / run_suite /
summarize, bench.py:90-472).
"""

import json
from pathlib import Path

import pytest

from paper_2605_08243_b200 import cli, suite
from paper_2605_08243_b200.expr import to_infix

GOLD = json.loads((Path(__file__).parent / "golden" / "suite.json").read_text())


def _suite_from_text(tmp_path):
    p = tmp_path / "suite.jsonl"
    p.write_text(GOLD["suite_jsonl"])
    return suite.read_suite(p)


def test_instance_seeds_match_reference():
    items = [json.loads(l) for l in GOLD["suite_jsonl"].splitlines()[1:]]
    for rec in items:
        s, k, i = int(rec["id"][1:3]), rec["k"], int(rec["id"].split("_i")[1])
        assert suite.instance_seed(GOLD["seed"], k, s, i) == rec["seed"]


def test_suite_file_round_trip_is_byte_identical(tmp_path):
    items = _suite_from_text(tmp_path)
    assert [to_infix(i.ground_truth) for i in items] == GOLD["ground_truth"]
    out = tmp_path / "again.jsonl"
    suite.write_suite(out, items, seed=GOLD["seed"])
    assert out.read_text() == GOLD["suite_jsonl"]


def _fake_records():
    return [suite.RunRecord(i, s, st, z, ms, rep) for i, s, st, z, ms, rep in GOLD["fake_records"]]


def test_records_csv_matches_reference(tmp_path):
    recs = _fake_records()
    p = tmp_path / "r.csv"
    suite.write_records_csv(p, recs)
    assert p.read_text() == GOLD["fake_records_csv"]
    assert suite.read_records_csv(p) == [suite.RunRecord(r.instance, r.solver, r.status, r.size,
                                                         float(f"{r.millis:.3f}"), r.repeat) for r in recs]


def test_summaries_match_reference(tmp_path):
    items = _suite_from_text(tmp_path)
    recs = _fake_records()
    th = [0.05, 0.1, 0.2, 0.4]
    summ = suite.summarize(recs, items, thresholds=th)
    gold = GOLD["summary"]
    assert {s: [list(r) for r in rows] for s, rows in summ["solved_curve"].items()} == gold["solved_curve"]
    for key in ("solved_by_size", "solved_by_vars"):
        assert {s: {str(g): v for g, v in row.items()} for s, row in summ[key].items()} == gold[key]
    assert [[a, b, h] for (a, b), h in summ["head_to_head"].items()] == gold["head_to_head"]
    suite.write_summaries(tmp_path / "out", recs, items, thresholds=th)
    for name, text in GOLD["summary_csvs"].items():
        assert (tmp_path / "out" / name).read_text() == text, name


def test_bench_cli_rejects_unknown_solver(tmp_path, capsys):
    p = tmp_path / "suite.jsonl"
    p.write_text(GOLD["suite_jsonl"])
    rc = cli.main(["bench", "run", "--suite", str(p), "--solvers", "vfb", "--records", str(tmp_path / "r.csv")])
    assert rc == cli.EXIT_IO


@pytest.mark.gpu
def test_generate_suite_matches_reference(tmp_path):
    lo, hi = GOLD["sizes"]
    vlo, vhi = GOLD["vars"]
    items = suite.generate_suite(GOLD["seed"], sizes=range(lo, hi + 1), var_counts=range(vlo, vhi + 1),
                                 per_cell=GOLD["per_cell"])
    out = tmp_path / "gen.jsonl"
    suite.write_suite(out, items, seed=GOLD["seed"])
    assert out.read_text() == GOLD["suite_jsonl"]


@pytest.mark.gpu
def test_run_suite_matches_reference(tmp_path):
    items = _suite_from_text(tmp_path)
    records, normalized = suite.run_suite(items, solvers=("simba", "simba-rtid", "baseline"), timeout=None)
    assert [{"instance": r.instance, "solver": r.solver, "status": r.status, "size": r.size}
            for r in records] == GOLD["records"]
    assert [{"id": i.id, "norm_size": i.norm_size, "norm_vars": i.norm_vars,
             "norm_upper_bound": i.norm_upper_bound} for i in normalized] == GOLD["normalized"]


@pytest.mark.gpu
def test_bench_cli_end_to_end(tmp_path):
    p = tmp_path / "suite.jsonl"
    assert cli.main(["bench", "gen", "--seed", str(GOLD["seed"]), "--out", str(p), "--sizes", "3..4",
                     "--vars", "2", "--per-cell", "2"]) == 0
    rc = cli.main(["bench", "run", "--suite", str(p), "--solvers", "simba,simba-rtid,baseline", "--timeout", "30",
                   "--records", str(tmp_path / "r.csv"), "--summary-dir", str(tmp_path / "sum")])
    assert rc == 0
    recs = suite.read_records_csv(tmp_path / "r.csv")
    assert len(recs) == 12 and all(r.status == "found" for r in recs)
    assert sorted(x.name for x in (tmp_path / "sum").iterdir()) == sorted(GOLD["summary_csvs"])
