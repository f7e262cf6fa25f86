"""CLI drop-in (cli.py of the reference): formats and exit codes.
CPU tests cover parsing / usage / I-O errors; GPU tests run synth."""

import json

import pytest

import paper_2605_08243_b200 as S
from paper_2605_08243_b200 import _native as N
from paper_2605_08243_b200.cli import EXIT_IO, EXIT_NOT_FOUND, EXIT_TIMED_OUT, EXIT_USAGE, main, write_spec_file


def run(capsys, *argv):
    code = main(list(argv))
    out, err = capsys.readouterr()
    return code, out, err


def identity_spec(path):
    write_spec_file(path, S.Specification.of([((i,), i) for i in range(1, 17)], k=1))
    return path


def test_count_table_tsv(capsys):
    code, out, _ = run(capsys, "count", "--k", "5", "--max-size", "10", "--cumulative")
    assert code == 0
    assert out.strip().splitlines()[-1].split("\t")[-1] == "438822815"


def test_missing_spec_is_io_error(capsys, tmp_path):
    code, _, err = run(capsys, "synth", "--spec", str(tmp_path / "nope.json"))
    assert code == EXIT_IO and "cannot read" in err


def test_bad_spec_is_io_error(capsys, tmp_path):
    p = tmp_path / "bad.json"
    p.write_text('{"w": 8, "k": 1, "pairs": [{"in": ["0x1ff"], "out": "0x01"}]}')
    code, _, _ = run(capsys, "synth", "--spec", str(p))
    assert code == EXIT_IO


def test_usage_error(capsys):
    with pytest.raises(SystemExit) as exc:
        main(["synth"])
    assert exc.value.code == EXIT_USAGE


@pytest.mark.gpu
def test_synth_found_json_and_exit_codes(capsys, tmp_path):
    assert N.device_count() > 0
    path = identity_spec(tmp_path / "id.spec")
    code, out, _ = run(capsys, "synth", "--spec", str(path))
    assert code == 0 and out.strip() == "x0"
    code, out, _ = run(capsys, "synth", "--spec", str(path), "--json")
    doc = json.loads(out)
    assert (doc["status"], doc["expr"], doc["size"], doc["rank"]) == ("found", "x0", 1, "0")
    assert doc["per_size"][0]["candidates"] == 1
    no = tmp_path / "no.spec"
    write_spec_file(no, S.Specification.of([((0,), 1), ((1,), 0)], k=1))
    code, out, _ = run(capsys, "synth", "--spec", str(no), "--max-size", "2")
    assert code == EXIT_NOT_FOUND and "not_found" in out


@pytest.mark.gpu
def test_synth_timeout_exit_two(capsys, tmp_path):
    spec = S.Specification.of([((i, 2 * i, 3 * i), (i * 0x9E3779B9) & 0xFFFFFFFF) for i in range(1, 17)], k=3)
    path = tmp_path / "hard.spec"
    write_spec_file(path, spec)
    code, _, _ = run(capsys, "synth", "--spec", str(path), "--max-size", "14", "--timeout", "0.02")
    assert code == EXIT_TIMED_OUT


@pytest.mark.gpu
def test_count_solutions_cli(capsys, tmp_path):
    path = identity_spec(tmp_path / "id.spec")
    code, out, _ = run(capsys, "count-solutions", "--spec", str(path), "--max-size", "3")
    doc = json.loads(out)
    assert code == 0 and doc[0]["count"] == 1 and doc[0]["first_rank"] == "0"


@pytest.mark.gpu
def test_baseline_subcommand(capsys, tmp_path):
    """reference test_cli.py:145-152: the cache report, then the formula."""
    path = identity_spec(tmp_path / "id.spec")
    code, out, _ = run(capsys, "baseline", "--spec", str(path), "--max-size", "3")
    assert code == 0
    assert "#VFB cache" in out
    assert "found: x0 (size 1)" in out
    code, out, _ = run(capsys, "baseline", "--spec", str(path), "--max-size", "3", "--report", "csv")
    assert code == 0 and out.startswith("Size,#MBA,#VFB cache")


def test_baseline_usage(capsys):
    with pytest.raises(SystemExit) as exc:
        main(["baseline", "--max-size", "3"])
    assert exc.value.code == EXIT_USAGE
