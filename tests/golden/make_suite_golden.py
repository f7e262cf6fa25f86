"""Golden fixtures for the benchmark-suite harness (suite.py), from the
UNMODIFIED reference ``mbasynth.bench``.

Test infrastructure only; run in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_suite_golden.py

Writes tests/golden/suite.json with
  suite      bench.generate_suite(seed, sizes, vars, per_cell) written by
             bench.write_suite (the exact JSONL text)            [bench.py:90-137, 172-194]
  records    bench.run_suite(suite, solvers=("simba", "simba-rtid", "baseline"), timeout=None)
             statuses/sizes per instance and the normalized labels [bench.py:234-304, 140-163]
  summary    bench.summarize on a fixed synthetic record set      [bench.py:340-440]
"""

from __future__ import annotations

import io
import json
import os
import tempfile
from pathlib import Path

from mbasynth import bench
from mbasynth.expr import to_infix

HERE = Path(__file__).resolve().parent
SEED, SIZES, VARS, PER_CELL = 20261017, range(3, 7), range(2, 4), 3


def main():
    suite = bench.generate_suite(SEED, sizes=SIZES, var_counts=VARS, per_cell=PER_CELL)
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "suite.jsonl")
        bench.write_suite(path, suite, seed=SEED)
        text = Path(path).read_text()
    records, normalized = bench.run_suite(suite, solvers=("simba", "simba-rtid", "baseline"), timeout=None)
    rec = [{"instance": r.instance, "solver": r.solver, "status": r.status, "size": r.size} for r in records]
    norm = [{"id": i.id, "norm_size": i.norm_size, "norm_vars": i.norm_vars,
             "norm_upper_bound": i.norm_upper_bound} for i in normalized]
    # summaries over a fixed record set (timings synthetic so the output is deterministic)
    fake = []
    for j, inst in enumerate(suite):
        for rep in range(2):
            for solver, scale in (("simba", 1.0), ("simba-rtid", 3.0)):
                status = "found" if (j + rep) % 5 else "timed_out"
                fake.append(bench.RunRecord(inst.id, solver, status, inst.gen_size if status == "found" else None,
                                            scale * (10.0 + 7.0 * j + rep), rep))
    summ = bench.summarize(fake, suite, thresholds=[0.05, 0.1, 0.2, 0.4])
    summ_json = {
        "solved_curve": summ["solved_curve"],
        "solved_by_size": {s: {str(k): v for k, v in g.items()} for s, g in summ["solved_by_size"].items()},
        "solved_by_vars": {s: {str(k): v for k, v in g.items()} for s, g in summ["solved_by_vars"].items()},
        "head_to_head": [[a, b, h] for (a, b), h in summ["head_to_head"].items()],
    }
    with tempfile.TemporaryDirectory() as td:
        bench.write_records_csv(os.path.join(td, "r.csv"), fake)
        rec_csv = Path(td, "r.csv").read_text()
        bench.write_summaries(td, fake, suite, thresholds=[0.05, 0.1, 0.2, 0.4])
        csvs = {n: Path(td, n).read_text() for n in sorted(os.listdir(td)) if n != "r.csv"}
    fake_json = [[r.instance, r.solver, r.status, r.size, r.millis, r.repeat] for r in fake]
    out = {"seed": SEED, "sizes": [SIZES.start, SIZES.stop - 1], "vars": [VARS.start, VARS.stop - 1],
           "per_cell": PER_CELL, "suite_jsonl": text,
           "ground_truth": [to_infix(i.ground_truth) for i in suite],
           "records": rec, "normalized": norm,
           "fake_records": fake_json, "fake_records_csv": rec_csv,
           "summary": summ_json, "summary_csvs": csvs}
    (HERE / "suite.json").write_text(json.dumps(out, indent=0))
    print(f"{len(suite)} instances, {len(records)} records -> suite.json")


if __name__ == "__main__":
    main()
