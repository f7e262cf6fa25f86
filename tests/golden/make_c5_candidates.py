"""C5 inputs for the production-path goldens, drawn with the UNMODIFIED reference.

Test infrastructure only.  Run in the build container (where /root/reference
exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_c5_candidates.py

Writes tests/golden/c5_candidates.json:

  planted   two k=4 w=32 n=10 specs labelled by a known target
            (bench.spec_for_target, bench.py:67-82): "dense" = x0 + x1 (size 3:
            satisfying candidates at every level 3..13), "sparse" = a uniform
            size-9 expression (codec.sample_uniform, codec.py:239-244).  Their
            per-level counts and first ranks over sizes 1..13 (1.12e11
            candidates each) are computed by make_c5_golden.py with the
            multithreaded CPU oracle.
  suite     the reference's own suite generator (bench.generate_suite,
            bench.py:90-137) for k=4, w=32, n=10, sizes 11..13, PER_CELL
            instances per size.  make_c5_golden.py keeps, per size, the first
            ten whose minimal solution size equals the generated size (the
            difficulty label of bench.normalize, bench.py:140-163) and pins
            their oracle (size, rank, tokens).
"""

from __future__ import annotations

import json
import random
from pathlib import Path

from mbasynth import bench, codec, counting
from mbasynth.expr import parse_infix

HERE = Path(__file__).resolve().parent
MASTER_SEED = 2605_08243
PER_CELL = 60
SIZES = (11, 12, 13)
K, W, N = 4, 32, 10


def spec_json(spec):
    return {"k": spec.k, "w": spec.w, "pairs": [[list(i), o] for i, o in spec.pairs]}


def main():
    table = counting.build(K, 13)
    planted = []
    dense = parse_infix("x0 + x1", K)
    planted.append({"name": "dense_x0_plus_x1", "target": list(dense.tokens),
                    "spec": spec_json(bench.spec_for_target(dense, K, random.Random(11), n=N, w=W))})
    rng = random.Random(9)
    sparse = codec.sample_uniform(9, table, rng)
    planted.append({"name": "sparse_size9", "target": list(sparse.tokens),
                    "spec": spec_json(bench.spec_for_target(sparse, K, rng, n=N, w=W))})
    suite = bench.generate_suite(MASTER_SEED, sizes=SIZES, var_counts=(K,), per_cell=PER_CELL, n_pairs=N, w=W)
    out = {
        "generator": "reference mbasynth bench.generate_suite / spec_for_target (unmodified)",
        "master_seed": MASTER_SEED, "per_cell": PER_CELL, "k": K, "w": W, "n": N,
        "planted": planted,
        "suite": [{"id": b.id, "gen_size": b.gen_size, "target": list(b.ground_truth.tokens),
                   "spec": spec_json(b.spec)} for b in suite],
    }
    (HERE / "c5_candidates.json").write_text(json.dumps(out) + "\n")
    print(f"{len(planted)} planted specs, {len(out['suite'])} suite instances")


if __name__ == "__main__":
    main()
