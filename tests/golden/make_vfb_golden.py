"""Golden fixtures for the VFB cache baseline, from the UNMODIFIED reference
``mbasynth.baseline.run_baseline`` (baseline.py:88-249).

Test infrastructure only; run in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_vfb_golden.py

Writes tests/golden/vfb.json: per case the spec (k, w, pairs), size bound and
memory budget, and the reference's status, size, RPN tokens, oom_at,
expr_tokens_total and per-size rows (size, stored, stored_cum, candidates).
"""

from __future__ import annotations

import json
import random
from pathlib import Path

from mbasynth.baseline import entry_bytes, run_baseline
from mbasynth.engine import Specification
from mbasynth.expr import evaluate, parse_infix

HERE = Path(__file__).resolve().parent


def spec(k, w, n, seed, target=None):
    rng = random.Random(seed)
    pairs, seen = [], set()
    tgt = parse_infix(target, k) if target else None
    while len(pairs) < n:
        x = tuple(rng.getrandbits(w) for _ in range(k))
        if x in seen:
            continue
        seen.add(x)
        pairs.append((x, evaluate(tgt, x, w) if tgt else rng.getrandbits(w)))
    return Specification(k=k, w=w, pairs=tuple(pairs))


CASES = [
    # (k, w, n, seed, target or None for random outputs, size bound, budget entries or None)
    (1, 32, 16, 2, "~(x0)", 3, None),
    (2, 32, 16, 9, "x0 + x1", 4, None),
    (2, 32, 16, 9, "x0 + x1", 6, 5),            # OOM at size 2 (test_baseline.py:90-96)
    (2, 32, 16, 4, "x0 ^ x1", 4, 8),
    (2, 8, 4, 0, "(x0 ^ x1) + ((x0 & x1) + (x0 & x1))", 5, None),  # C1
    (2, 32, 10, 11, "(x1 - x0) & x1", 5, None),
    (2, 32, 10, 12, "~(x0 * x1)", 6, None),
    (3, 32, 10, 13, "(x0 * x1) ^ (x2 + x0)", 7, None),
    (3, 32, 10, 14, None, 6, None),              # unsat: full sweep
    (3, 32, 10, 14, None, 6, 2000),              # unsat with a budget: OOM mid-size
    (1, 32, 16, 15, "x0 * x0 + x0", 6, None),
    (2, 3, 5, 16, None, 6, None),                # tiny width: heavy deduplication
    (2, 2, 3, 17, "x0 - x1", 5, None),
    (4, 64, 6, 18, "(x0 & x3) - x1", 4, None),   # w = 64
    (3, 64, 20, 19, None, 5, 400),
    (2, 16, 8, 20, "-(x0 | x1)", 5, None),
    # larger sweeps: several device batches with a small batch size
    (3, 32, 10, 21, None, 9, None),
    (2, 32, 10, 22, None, 10, None),
    (4, 32, 10, 23, None, 7, None),
    (3, 32, 10, 24, None, 9, 300_000),
    (3, 32, 10, 25, "((x0 + x2) * x1) - (x2 ^ x0)", 9, None),
]


def main():
    out = []
    for k, w, n, seed, target, bound, budget_entries in CASES:
        sp = spec(k, w, n, seed, target)
        budget = 2_500_000_000 if budget_entries is None else budget_entries * entry_bytes(n, w)
        outcome, stats = run_baseline(sp, bound, memory_budget=budget)
        out.append({
            "k": k, "w": w, "pairs": [[list(x), y] for x, y in sp.pairs], "size_bound": bound,
            "memory_budget": budget, "target": target,
            "status": outcome.status.value, "size": outcome.size,
            "tokens": list(outcome.expr.tokens) if outcome.expr is not None else None,
            "oom_at": stats.oom_at, "expr_tokens_total": stats.expr_tokens_total,
            "rows": [[r.size, r.stored, r.stored_cum, r.candidates] for r in stats.rows],
        })
    (HERE / "vfb.json").write_text(json.dumps(out, indent=0))
    print(len(out), "cases ->", HERE / "vfb.json")


if __name__ == "__main__":
    main()
