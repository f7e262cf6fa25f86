"""CPU restatement of the VFB cache-based baseline (reference baseline.py:88-249).

TEST INFRASTRUCTURE ONLY -- the checker for paper_2605_08243_b200.baseline's
device enumeration (csrc/vfb_impl.cuh); imported by tests/ only, never by the
product package.  Pure Python, for the small cases the parity tests use.

Pinned against the reference itself: tests/golden/vfb.json holds outcomes and
per-size rows of the unmodified ``mbasynth.baseline.run_baseline`` on seeded
specs (tests/golden/make_vfb_golden.py), and tests/test_vfb.py checks this
restatement against every record there.
"""

from __future__ import annotations

NOT, AND, OR, XOR, NEG, ADD, SUB, MUL = range(8)  # operator slots (expr.py:22-32)
COMMUTATIVE = (AND, OR, XOR, ADD, MUL)


def _combine(slot, a, b, mask):
    """Element-wise operator on behaviour tuples (baseline.py:70-85)."""
    if slot == NOT:
        return tuple(x ^ mask for x in a)
    if slot == NEG:
        return tuple((-x) & mask for x in a)
    f = {AND: lambda x, y: x & y, OR: lambda x, y: x | y, XOR: lambda x, y: x ^ y,
         ADD: lambda x, y: (x + y) & mask, SUB: lambda x, y: (x - y) & mask,
         MUL: lambda x, y: (x * y) & mask}[slot]
    return tuple(f(x, y) for x, y in zip(a, b))


def candidates(size, cache, k, pairs, mask):
    """Candidates of one size in the reference's order (baseline.py:180-204):
    yields (behaviour, tokens)."""
    if size == 1:
        for i in range(k):
            yield tuple(x[i] for x, _ in pairs), (i,)
        return
    for slot in range(8):
        tok = -(slot + 1)
        if slot in (NOT, NEG):
            for beh, toks in cache[size - 1]:
                yield _combine(slot, beh, None, mask), toks + (tok,)
            continue
        top = (size - 1) // 2 if slot in COMMUTATIVE else size - 2
        for j in range(1, top + 1):
            for lb, lt in cache[j]:
                for rb, rt in cache[size - 1 - j]:
                    yield _combine(slot, lb, rb, mask), lt + rt + (tok,)


def vfb(k, w, pairs, size_bound, memory_budget=2_500_000_000):
    """-> dict(status, size, tokens, oom_at, rows=[(size, stored, stored_cum, candidates)]).

    status: "found" | "not_found" | "oom_aborted" (no time budget here)."""
    mask = (1 << w) - 1
    target = tuple(y for _, y in pairs)
    per = len(pairs) * w // 8
    cache = {s: [] for s in range(1, size_bound + 1)}
    known = set()
    total = 0
    rows = []
    for s in range(1, size_bound + 1):
        seen_here = 0
        new_here = 0
        end = None
        for beh, toks in candidates(s, cache, k, pairs, mask):
            seen_here += 1
            if beh == target:
                end = ("found", toks)
                break
            if beh in known:
                continue
            if (total + 1) * per > memory_budget:
                end = ("oom_aborted", None)
                break
            known.add(beh)
            cache[s].append((beh, toks))
            new_here += 1
            total += 1
        rows.append((s, new_here, total, seen_here))
        if end is not None:
            if end[0] == "found":
                return dict(status="found", size=s, tokens=end[1], oom_at=None, rows=rows)
            return dict(status="oom_aborted", size=None, tokens=None, oom_at=s, rows=rows)
    return dict(status="not_found", size=None, tokens=None, oom_at=None, rows=rows)
