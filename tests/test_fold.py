"""The tile engine's predicate fold is an identity of the test.

CPU part: a restatement of fold_affine / fold_outer / fold_p (simba.cu) checked
exhaustively against brute force at small word widths -- every segment chain
of up to three ancestors over all operand values, every output value, every
candidate value.  The CUDA code is the product; this pins the algebra it
implements.  GPU part: exhaustive satisfying counts on random specs across
widths 1..64 (always/never fold states, partial masks, even multipliers)
against the CPU oracle on the same ranks.
"""

import itertools
import random

import pytest

AND, OR, XOR, ADD, SUB, MUL, NOT, NEG = range(8)


def seg_of(op, s, w):
    """Fixed-left-operand ancestor as (m, x, a, b): v -> a*((v & m) ^ x) + b."""
    M = (1 << w) - 1
    return {AND: (s, 0, 1, 0), OR: (~s & M, s, 1, 0), XOR: (M, s, 1, 0), ADD: (M, 0, 1, s),
            SUB: (M, 0, M, s), MUL: (M, 0, s, 0), NOT: (M, M, 1, 0), NEG: (M, 0, M, 0)}[op]


def seg_apply(g, v, w):
    m, x, a, b = g
    return (a * ((v & m) ^ x) + b) & ((1 << w) - 1)


def is_low(tm):
    return tm & (tm + 1) == 0


def fold_affine(a, b, tm, tc, w):
    M = (1 << w) - 1
    if tc & ~tm:
        return 0, 1
    d = (tc - b) & tm
    if a & tm == 0:
        return 0, d
    t = (a & -a).bit_length() - 1
    if d & ((1 << t) - 1):
        return 0, 1
    tm >>= t
    o = (a >> t) & M
    inv = pow(o, -1, 1 << w) if o & 1 else None
    return tm, ((d >> t) * inv) & tm


def fold_outer(segs, y0, w):
    """segs in application order (innermost first); returns (tm, tc, nres)."""
    tm, tc = (1 << w) - 1, y0
    for i in range(len(segs) - 1, -1, -1):
        m, x, a, b = segs[i]
        aff = not (a == 1 and b == 0)
        if aff and not is_low(tm):
            return tm, tc, i + 1
        if aff:
            tm, tc = fold_affine(a, b, tm, tc, w)
        tc ^= x & tm
        tm &= m
    return tm, tc, 0


def fold_p(op, f, f_left, tm, tc, w):
    M = (1 << w) - 1
    if op == AND:
        return tm & f, tc
    if op == OR:
        return tm & ~f & M, tc ^ (f & tm)
    if op == XOR:
        return tm, tc ^ (f & tm)
    if op == ADD:
        a, b = 1, f
    elif op == SUB:
        a, b = (M, f) if f_left else (1, (-f) & M)
    else:
        a, b = f, 0
    return fold_affine(a, b, tm, tc, w)


def passes(tm, tc, v):
    return (v & tm) ^ tc == 0


@pytest.mark.parametrize("w", [1, 2, 3])
def test_fold_outer_is_exact(w):
    """For every chain of up to 3 ancestors (operators x fixed operands), every
    target y0 and every value v: folded test on the residual's output ==
    (chain(v) == y0)."""
    M = (1 << w) - 1
    ops = [AND, OR, XOR, ADD, SUB, MUL, NOT, NEG]
    for depth in (1, 2, 3):
        for chain_ops in itertools.product(ops, repeat=depth):
            operand_sets = [range(M + 1) if op not in (NOT, NEG) else [0] for op in chain_ops]
            for operands in itertools.product(*operand_sets):
                segs = [seg_of(op, s, w) for op, s in zip(chain_ops, operands)]  # innermost first
                for y0 in range(M + 1):
                    tm, tc, nres = fold_outer(segs, y0, w)
                    for v in range(M + 1):
                        want = v
                        for g in segs:
                            want = seg_apply(g, want, w)
                        got = v
                        for g in segs[:nres]:
                            got = seg_apply(g, got, w)
                        assert passes(tm, tc, got) == (want == y0), (chain_ops, operands, y0, v)


@pytest.mark.parametrize("w", [1, 2, 3, 4])
def test_fold_p_is_exact(w):
    """P with one operand fixed folded under every low-bit (tm, tc) reachable
    from a full fold: ((v & m) ^ c) == 0 iff P(...) passes (tm, tc)."""
    M = (1 << w) - 1
    states = {(M, y) for y in range(M + 1)} | {((1 << j) - 1, y & ((1 << j) - 1)) for j in range(w + 1)
                                               for y in range(M + 1)} | {(0, 1), (0, 0)}
    for op in (AND, OR, XOR, ADD, SUB, MUL):
        for f in range(M + 1):
            for left in (True, False):
                for tm, tc in states:
                    if op in (ADD, SUB, MUL) and not is_low(tm):
                        continue
                    m, c = fold_p(op, f, left, tm, tc, w)
                    for v in range(M + 1):
                        lhs, rhs = (f, v) if left else (v, f)
                        val = {AND: lhs & rhs, OR: lhs | rhs, XOR: lhs ^ rhs, ADD: lhs + rhs,
                               SUB: lhs - rhs, MUL: lhs * rhs}[op] & M
                        assert passes(m, c, v) == passes(tm, tc, val), (op, f, left, tm, tc, v)


def test_bitwise_fold_under_partial_masks():
    """AND/OR/XOR fold under any (non-low) mask, the case that leaves
    arithmetic ancestors as a residual chain."""
    w, M = 4, 15
    for tm in range(M + 1):
        for tc in range(M + 1):
            for op in (AND, OR, XOR):
                for f in range(M + 1):
                    m, c = fold_p(op, f, True, tm, tc, w)
                    for v in range(M + 1):
                        val = {AND: f & v, OR: f | v, XOR: f ^ v}[op]
                        assert passes(m, c, v) == passes(tm, tc, val)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(12))
def test_random_spec_counts_match_oracle(seed):
    """Exhaustive satisfying counts and first ranks on random specs (planted
    or random outputs) across widths, against the CPU oracle."""
    import oracle as O
    import paper_2605_08243_b200 as S

    rng = random.Random(1000 + seed)
    w = [1, 2, 3, 5, 8, 13, 16, 24, 32, 33, 48, 64][seed]
    k = rng.choice([1, 2, 3, 4]) if w > 2 else rng.choice([1, 2])
    n = rng.choice([1, 2, 3, 5, 10])
    size = {1: 9, 2: 8, 3: 7, 4: 7}[k]
    tab = O.OracleTable(k, size)
    xs, seen = [], set()
    while len(xs) < min(n, (1 << (k * w)) if k * w < 20 else n):
        x = tuple(rng.getrandbits(w) for _ in range(k))
        if x not in seen:
            seen.add(x)
            xs.append(x)
    planted = rng.random() < 0.5
    target = O.decode(tab, rng.randrange(tab.total(size)), size) if planted else None
    pairs = [(x, O.eval_tokens(list(target), list(x), w) if planted else rng.getrandbits(w)) for x in xs]
    spec = S.Specification(k=k, w=w, pairs=tuple(pairs))
    got = S.count_solutions(spec, S.build(k, size), S.EngineConfig(size_bound=size))
    for c in got:
        _, cnt, first, _ = O.scan_range(tab, k, w, pairs, c.size, 0, tab.total(c.size), 0, tab.total(c.size),
                                        threads=O.cpu_count())
        assert (c.count, c.first_rank) == (cnt, first), (w, k, n, c.size)
