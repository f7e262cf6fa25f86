"""Generate golden vectors for the SIMBA hot path from the UNMODIFIED reference.

Test infrastructure only.  Run in the build container (where /root/reference
exists) with:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the reference package ``mbasynth`` read-only and writes small JSON
fixtures next to this script.  The GPU box never runs this script: the tests
only read the committed JSON.

What is pinned (reference file:line in brackets):
  tables.json   counting.build rows/cumulative           [counting.py:88-128]
  decode.json   codec.decode of chosen / random ranks      [codec.py:89-144]
                plus a digest of every decode at small (k, s)
  eval.json     expr.evaluate on decoded expressions        [expr.py:146-198]
  search.json   engine.synthesize outcomes (status, size, rank, tokens, per-size
                visited counts) for configs C1..C4          [engine.py:190-276]
  counts.json   exhaustive satisfying counts per size (and min rank per size)
                assembled from Decoder.decode_into + eval_tokens, the reference's
                own primitives (the reference has no count mode),
                and rank windows at C5 sizes 11..13          [engine.py:128-156]
"""

from __future__ import annotations

import hashlib
import json
import multiprocessing as mp
import os
import random
import sys
import time
from pathlib import Path

from mbasynth import bench, codec, counting
from mbasynth.codec import Decoder, decode
from mbasynth.engine import EngineConfig, Specification, synthesize
from mbasynth.expr import eval_tokens, evaluate, parse_infix

HERE = Path(__file__).resolve().parent


# ---------------------------------------------------------------------------
# spec helpers (all inputs drawn with the reference's own generators)
# ---------------------------------------------------------------------------

def spec_json(spec: Specification) -> dict:
    return {"k": spec.k, "w": spec.w, "pairs": [[list(i), o] for i, o in spec.pairs]}


def random_output_spec(k, w, n, seed, low_first=0):
    """Random-output spec in the style of test_acceptance.py:278-289."""
    rng = random.Random(seed)
    pairs, seen = [], set()
    while len(pairs) < n:
        if len(pairs) < low_first:
            inputs = tuple(rng.randrange(4) for _ in range(k))
        else:
            inputs = tuple(rng.getrandbits(w) for _ in range(k))
        if inputs in seen:
            continue
        seen.add(inputs)
        pairs.append((inputs, rng.getrandbits(w)))
    return Specification(k=k, w=w, pairs=tuple(pairs))


def stress_spec_for_target(target, k, seed, n=100, w=64, low_first=16):
    """C4 'stress' variant: the first 16 examples draw inputs from {0..3}."""
    rng = random.Random(seed)
    pairs, seen = [], set()
    while len(pairs) < n:
        if len(pairs) < low_first:
            inputs = tuple(rng.randrange(4) for _ in range(k))
        else:
            inputs = tuple(rng.getrandbits(w) for _ in range(k))
        if inputs in seen:
            continue
        seen.add(inputs)
        pairs.append((inputs, evaluate(target, inputs, w)))
    return Specification(k=k, w=w, pairs=tuple(pairs))


def dense_spec(k, w, n, seed, size):
    """Target-derived spec at a tiny width: example-0 matches are frequent,
    which stresses the hit path (many satisfying candidates per window)."""
    rng = random.Random(seed)
    table = counting.build(k, size)
    target = codec.sample_uniform(size, table, rng)
    return bench.spec_for_target(target, k, rng, n=n, w=w)


def c1_spec(seed):
    target = parse_infix("(x0 ^ x1) + ((x0 & x1) + (x0 & x1))", 2)
    return bench.spec_for_target(target, 2, random.Random(seed), n=4, w=8)


def c2_spec(size, idx, table):
    rng = random.Random(1000 * size + idx)
    target = codec.sample_uniform(size, table, rng)
    return target, bench.spec_for_target(target, 2, rng, n=10, w=32)


def c3_spec(idx, table, w=32, n=10, size=9):
    rng = random.Random(3000 + idx)
    target = codec.sample_uniform(size, table, rng)
    return target, bench.spec_for_target(target, 3, rng, n=n, w=w)


# ---------------------------------------------------------------------------
# workers
# ---------------------------------------------------------------------------

def run_search(args):
    name, spec_d, C, meta = args
    spec = Specification(k=spec_d["k"], w=spec_d["w"],
                         pairs=tuple((tuple(i), o) for i, o in spec_d["pairs"]))
    table = counting.build(spec.k, C)
    t0 = time.perf_counter()
    out = synthesize(spec, table, EngineConfig(size_bound=C))
    dt = time.perf_counter() - t0
    return {
        "name": name, "spec": spec_d, "size_bound": C, "meta": meta,
        "status": out.status.value,
        "size": out.size, "rank": out.rank,
        "tokens": list(out.expr.tokens) if out.expr is not None else None,
        "per_size": [[s.size, s.candidates] for s in out.stats],
        "ref_seconds": round(dt, 3),
    }


def count_range(spec, table, size, lo, hi, want_hits=False):
    """#{n in [lo,hi) : check(decode(n,size))} using the reference primitives
    Decoder.decode_into (codec.py:89) and eval_tokens (expr.py:157), exactly the
    body of _scan_range (engine.py:144-155) with a counter instead of min."""
    dec = Decoder(table)
    mask = (1 << spec.w) - 1
    pairs = spec.pairs
    stack = [0] * (size // 2 + 2)
    count, first, hits = 0, None, []
    for n in range(lo, hi):
        buf = dec.decode_into(n, size)
        for inputs, output in pairs:
            if eval_tokens(buf, size, inputs, mask, stack) != output:
                break
        else:
            count += 1
            if first is None:
                first = n
            if want_hits and len(hits) < 4096:
                hits.append(n)
    return count, first, hits


def run_counts(args):
    name, spec_d, C, meta = args
    spec = Specification(k=spec_d["k"], w=spec_d["w"],
                         pairs=tuple((tuple(i), o) for i, o in spec_d["pairs"]))
    table = counting.build(spec.k, C)
    per = []
    t0 = time.perf_counter()
    for s in range(1, C + 1):
        c, first, _ = count_range(spec, table, s, 0, table.total(s))
        per.append([s, c, first])
    return {"name": name, "spec": spec_d, "size_bound": C, "meta": meta,
            "per_size": per, "ref_seconds": round(time.perf_counter() - t0, 3)}


def run_window(args):
    name, spec_d, C, size, lo, hi, meta = args
    spec = Specification(k=spec_d["k"], w=spec_d["w"],
                         pairs=tuple((tuple(i), o) for i, o in spec_d["pairs"]))
    table = counting.build(spec.k, C)
    c, first, hits = count_range(spec, table, size, lo, hi, want_hits=True)
    return {"name": name, "spec": spec_d, "size_bound": C, "size": size,
            "lo": lo, "hi": hi, "count": c, "first": first, "hits": hits, "meta": meta}


# ---------------------------------------------------------------------------
# fixture builders
# ---------------------------------------------------------------------------

def make_tables():
    out = []
    for k, C in [(1, 24), (2, 20), (3, 16), (4, 16), (5, 14), (6, 12), (7, 11), (8, 11), (10, 9)]:
        t = counting.build(k, C)
        out.append({"k": k, "max_size": C, "rows": [list(r) for r in t.rows],
                    "cumulative": list(t.cumulative)})
    # capacity error location (counting.py:115-117)
    try:
        counting.build(10, 60)
        cap = None
    except counting.CountCapacityError as exc:
        cap = {"k": 10, "max_size": 60, "s": exc.s, "op": exc.op}
    return {"tables": out, "capacity_error": cap}


def make_decode():
    out = {"digests": [], "samples": []}
    # Every rank at small (k, s): explicit tokens for tiny sizes, digest otherwise.
    for k, smax in [(1, 9), (2, 8), (3, 7), (4, 6)]:
        table = counting.build(k, smax)
        dec = Decoder(table)
        for s in range(1, smax + 1):
            h = hashlib.sha256()
            total = table.total(s)
            explicit = []
            for n in range(total):
                toks = dec.decode_into(n, s)[:s]
                h.update(bytes((t & 0xFF) for t in toks))
                if total <= 1200:
                    explicit.append(list(toks))
            out["digests"].append({"k": k, "s": s, "total": total,
                                   "sha256": h.hexdigest(),
                                   "tokens": explicit if explicit else None})
    rng = random.Random(20261017)
    for k, C, sizes in [(1, 24, (16, 20, 24)), (2, 16, (9, 12, 16)), (3, 14, (9, 11, 14)),
                        (4, 16, (11, 12, 13, 16)), (5, 12, (10, 12)), (8, 10, (8, 10))]:
        table = counting.build(k, C)
        for s in sizes:
            total = table.total(s)
            ranks = {0, total - 1}
            for op in range(8):
                off = table.operator_offset(s, op)
                if table.count(s, op):
                    ranks.add(off)
                    ranks.add(off + table.count(s, op) - 1)
            while len(ranks) < 64:
                ranks.add(rng.randrange(total))
            for n in sorted(ranks):
                if n >= 1 << 64:
                    continue
                out["samples"].append({"k": k, "s": s, "rank": n,
                                       "tokens": list(decode(n, s, table).tokens)})
    return out


def make_eval():
    rng = random.Random(77)
    out = []
    for w in (1, 2, 3, 8, 16, 31, 32, 33, 48, 63, 64):
        for k, C in [(1, 9), (2, 9), (3, 11), (4, 13)]:
            table = counting.build(k, C)
            for _ in range(12):
                s = rng.randrange(1, C + 1)
                e = decode(rng.randrange(table.total(s)), s, table)
                inputs = tuple(rng.getrandbits(w) for _ in range(k))
                out.append({"w": w, "k": k, "tokens": list(e.tokens),
                            "inputs": list(inputs), "value": evaluate(e, inputs, w)})
    return out


def search_tasks():
    tasks = []
    # C1: deobfuscate (x^y)+2*(x&y) -> x+y; k=2, w=8, n=4, C=5; seeds 0..99
    for seed in range(100):
        tasks.append((f"C1_seed{seed}", spec_json(c1_spec(seed)), 5, {"config": "C1", "seed": seed}))
    # C2: k=2, w=32, n=10, uniform targets at s=3..7 (10 each), C=7
    t2 = counting.build(2, 7)
    for s in range(3, 8):
        for i in range(10):
            target, spec = c2_spec(s, i, t2)
            tasks.append((f"C2_s{s}_i{i}", spec_json(spec), 7,
                          {"config": "C2", "target": list(target.tokens)}))
    # C3: k=3, w=32, n=10, size-9 targets (10), plus one unsat random-output spec
    t3 = counting.build(3, 9)
    for i in range(10):
        target, spec = c3_spec(i, t3)
        tasks.append((f"C3_i{i}", spec_json(spec), 9, {"config": "C3", "target": list(target.tokens)}))
    tasks.append(("C3_unsat777", spec_json(random_output_spec(3, 32, 10, 777)), 9,
                  {"config": "C3", "unsat": True}))
    # C4: k=3, w=64, n=100, size-9 targets: uniform and low-entropy 'stress' prefix
    for i in range(5):
        target, spec = c3_spec(100 + i, t3, w=64, n=100)
        tasks.append((f"C4_uniform_i{i}", spec_json(spec), 9,
                      {"config": "C4", "dist": "uniform", "target": list(target.tokens)}))
    for i in range(5):
        rng = random.Random(4000 + i)
        target = codec.sample_uniform(9, t3, rng)
        spec = stress_spec_for_target(target, 3, 4100 + i)
        tasks.append((f"C4_stress_i{i}", spec_json(spec), 9,
                      {"config": "C4", "dist": "stress", "target": list(target.tokens)}))
    tasks.append(("C4_unsat", spec_json(random_output_spec(3, 64, 100, 4242)), 9,
                  {"config": "C4", "unsat": True}))
    # small engine-test style instances (test_engine.py:33-77)
    tasks.append(("and_k2", spec_json(bench.spec_for_target(parse_infix("x0 & x1", 2), 2,
                                                            random.Random(0), n=16)), 3, {}))
    return tasks


def count_tasks():
    tasks = []
    for seed in range(10):
        tasks.append((f"C1_seed{seed}", spec_json(c1_spec(seed)), 5, {"config": "C1"}))
    t2 = counting.build(2, 7)
    for s in (5, 7):
        for i in range(2):
            _, spec = c2_spec(s, i, t2)
            tasks.append((f"C2_s{s}_i{i}", spec_json(spec), 7, {"config": "C2"}))
    t3 = counting.build(3, 9)
    _, spec = c3_spec(0, t3)
    tasks.append(("C3_i0", spec_json(spec), 9, {"config": "C3"}))
    tasks.append(("C3_unsat777", spec_json(random_output_spec(3, 32, 10, 777)), 9, {"config": "C3"}))
    # dense-hit specs: tiny widths make example-0 matches frequent (hit-path stress)
    tasks.append(("dense_k3_w3_n2", spec_json(random_output_spec(3, 3, 2, 5)), 9, {"dense": True}))
    tasks.append(("dense_k2_w2_n3", spec_json(dense_spec(2, 2, 3, 6, 5)), 9, {"dense": True}))
    rng = random.Random(4000)
    target = codec.sample_uniform(9, t3, rng)
    tasks.append(("C4_stress_i0", spec_json(stress_spec_for_target(target, 3, 4100)), 9,
                  {"config": "C4", "dist": "stress"}))
    rng = random.Random(4001)
    target = codec.sample_uniform(7, t3, rng)
    tasks.append(("dense_k3_w64_stress", spec_json(stress_spec_for_target(target, 3, 8, n=4, low_first=4)), 9,
                  {"dense": True}))
    return tasks


def window_tasks():
    tasks = []
    rng = random.Random(555)
    t4 = counting.build(4, 13)
    for s in (11, 12, 13):
        for i in range(3):
            total = t4.total(s)
            trank = rng.randrange(total)
            target = decode(trank, s, t4)
            spec = bench.spec_for_target(target, 4, random.Random(9000 + 10 * s + i), n=10, w=32)
            lo = max(0, trank - 40000)
            hi = min(total, trank + 40000)
            tasks.append((f"C5_s{s}_t{i}", spec_json(spec), 13, s, lo, hi,
                          {"config": "C5", "target_rank": trank}))
        # operator-block boundaries with a dense spec (many hits, ragged units)
        dense = spec_json(dense_spec(4, 4, 3, 100 + s, 7))
        for op in range(1, 8):
            off = t4.operator_offset(s, op)
            tasks.append((f"C5dense_s{s}_op{op}", dense, 13, s, max(0, off - 20000),
                          min(t4.total(s), off + 20000), {"dense": True}))
    # k=4 w=32 n=10 window near the end of the size-13 level
    total = t4.total(13)
    spec = spec_json(random_output_spec(4, 32, 10, 31337))
    tasks.append(("C5_unsat_tail", spec, 13, 13, total - 50000, total, {"config": "C5"}))
    # k=1 long sizes and k=5 (more variables than the common configs)
    t1 = counting.build(1, 20)
    tasks.append(("k1_s20_dense", spec_json(dense_spec(1, 3, 2, 11, 6)), 20, 20, 123456, 123456 + 60000, {}))
    t5 = counting.build(5, 11)
    tasks.append(("k5_s11_dense", spec_json(dense_spec(5, 3, 3, 12, 6)), 11, 11,
                  t5.total(11) // 3, t5.total(11) // 3 + 60000, {}))
    return tasks


def main():
    t0 = time.time()
    (HERE / "tables.json").write_text(json.dumps(make_tables()))
    (HERE / "decode.json").write_text(json.dumps(make_decode()))
    (HERE / "eval.json").write_text(json.dumps(make_eval()))
    print(f"tables/decode/eval written in {time.time() - t0:.1f}s", flush=True)
    procs = int(os.environ.get("GOLDEN_PROCS", os.cpu_count() or 1))
    with mp.get_context("fork").Pool(procs) as pool:
        wins = pool.map_async(run_window, window_tasks(), chunksize=1)
        counts = pool.map_async(run_counts, count_tasks(), chunksize=1)
        search = pool.map_async(run_search, search_tasks(), chunksize=1)
        (HERE / "search.json").write_text(json.dumps(search.get()))
        print(f"search written {time.time() - t0:.1f}s", flush=True)
        (HERE / "counts.json").write_text(json.dumps(counts.get()))
        print(f"counts written {time.time() - t0:.1f}s", flush=True)
        (HERE / "windows.json").write_text(json.dumps(wins.get()))
        print(f"windows written {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    sys.setrecursionlimit(10000)
    main()
