"""C5 goldens on the production paths, computed by the multithreaded CPU oracle.

Test infrastructure only.  Runs on the GPU box (whose host has the cores for
1.1e11-candidate oracle sweeps):

    python tests/golden/make_c5_golden.py --out gpurun_out/c5.json

and the result is committed as tests/golden/c5.json.  Inputs come from
tests/golden/c5_candidates.json (drawn with the unmodified reference by
make_c5_candidates.py).  Every number written here is the ORACLE's
(oracle/simba_oracle.c: decode_into + eval_tokens + _scan_range restated,
pinned to the reference's own goldens by tests/test_oracle_golden.py):

  planted[i].levels   per level s = 1..13: exhaustive satisfying count and the
                      first satisfying rank (enumerate_all + check,
                      engine.py:279-293, expr.py:201-218)
  tts[s]              ten suite instances per size s = 11, 12, 13 whose minimal
                      solution size is s: Alg. 1's (size, rank, tokens)
                      (engine.py:190-276, local order), plus the oracle's own
                      time-to-solve on this host

The GPU is used only to choose which suite instances to verify (an instance
whose device answer is below its generated size is skipped); the device's
answer for every chosen instance is recorded beside the oracle's, and a
mismatch is reported (and fails the run).
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import oracle as O  # noqa: E402

C = 13
PER_SIZE = 10
CHUNK = 1 << 30


def pairs_of(sp):
    return [(tuple(i), o) for i, o in sp["pairs"]]


def level_sweep(tab, sp, threads, log):
    k, w, pairs = sp["k"], sp["w"], pairs_of(sp)
    out = []
    for s in range(1, C + 1):
        t0 = time.perf_counter()
        total = tab.total(s)
        cnt, first = 0, None
        for a in range(0, total, CHUNK * 8):
            v, c, b, _ = O.scan_range(tab, k, w, pairs, s, 0, total, a, min(total, a + CHUNK * 8), threads=threads)
            assert v == min(total, a + CHUNK * 8) - a
            cnt += c
            if b is not None and first is None:
                first = b
        out.append({"size": s, "candidates": total, "count": cnt, "first": first})
        log(f"  level {s}: {total} candidates, count {cnt}, first {first} ({time.perf_counter() - t0:.1f}s)")
    return out


def oracle_search(tab, sp, bound, threads):
    """Alg. 1 (engine.py:190-276, local order): the first level with a hit,
    its minimum rank.  Chunks ascend, so the first chunk with a hit holds the
    minimum."""
    k, w, pairs = sp["k"], sp["w"], pairs_of(sp)
    visited = []
    for s in range(1, bound + 1):
        total = tab.total(s)
        vis = 0
        for a in range(0, total, CHUNK):
            b = min(total, a + CHUNK)
            v, _, best, toks = O.scan_range(tab, k, w, pairs, s, 0, total, a, b, threads=threads)
            vis += v
            if best is not None:
                visited.append(vis)
                return {"status": "found", "size": s, "rank": best, "tokens": list(toks), "visited": visited}
        visited.append(vis)
    return {"status": "not_found", "size": None, "rank": None, "tokens": None, "visited": visited}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "c5.json"))
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--skip-planted", action="store_true")
    ap.add_argument("--sizes", default="11,12,13")
    args = ap.parse_args()
    threads = args.threads or O.cpu_count()
    cand = json.loads((ROOT / "tests" / "golden" / "c5_candidates.json").read_text())
    out_path = Path(args.out)
    out_path.parent.mkdir(parents=True, exist_ok=True)
    res = {"threads": threads, "generator": "make_c5_golden.py (oracle/simba_oracle.c, multithreaded)",
           "inputs": "c5_candidates.json", "planted": [], "tts": {}, "mismatches": []}
    if out_path.exists():
        res = json.loads(out_path.read_text())

    def save():
        out_path.write_text(json.dumps(res, indent=1) + "\n")

    def log(msg):
        print(msg, flush=True)

    tab = O.OracleTable(4, C)
    if not args.skip_planted:
        done = {p["name"] for p in res["planted"]}
        for p in cand["planted"]:
            if p["name"] in done:
                continue
            log(f"planted {p['name']}")
            t0 = time.perf_counter()
            lv = level_sweep(tab, p["spec"], threads, log)
            res["planted"].append({"name": p["name"], "spec": p["spec"], "target": p["target"], "levels": lv,
                                   "oracle_s": round(time.perf_counter() - t0, 1)})
            save()

    import paper_2605_08243_b200 as S

    table = S.build(4, C)
    for gs in [int(x) for x in args.sizes.split(",")]:
        chosen = res["tts"].setdefault(str(gs), [])
        seen = {c["id"] for c in chosen}
        skipped = res.setdefault("skipped", {}).setdefault(str(gs), [])
        for inst in cand["suite"]:
            if len(chosen) >= PER_SIZE:
                break
            if inst["gen_size"] != gs or inst["id"] in seen or inst["id"] in {x[0] for x in skipped}:
                continue
            sp = inst["spec"]
            spec = S.Specification(k=sp["k"], w=sp["w"], pairs=tuple(pairs_of(sp)))
            g = S.synthesize(spec, table, S.EngineConfig(size_bound=gs))
            if g.size != gs:
                skipped.append([inst["id"], g.size])
                save()
                continue
            t0 = time.perf_counter()
            o = oracle_search(tab, sp, gs, threads)
            dt = time.perf_counter() - t0
            dev = {"status": g.status.value, "size": g.size, "rank": g.rank,
                   "tokens": list(g.expr.tokens) if g.expr else None}
            rec = {"id": inst["id"], "gen_size": gs, "spec": sp, "target": inst["target"],
                   "oracle": o, "oracle_s": round(dt, 2), "device": dev}
            if (o["status"], o["size"], o["rank"], o["tokens"]) != (dev["status"], dev["size"], dev["rank"],
                                                                     dev["tokens"]):
                res["mismatches"].append(rec)
                log(f"MISMATCH {inst['id']}: oracle {o} device {dev}")
            if o["size"] == gs:
                chosen.append(rec)
            else:
                skipped.append([inst["id"], o["size"]])
            log(f"tts {inst['id']}: oracle size {o['size']} rank {o['rank']} ({dt:.1f}s), device {g.size} {g.rank}")
            save()
    save()
    return 1 if res["mismatches"] else 0


if __name__ == "__main__":
    sys.exit(main())
