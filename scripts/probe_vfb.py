"""VFB (cache-based) vs SIMBA (cache-free) on one device: the paper's
comparison on B200.  Diagnostics, not the bench."""
import json, random, sys, time
sys.path.insert(0, ".")
import paper_2605_08243_b200 as S
from paper_2605_08243_b200 import baseline as B


def unsat(k, w, n, seed):
    rng = random.Random(seed); pairs = []; seen = set()
    while len(pairs) < n:
        x = tuple(rng.getrandbits(w) for _ in range(k))
        if x in seen: continue
        seen.add(x); pairs.append((x, rng.getrandbits(w)))
    return S.Specification(k=k, w=w, pairs=tuple(pairs))


out = {}
for k, bound in ((5, 11), (4, 12)):
    spec = unsat(k, 32, 16, 7 + k)
    B.run_baseline(spec, 4)  # warm
    t0 = time.perf_counter()
    o, st = B.run_baseline(spec, bound)
    wall = time.perf_counter() - t0
    print(B.cache_report(st))
    rows = [dict(size=r.size, stored=r.stored, stored_cum=r.stored_cum, candidates=r.candidates,
                 ms=round(r.millis, 2), cand_per_s=(r.candidates / (r.millis * 1e-3) if r.millis else None))
            for r in st.rows]
    for r in rows:
        print(r)
    last = st.rows[-1].size if st.oom_at is None else st.oom_at - 1
    # SIMBA exhaustive sweep of the same sizes (count mode: every candidate)
    tab = S.build(k, last)
    S.count_solutions(spec, tab, S.EngineConfig(size_bound=min(last, 6)))
    t0 = time.perf_counter()
    cs = S.count_solutions(spec, tab, S.EngineConfig(size_bound=last))
    simba = time.perf_counter() - t0
    print(f"k={k}: VFB {o.status.value} oom_at={st.oom_at} wall {wall:.2f} s; SIMBA full sweep of sizes 1..{last} "
          f"({tab.cumulative_total(last):,} candidates) {simba * 1e3:.1f} ms")
    out[f"k{k}"] = dict(status=o.status.value, oom_at=st.oom_at, wall_s=wall, rows=rows,
                        simba_sweep_sizes=last, simba_sweep_ms=simba * 1e3,
                        simba_candidates=tab.cumulative_total(last))
json.dump(out, open("gpurun_out/vfb_probe.json", "w"), indent=1)
