"""Per-config report on one GPU: C1-C4 latency (every golden instance, checked
against the reference outcome), exhaustive-count throughput at C3/C4, C5
time-to-solve, and the RTid locality ablation (shuffled
thread ids vs the locally consistent order).  Prints one JSON document."""

import json
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2605_08243_b200 as S  # noqa: E402
from paper_2605_08243_b200.engine import DeviceContext  # noqa: E402


def spec_of(d):
    return S.Specification(k=d["k"], w=d["w"], pairs=tuple((tuple(i), o) for i, o in d["pairs"]))


def main():
    g = ROOT / "tests" / "golden"
    search = json.loads((g / "search.json").read_text())
    counts = json.loads((g / "counts.json").read_text())
    wins = json.loads((g / "windows.json").read_text())
    rep = {}
    # warm the CUDA context
    S.synthesize(spec_of(search[0]["spec"]), S.build(2, 5), S.EngineConfig(size_bound=5))
    for cfg in ("C1", "C2", "C3", "C4"):
        ms, ref_ms, ok = [], [], True
        for r in [r for r in search if r["meta"].get("config") == cfg]:
            spec = spec_of(r["spec"])
            t0 = time.perf_counter()
            o = S.synthesize(spec, S.build(spec.k, r["size_bound"]), S.EngineConfig(size_bound=r["size_bound"]))
            ms.append((time.perf_counter() - t0) * 1e3)
            ref_ms.append(r["ref_seconds"] * 1e3)
            ok &= (o.status.value, o.size, o.rank) == (r["status"], r["size"], r["rank"])
        rep[cfg] = {"instances": len(ms), "all_match_reference": ok,
                    "time_to_solve_ms": {"median": statistics.median(ms), "max": max(ms)},
                    "reference_python_1core_ms": {"median": statistics.median(ref_ms), "max": max(ref_ms)}}
    # exhaustive-count throughput (device time of the scans)
    for name in ("C3_unsat777", "C4_stress_i0", "dense_k3_w64_stress"):
        r = [r for r in counts if r["name"] == name][0]
        spec = spec_of(r["spec"])
        with DeviceContext(spec, r["size_bound"]) as ctx:
            ctx.count(r["size_bound"])
            tot, kms, cnt = 0, 0.0, []
            for s in range(1, r["size_bound"] + 1):
                x = ctx.count(s)
                tot += x.visited
                kms += x.kernel_ms
                cnt.append(x.count)
        rep[f"count_{name}"] = {"candidates": tot, "kernel_ms": kms, "cand_per_s": tot / (kms * 1e-3),
                                "counts_match_reference": cnt == [c for _, c, _ in r["per_size"]],
                                "reference_python_1core_s": r["ref_seconds"]}
    # C5 time to solve: the 30-target suite of tests/golden/c5.json (answers asserted)
    import bench

    rep["C5_time_to_solve"] = bench.time_to_solve(S, 13)["by_size"]
    # RTid ablation: one operator block at k=4 size 11, same kernel, local vs shuffled
    spec = spec_of([r for r in wins if r["name"] == "C5_s11_t0"][0]["spec"])
    t = S.build(4, 11)
    off, cnt = t.operator_offset(11, S.Op.ADD), t.count(11, S.Op.ADD)
    abl = {}
    with DeviceContext(spec, 11, kernel="direct") as ctx:
        for shuffled in (False, True):
            ctx.scan_range(11, off, cnt, 0, cnt, shuffled)
            t0 = time.perf_counter()
            res = ctx.scan_range(11, off, cnt, 0, cnt, shuffled)
            abl["shuffled" if shuffled else "local"] = {"s": time.perf_counter() - t0, "best": res[1]}
    with DeviceContext(spec, 11) as ctx:
        ctx.scan_range(11, off, cnt, 0, cnt, False)
        t0 = time.perf_counter()
        res = ctx.scan_range(11, off, cnt, 0, cnt, False)
        abl["unit_kernel_local"] = {"s": time.perf_counter() - t0, "best": res[1]}
    abl["block"] = {"size": 11, "op": "ADD", "candidates": cnt}
    abl["direct_shuffled_over_local"] = abl["shuffled"]["s"] / abl["local"]["s"]
    abl["direct_shuffled_over_unit_local"] = abl["shuffled"]["s"] / abl["unit_kernel_local"]["s"]
    abl["same_min_rank"] = abl["shuffled"]["best"] == abl["local"]["best"] == abl["unit_kernel_local"]["best"]
    rep["rtid_ablation"] = abl
    print(json.dumps(rep, indent=1))


if __name__ == "__main__":
    main()
