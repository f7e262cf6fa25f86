"""C3/C4 exhaustive-count throughput under kernel configurations (diagnostics)."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_08243_b200 as S
from paper_2605_08243_b200.engine import DeviceContext

counts = json.loads((Path(__file__).resolve().parents[1] / "tests" / "golden" / "counts.json").read_text())
def spec_of(d):
    return S.Specification(k=d["k"], w=d["w"], pairs=tuple((tuple(i), o) for i, o in d["pairs"]))
configs = [dict(), dict(block_threads=512, r0=5), dict(block_threads=256)]
for name in ("C4_stress_i0", "dense_k3_w64_stress", "C3_unsat777"):
    r = [r for r in counts if r["name"] == name][0]
    spec = spec_of(r["spec"])
    for kw in configs:
        try:
            with DeviceContext(spec, r["size_bound"], **kw) as ctx:
                ctx.count(r["size_bound"])
                tot, kms, cnt = 0, 0.0, []
                for s in range(1, r["size_bound"] + 1):
                    x = ctx.count(s)
                    tot += x.visited; kms += x.kernel_ms; cnt.append(x.count)
                ok = cnt == [c for _, c, _ in r["per_size"]]
                print(name, kw, ctx.info(), f"{tot / (kms * 1e-3):.3e} cand/s {kms:.2f} ms ok={ok}", flush=True)
        except Exception as e:
            print(name, kw, "ERR", e, flush=True)
