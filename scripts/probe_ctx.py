"""Context creation and synthesize latency of small configs (C2, C4 golden
specs): where a sub-millisecond search spends its time (diagnostics)."""
import json
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2605_08243_b200 as S  # noqa: E402
from paper_2605_08243_b200.engine import DeviceContext  # noqa: E402

search = json.loads((ROOT / "tests" / "golden" / "search.json").read_text())
for cfg in ("C2", "C4"):
    r = [r for r in search if r["meta"].get("config") == cfg][0]
    spec = S.Specification(k=r["spec"]["k"], w=r["spec"]["w"], pairs=tuple((tuple(i), o) for i, o in r["spec"]["pairs"]))
    C = r["size_bound"]
    table = S.build(spec.k, C)
    S.synthesize(spec, table, S.EngineConfig(size_bound=C))
    cre, syn, raw = [], [], []
    for _ in range(20):
        t0 = time.perf_counter()
        ctx = DeviceContext(spec, C)
        t1 = time.perf_counter()
        o = ctx.synthesize_raw(C)
        t2 = time.perf_counter()
        ctx.close()
        cre.append((t1 - t0) * 1e3)
        raw.append((t2 - t1) * 1e3)
        t0 = time.perf_counter()
        S.synthesize(spec, table, S.EngineConfig(size_bound=C))
        syn.append((time.perf_counter() - t0) * 1e3)
    print(f"{cfg}: create {statistics.median(cre):.3f} ms, synthesize_raw {statistics.median(raw):.3f} ms "
          f"(device {o.kernel_ms:.3f} ms, {o.launches} launches), engine.synthesize {statistics.median(syn):.3f} ms",
          flush=True)
