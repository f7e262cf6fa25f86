"""C4-stress size-9 exhaustive count (diagnostics for ncu)."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_08243_b200 as S
from paper_2605_08243_b200.engine import DeviceContext
counts = json.loads((Path(__file__).resolve().parents[1] / "tests" / "golden" / "counts.json").read_text())
r = [r for r in counts if r["name"] == "C4_stress_i0"][0]
d = r["spec"]
spec = S.Specification(k=d["k"], w=d["w"], pairs=tuple((tuple(i), o) for i, o in d["pairs"]))
with DeviceContext(spec, 9) as ctx:
    for s in (9, 9):
        x = ctx.count(s)
        print(s, x.count, x.kernel_ms, x.ex0_hits, ctx.info(), flush=True)
