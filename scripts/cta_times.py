"""Summarise CTA start/end lines: spread of start and end times (ms)."""
import re, sys
rows = [tuple(map(int, m.groups())) for m in re.finditer(r"CTA (\d+) start (\d+) end (\d+) phases (\d+) dry (\d+)", open(sys.argv[1]).read())]
t0 = min(r[1] for r in rows)
st = sorted((r[1] - t0) / 1e6 for r in rows)
en = sorted((r[2] - t0) / 1e6 for r in rows)
ph = sorted(r[3] for r in rows)
q = lambda a, f: a[min(len(a) - 1, int(f * len(a)))]
print(f"CTAs {len(rows)} start max {st[-1]:.3f} ms; end min {en[0]:.3f} p10 {q(en,.1):.3f} p50 {q(en,.5):.3f} p90 {q(en,.9):.3f} max {en[-1]:.3f}; phases {ph[0]}..{ph[-1]}")
dry = sorted((r[4] - t0) / 1e6 for r in rows)
print(f"first dry claim per CTA: min {dry[0]:.3f} p50 {q(dry,.5):.3f} max {dry[-1]:.3f} ms")
ext = [tuple(map(int, m.groups())) for m in re.finditer(
    r"CTA (\d+) start \d+ end (\d+) phases \d+ dry \d+ plan_max (\d+) at (\d+) exec_max (\d+) at (\d+) q (\d+)", open(sys.argv[1]).read())]
if ext:
    for name, i in (("plan", 2), ("exec", 4)):
        top = sorted(ext, key=lambda r: -r[i])[:4]
        print(f"longest {name} parts (ms, at ms, CTA end ms, queue):",
              [(round(r[i] / 1e6, 3), round((r[i + 1] - t0) / 1e6, 3), round((r[1] - t0) / 1e6, 3), r[6]) for r in top])
    last = sorted(ext, key=lambda r: -r[1])[:4]
    print("last CTAs (end ms, plan_max ms at, exec_max ms at, q):",
          [(round((r[1] - t0) / 1e6, 3), round(r[2] / 1e6, 3), round((r[3] - t0) / 1e6, 3), round(r[4] / 1e6, 3), round((r[5] - t0) / 1e6, 3), r[6]) for r in last])
