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
