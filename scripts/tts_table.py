"""Summarise probe_tts logs with '== label' sections: median / max per size
of each target's best repeat after the first (usage: tts_table.py log)."""
import re
import statistics
import sys

cur, res = None, {}
for line in open(sys.argv[1]):
    if line.startswith("=="):
        cur = line[2:].strip()
        res.setdefault(cur, {})
        continue
    m = re.match(r"(s(\d+)_\S+) (.*)", line)
    if not m or cur is None:
        continue
    ms = [float(x) for x in re.findall(r"([\d.]+)ms\(", m.group(3))]
    res[cur].setdefault(m.group(2), []).append(min(ms[1:] or ms))
for label, d in res.items():
    print(f"{label:60s}", "  ".join(f"s{s}: {statistics.median(v):6.2f} / {max(v):6.2f}" for s, v in sorted(d.items())))
