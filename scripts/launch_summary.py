"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into profiles/.

usage: python scripts/launch_summary.py gpurun_out/launches.csv profiles/name.json "command"
"""
import csv
import json
import sys
from collections import OrderedDict


def main(src, dst, command):
    rows = [r for r in csv.reader(l for l in open(src) if l.startswith('"'))]
    hdr, rows = rows[0], rows[1:]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    per = [{"kernel": r[ik][:60], "ns": float(r[iv].replace(",", ""))} for r in rows]
    tot = sum(p["ns"] for p in per) or 1.0
    agg = OrderedDict()
    for p in per:
        a = agg.setdefault(p["kernel"], {"kernel": p["kernel"], "count": 0, "total_ns": 0.0})
        a["count"] += 1
        a["total_ns"] += p["ns"]
    for a in agg.values():
        a["share"] = a["total_ns"] / tot
    out = {"command": command, "note": "cold-cache serialised per-launch times; compare shares, not absolutes",
           "launches": list(agg.values()), "per_launch": per}
    json.dump(out, open(dst, "w"), indent=1)
    for a in agg.values():
        print(f"{a['count']:4d} {a['total_ns']/1e6:10.3f} ms {100*a['share']:6.2f}%  {a['kernel']}")


if __name__ == "__main__":
    main(*sys.argv[1:4])
