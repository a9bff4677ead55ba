"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_summary.py launches.csv "<command>" > summary.json
"""
import csv
import io
import json
import sys

path, command = sys.argv[1], sys.argv[2]
lines = [ln for ln in open(path) if ln.startswith('"')]
rows = list(csv.reader(io.StringIO("".join(lines))))
h = rows[0]
kn, mn, mv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
agg = {}
for r in rows[1:]:
    if r[mn] != "gpu__time_duration.sum":
        continue
    name = r[kn].split("(")[0]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += float(r[mv].replace(",", "")) / 1e6
tot = sum(v[1] for v in agg.values()) or 1.0
out = {"command": command, "launches": sum(v[0] for v in agg.values()),
       "note": "cold-cache, serialised per-launch times: compare shares, not absolutes",
       "kernels": {k: {"launches": v[0], "total_ms": round(v[1], 3), "share": round(v[1] / tot, 4)}
                   for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}}
json.dump(out, sys.stdout, indent=1)
print()
