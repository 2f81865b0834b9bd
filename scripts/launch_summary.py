"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel totals.

    python scripts/launch_summary.py gpurun_out/launches.csv "<command>" "<note>" > profiles/<name>.json
"""
import csv, json, sys
from collections import defaultdict

path, cmd, note = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
rows = [r for r in csv.reader(open(path)) if r]
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
kn, mn, mv, un = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[hdr_i + 1:]:
    if len(r) <= mv or r[mn] != "gpu__time_duration.sum":
        continue
    v = float(r[mv].replace(",", ""))
    u = r[un]
    us = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}[u] * v
    name = r[kn][:100]
    tot[name] += us
    cnt[name] += 1
total = sum(tot.values())
ks = sorted(tot, key=lambda k: -tot[k])
print(json.dumps({"command": cmd, "tool": "ncu --metrics gpu__time_duration.sum --clock-control none "
                  "(cold-cache, serialised per launch)", "note": note, "total_us": round(total, 1),
                  "launches": sum(cnt.values()),
                  "kernels": [{"kernel": k, "launches": cnt[k], "total_us": round(tot[k], 1),
                               "share": round(tot[k] / total, 4)} for k in ks]}, indent=1))
