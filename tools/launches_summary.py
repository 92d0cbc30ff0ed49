"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel launch counts and mean durations.
usage: launches_summary.py launches.csv "<command>" > out.json"""
import csv
import json
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
h = rows[0]
iK, iM, iV, iU = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
k = OrderedDict()
for r in rows[1:]:
    if len(r) <= iV or r[iM] != "gpu__time_duration.sum":
        continue
    v = float(r[iV].replace(",", ""))
    v = {"ns": v / 1e3, "us": v, "usecond": v, "msecond": v * 1e3, "ms": v * 1e3, "nsecond": v / 1e3}[r[iU]]
    name = r[iK].split("(")[0].replace("(anonymous namespace)::", "")
    e = k.setdefault(name, {"launches": 0, "avg_us": 0.0})
    e["avg_us"] = (e["avg_us"] * e["launches"] + v) / (e["launches"] + 1)
    e["launches"] += 1
json.dump({"command": sys.argv[2] if len(sys.argv) > 2 else "", "kernels": k}, sys.stdout, indent=1)
