#!/usr/bin/env python3
"""Per-kernel summary of an ncu --metrics gpu__time_duration.sum --csv launch list.
usage: launch_summary.py launches.csv [frames]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
frames = float(sys.argv[2]) if len(sys.argv) > 2 else None
hdr = None
data = collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            v = float(d["Metric Value"]) * (1000.0 if d.get("Metric Unit") == "us" else 1.0)
            data[d["Kernel Name"].split("(")[0][:60]].append(v)
tot = sum(sum(v) for v in data.values())
for k, v in sorted(data.items(), key=lambda kv: -sum(kv[1])):
    line = f"{k:60s} n={len(v):3d} avg={sum(v) / len(v) / 1000:8.1f}us share={sum(v) / tot:6.3f}"
    if frames:
        line += f" per_frame={sum(v) / frames / 1000:8.1f}us"
    print(line)
