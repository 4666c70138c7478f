#!/usr/bin/env python3
"""Hottest source lines (warp-stall samples, top stall reasons) of an ncu report
captured with --import-source on.  usage: ncu_source_hot.py REPORT [N] [file-substring] [inst]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
filt = sys.argv[3] if len(sys.argv) > 3 else ""
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
H = None
fname = None
out = []
for r in csv.reader(txt.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        H = r
        continue
    if not H or len(r) < 5 or r[0] == "":
        continue
    m = r[-(len(H) - 4):]            # metric columns, counted from the right (source text may hold quotes)
    out.append((fname, int(r[0]), r[1][:60], m))
Hm = H[4:]
st = Hm.index("Warp Stall Sampling (All Samples)")
ie = Hm.index("Instructions Executed")
reasons = [h for h in Hm if h.startswith("stall_") and "Not Issued" not in h]


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


tot = sum(num(m[st]) for *_, m in out)
print("total stall samples", tot)
key = ie if (len(sys.argv) > 4 and sys.argv[4] == "inst") else st     # sort by stall samples or instructions
rows = sorted([o for o in out if filt in o[0]], key=lambda o: -num(o[3][key]))[:N]
for fn, ln, t, m in rows:
    s = num(m[st])
    rs = sorted(((num(m[Hm.index(k)]), k[6:]) for k in reasons), reverse=True)[:3]
    print(f"{fn}:{ln:4d} {100 * s / max(tot, 1):5.1f}% inst {num(m[ie]):9d} {rs} | {t}")
