#!/usr/bin/env python
"""Summarise an ncu report of one kernel: headline metrics and, per
barrier/exit-delimited SASS segment, the share of samples and instructions
and the top stall reasons. Usage: python tools/ncu_segments.py REPORT"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(det)))
h = r[0]
keys = ["Duration", "DRAM Throughput", "L1/TEX Cache Throughput", "Issue Slots Busy", "No Eligible",
        "Warp Cycles Per Issued Instruction", "Achieved Active Warps Per SM", "Issued Instructions",
        "Theoretical Occupancy"]
for row in r[1:]:
    d = dict(zip(h, row))
    if d.get("Metric Name") in keys:
        print(f"{d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(src)))
h = r[1]
rows = r[2:]
iS, iE, iSrc = h.index("# Samples"), h.index("Instructions Executed"), h.index("Source")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tS = sum(int(x[iS]) for x in rows) or 1
tE = sum(int(x[iE]) for x in rows) or 1
acc = [0, 0]
st = dict.fromkeys(cols, 0)
for i, x in enumerate(rows):
    s = x[iSrc].strip()
    acc[0] += int(x[iS])
    acc[1] += int(x[iE])
    for c in cols:
        st[c] += int(x[h.index(c)] or 0)
    if any(k in s for k in ("BAR.SYNC", "EXIT", "TRYWAIT")) or i == len(rows) - 1:
        if acc[0] > 0.005 * tS:
            top = sorted(st.items(), key=lambda t: -t[1])[:4]
            print(f"{i:5d} {s[:30]:30s} samples {100 * acc[0] / tS:5.1f}% inst {100 * acc[1] / tE:5.1f}%  " +
                  " ".join(f"{c[6:]}={v}" for c, v in top))
        acc = [0, 0]
        st = dict.fromkeys(cols, 0)
