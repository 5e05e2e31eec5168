#!/usr/bin/env python
"""Per-SASS-instruction stall samples of one kernel in an ncu report, grouped
into the regions between barriers (BAR/SYNCS waits). Read here, no GPU.
usage: python tools/ncu_stalls.py report.ncu-rep kernel_substring [top]"""
import csv
import io
import subprocess
import sys

rep, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kname}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
i0 = starts[0]
hdr = rows[i0 + 1]
end = starts[1] if len(starts) > 1 else len(rows)
data = [r for r in rows[i0 + 2:end] if len(r) == len(hdr)]
isrc = hdr.index("Source")
iss = hdr.index("Warp Stall Sampling (All Samples)")
iex = hdr.index("Instructions Executed")
tot = sum(int(r[iss]) for r in data) or 1
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ridx = [hdr.index(h) for h in reasons]


def why(rs):
    acc = [0] * len(ridx)
    for r in rs:
        for k, j in enumerate(ridx):
            acc[k] += int(r[j] or 0)
    t = sum(acc) or 1
    return " ".join(f"{reasons[k][6:]}:{100 * acc[k] // t}" for k in sorted(range(len(acc)), key=lambda k: -acc[k])[:3])

print(rows[i0][1][:100], "| samples", tot, "| sass", len(data))
seg, acc, acc_ex, start = [], 0, 0, 0
for i, r in enumerate(data):
    acc += int(r[iss])
    acc_ex += int(r[iex] or 0)
    s = r[isrc]
    if "BAR.SYNC" in s or "BAR.ARV" in s or "SYNCS.PHASECHK" in s or i == len(data) - 1:
        seg.append((start, i, acc, acc_ex, s.strip()[:40]))
        start, acc, acc_ex = i + 1, 0, 0
print("segments (start..end, % samples, warp-instr executed, closing op):")
for a, b, s, ex, op in seg:
    if s > tot * 0.01:
        print(f"  {a:5d}..{b:5d} {100 * s / tot:5.1f}%  {ex:12d}  {op}  [{why(data[a:b + 1])}]")
print("top instructions:")
for i, r in sorted(enumerate(data), key=lambda x: -int(x[1][iss]))[:top]:
    print(f"  {i:5d} {100 * int(r[iss]) / tot:5.1f}%  {r[isrc].strip()[:60]}  [{why([r])}]")
