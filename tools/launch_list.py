#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into a
markdown table of per-kernel launches, total time and share.
usage: python tools/launch_list.py launches.csv out.md "<command>" "<title>" """
import collections
import csv
import io
import re
import sys


def short(name: str) -> str:
    name = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    m = re.match(r"(?:void\s+)?([\w:]+(?:<[^()]*>)?)", name)
    return m.group(1) if m else name[:60]


def main():
    src, dst, cmd, title = sys.argv[1:5]
    text = open(src).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    ik, imn, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        if len(r) != len(hdr) or r[imn] != "gpu__time_duration.sum":
            continue
        v = float(r[iv].replace(",", ""))
        scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}[r[iu]]
        k = short(r[ik])
        tot[k] += v * scale
        cnt[k] += 1
    allms = sum(tot.values())
    out = [f"# {title}", "", f"Command: `{cmd}`", "(the same command first exited 0 without ncu). Per-launch times are cold-cache and",
           "serialised: compare SHARES with the CUDA-event pass times of the bench line.", "",
           "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k in sorted(tot, key=tot.get, reverse=True):
        out.append(f"| `{k}` | {cnt[k]} | {tot[k]:.2f} | {100 * tot[k] / allms:.1f}% |")
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main()
