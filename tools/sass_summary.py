#!/usr/bin/env python
"""Opcode histogram per kernel of libdqmc.so + stripped SASS of the hot kernels.
usage: python tools/sass_summary.py profiles/<round>_sass_summary.md profiles/<round>_sass_hot_kernels.txt"""
import collections
import os
import re
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(REPO, "paper_2302_10083_b200", "libdqmc.so")
HOT = ("k_strided_pipe<3, 3>", "k_merge_reduce_pipe<3, 3>", "k_c0_final<7, false>", "k_c0_final<7, true>", "k_sp_generate")
KEYS = ["LOP3", "SHF", "LDS", "STS", "LDG", "STG", "UTMALDG", "UTMASTG", "UBLKCP", "LDGSTS", "SYNCS", "POPC",
        "SHFL", "BAR", "IMAD", "IADD3", "ATOMG", "REDG"]


def main():
    if len(sys.argv) != 3 or not all(a.endswith((".md", ".txt")) for a in sys.argv[1:]):
        sys.exit("usage: sass_summary.py <out>.md <out>.txt (outputs only; reads libdqmc.so)")
    txt = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", txt)
    out = ["# SASS evidence (cuobjdump -sass paper_2302_10083_b200/libdqmc.so, sm_100a)", "",
           "Static opcode counts per kernel. TMA: UTMALDG/UTMASTG (cp.async.bulk.tensor), UBLKCP",
           "(cp.async.bulk), SYNCS.* (mbarrier); bit-slice math: LOP3.LUT, SHF (funnel shifts). No tensor-core",
           "opcodes: the path is pure bitwise streaming.", ""]
    hot = []
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        dem = dem.replace("(anonymous namespace)::", "")
        ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*(?:\.[A-Z0-9_]+)*)", f)
        c = collections.Counter(o.split(".")[0] for o in ops)
        out.append(f"## `{dem}`\n\ninstructions: {len(ops)}; " + ", ".join(f"{k} {c[k]}" for k in KEYS if c[k]))
        tma = sorted({o for o in ops if o.startswith(("UTMA", "UBLK", "LDGSTS", "SYNCS"))})
        if tma:
            out.append("\nasync/TMA opcodes: " + ", ".join(f"`{t}`" for t in tma))
        out.append("")
        if any(h in dem for h in HOT):
            body = re.sub(r"\s*/\* 0x[0-9a-f]+ \*/", "", f)
            hot.append("Function : " + dem + "\n" + re.sub(r"[ \t]+\n", "\n", body.split("\n", 1)[1]))
    with open(sys.argv[1], "w") as fh:
        fh.write("\n".join(out))
    with open(sys.argv[2], "w") as fh:
        fh.write("\n".join(hot))


if __name__ == "__main__":
    main()
