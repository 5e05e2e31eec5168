#!/usr/bin/env python
"""Summarise an ncu report (read here, no GPU): per-kernel time, DRAM bytes,
throughputs, issue/stall metrics -> profiles/ncu_summary.json + a markdown table.

usage: python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/<round>_ncu_full.md [n]
"""

import csv
import io
import json
import os
import re
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "launch__registers_per_thread",
    "launch__occupancy_limit_shared_mem",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "Tbyte": 1e12}


def short(name: str) -> str:
    m = re.search(r"(k_[a-z0-9_]+)(<[^>]*>)?", name)
    if not m:
        return name
    base = m.group(1)
    tmpl = m.group(2) or ""
    if base == "k_merge_reduce_pipe":
        return "k_strided<MERGE_REDUCE>"
    if base == "k_strided_pipe":  # pass D (reduce-only since round 2)
        return "k_strided<REDUCE>"
    if base == "k_strided":  # pass B (merge-only since round 2)
        return "k_strided<MERGE_ONLY>"
    return base


def main():
    rep, md = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 24
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = {"report": os.path.basename(rep), "n": n, "kernels": {}}
    lines = ["| kernel | ms | DRAM read GB | DRAM write GB | DRAM % peak | issue % | warps % | inst (warp) | regs |",
             "|---|---|---|---|---|---|---|---|---|"]
    for r in rows[2:]:
        name = short(r[hdr.index("Kernel Name")])
        vals = {}
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                v *= SCALE.get(units[i], 1.0)
                if units[i] == "ms":
                    pass
                elif units[i] == "us":
                    v /= 1e3
                elif units[i] == "ns":
                    v /= 1e6
                vals[w] = v
        dram = vals.get("dram__bytes_read.sum", 0) + vals.get("dram__bytes_write.sum", 0)
        out["kernels"][name] = {"n": n, "ms": vals.get("gpu__time_duration.sum"), "dram_bytes": dram, **vals}
        lines.append(
            f"| {name} | {vals.get('gpu__time_duration.sum', 0):.3f} | {vals.get('dram__bytes_read.sum', 0)/1e9:.2f} | "
            f"{vals.get('dram__bytes_write.sum', 0)/1e9:.2f} | {vals.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
            f"{vals.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):.1f} | "
            f"{vals.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):.1f} | "
            f"{vals.get('smsp__inst_executed.sum', 0):.3g} | {vals.get('launch__registers_per_thread', 0):.0f} |"
        )
    if "--no-json" not in sys.argv:  # the table bench.py reads its roofline traffic from
        with open(os.path.join(os.path.dirname(md) or ".", "ncu_summary.json"), "w") as fh:
            json.dump(out, fh, indent=1)
    with open(md, "w") as fh:
        fh.write(f"# ncu --set full summary ({os.path.basename(rep)}, n={n})\n\n")
        fh.write("Captured with `ncu --set full --clock-control none --import-source on` on one B200 ")
        fh.write("(`tools/run_once.py` or `tools/run_sparse_once.py`), one launch per kernel; per-launch values (cold-cache, serialised).\n\n")
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
