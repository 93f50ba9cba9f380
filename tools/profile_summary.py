#!/usr/bin/env python
"""Write a judged ncu summary for every kernel of one --set full report (under profiles/).

python tools/profile_summary.py <report.ncu-rep> <out.txt> "<command that produced it>"
Per kernel: the key metrics of tools/ncu_summary.py, the warp-stall reasons (pc sampling) and,
for single-kernel reports, the basic-block instruction profile (tools/ncu_sass_counts.py).
"""
import csv
import io
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary as ns  # noqa: E402

rep, out, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
lines = [f"# {cmd}", f"# report: {os.path.basename(rep)}", ""]
for r in rows[2:]:
    lines.append(f"kernel: {r[h.index('Kernel Name')]}")
    for k in ns.KEYS:
        if k in h:
            i = h.index(k)
            lines.append(f"  {k} = {r[i]} {units[i]}")
    st = [(h[i], float(r[i].replace(",", ""))) for i in range(len(h)) if "pcsamp_warps_issue_stalled" in h[i]
          and not h[i].endswith("not_issued") and r[i]]
    tot = sum(x for _, x in st) or 1
    lines.append("  warp stall reasons (pc sampling):")
    for k, x in sorted(st, key=lambda t: -t[1])[:8]:
        lines.append(f"    {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * x / tot:5.1f}%")
    lines.append("")
if len(rows) == 3:
    blk = subprocess.run([sys.executable, os.path.join(os.path.dirname(os.path.abspath(__file__)), "ncu_sass_counts.py"), rep],
                         capture_output=True, text=True).stdout
    lines.append("# basic blocks by warp instructions executed (offset, length x executions = share)")
    lines.append(blk)
open(out, "w").write("\n".join(lines) + "\n")
print(open(out).read()[:3000])
