"""Warp-stall reasons of the kernel in an ncu --set full report: average warps per issue slot in
each state (smsp__average_warps_issue_stalled_*_per_issue_active). python tools/ncu_stalls.py <report>"""
import csv, io, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, r = rows[0], rows[2]
out = []
for i, k in enumerate(h):
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
        out.append((float(r[i]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
tot = sum(v for v, _ in out)
for v, k in sorted(out, reverse=True)[:10]:
    print(f"{v:6.2f} ({100 * v / tot:4.1f}%)  {k}")
