"""Top SASS instructions by warp-stall samples: python tools/ncu_hot.py <report.ncu-rep> [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
si, ai = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
data = [(r[0], r[si], float(r[ai] or 0)) for r in rows[hi + 1:] if len(r) > ai]
tot = sum(d[2] for d in data) or 1
for addr, src, v in sorted(data, key=lambda d: -d[2])[:top]:
    print(f"{100 * v / tot:5.1f}%  {addr}  {src}")
