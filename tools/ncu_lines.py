"""Warp-stall samples per CUDA source line (interleaved cuda,sass source page).

python tools/ncu_lines.py <report.ncu-rep> [top] [column]

column: "stall" (default, warp-stall samples) or "inst" (warp instructions executed)
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
col = sys.argv[3] if len(sys.argv) > 3 else "stall"
col_name = {"stall": "Warp Stall Sampling (All Samples)", "inst": "Instructions Executed"}[col]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = {}
cur_file = None
hdr = None
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ai = r.index(col_name)
        continue
    if hdr is None or len(r) <= ai or not r[0].isdigit():
        continue
    try:
        v = float(r[ai] or 0)
    except ValueError:  # a source line whose quotes broke the CSV
        continue
    key = (cur_file, int(r[0]), r[1].strip()[:100])
    agg[key] = agg.get(key, 0.0) + v
tot = sum(agg.values()) or 1
for (f, ln, src), v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100 * v / tot:5.1f}%  {f}:{ln}  {src}")
