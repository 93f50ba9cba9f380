"""Per-source-line warp instructions executed (and stall samples) of a kernel in an ncu report.

python tools/ncu_lines_exec.py <report.ncu-rep> <source.cu> [top]
Uses the cuda,sass source view: every SASS row is attributed to the source line above it, so
inlined helpers count at their own lines. Prints the top lines and the total.
"""
import csv
import io
import subprocess
import sys

rep, src = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--resolve-source-file", src], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
per, text, stall = {}, {}, {}
tot = stot = 0.0
line = None
hdr = None
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        ei = r.index("Instructions Executed")
        wi = r.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= ei:
        continue
    if r[0]:
        line = int(r[0])
        text[line] = r[1].strip()
        continue
    if r[2] in ("...", "-"):
        continue
    v = float(r[ei] or 0)
    w = float(r[wi] or 0)
    per[line] = per.get(line, 0) + v
    stall[line] = stall.get(line, 0) + w
    tot += v
    stot += w
print(f"total warp instructions executed: {tot:.4g}; stall samples {stot:.4g}")
for ln, v in sorted(per.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100 * v / tot:5.1f}% inst {v:11.4g}  {100 * stall[ln] / max(stot, 1):5.1f}% stall  L{ln}: {text.get(ln, '')[:90]}")
