"""Dump (offset, SASS, warp instructions executed) of the kernel in an ncu report, and print the
execution-count profile in blocks: python tools/ncu_sass_counts.py <report> [--dump]"""
import csv, io, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
ei, si = h.index("Instructions Executed"), h.index("Source")
data = []
for r in rows[hi + 1:]:
    if len(r) <= ei:
        continue
    try:
        a = int(r[0], 16)
    except ValueError:
        continue
    data.append((a, r[si].strip(), float(r[ei] or 0)))
base = data[0][0]
tot = sum(d[2] for d in data)
print(f"total {tot:.4g}")
if "--dump" in sys.argv:
    for a, s, v in data:
        print(f"{a - base:6x} {int(v):10d}  {s}")
else:
    # runs of equal execution count = basic blocks
    cur, start, acc, n = None, 0, 0.0, 0
    out = []
    for a, s, v in data:
        if v != cur:
            if cur is not None and acc > 0.004 * tot:
                out.append((start, n, cur, acc))
            cur, start, acc, n = v, a - base, 0.0, 0
        acc += v
        n += 1
    if acc > 0.004 * tot:
        out.append((start, n, cur, acc))
    for st, n, c, acc in out:
        print(f"{st:6x} {n:4d} instr x {int(c):9d} = {100 * acc / tot:5.1f}%")
