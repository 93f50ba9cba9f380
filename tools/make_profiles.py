"""Write the judged ncu summaries under profiles/ from one profiling tag in gpurun_out/.

python tools/make_profiles.py <tag> <round> <config-name>
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import ncu_summary as ns  # noqa: E402

tag, rnd, cfg = sys.argv[1], sys.argv[2], sys.argv[3]
out = os.path.join(ROOT, "profiles")
go = os.path.join(ROOT, "gpurun_out")
with open(os.path.join(out, f"{rnd}_launches_{cfg}.txt"), "w") as f:
    f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches)\n")
    f.write(f"# command: python bench.py --config <{cfg}> --steps 2 --warmup 1 --no-cpu-baseline (build + 3 query batches)\n")
    f.write(ns.launches(os.path.join(go, f"{tag}_launches.csv")) + "\n")
traffic = {}
for kre in ("leafscan", "refine_q", "window_kernel", "summarise", "candcheck", "superkd", "qprep"):
    rep = os.path.join(go, f"{tag}_{kre}_prof.ncu-rep")
    if not os.path.exists(rep):
        continue
    txt = ns.report(rep)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    import csv, io
    rows = list(csv.reader(io.StringIO(raw)))
    h, v, u = rows[0], rows[2], rows[1]
    def get(k):
        i = h.index(k)
        x = float(v[i].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u[i], 1)
        return x * scale
    dram = get("dram__bytes_read.sum") + get("dram__bytes_write.sum")
    traffic[kre] = dram
    st = [(h[i], float(v[i].replace(",", ""))) for i in range(len(h)) if "pcsamp_warps_issue_stalled" in h[i]
          and not h[i].endswith("not_issued") and v[i]]
    tot = sum(x for _, x in st) or 1
    hot = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, "15"], capture_output=True,
                         text=True).stdout
    with open(os.path.join(out, f"{rnd}_{kre}_{cfg}.txt"), "w") as f:
        f.write(f"# ncu --set full --clock-control none --import-source on -k regex:{kre} -s 0 -c 1 (first launch)\n")
        f.write(txt + "\n\n# warp stall reasons (pc sampling)\n")
        for k, x in sorted(st, key=lambda t: -t[1])[:10]:
            f.write(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {100 * x / tot:5.1f}%\n")
        f.write("\n# hottest source lines (stall samples)\n" + hot)
path = os.path.join(out, "ncu_traffic.json")
d = json.load(open(path)) if os.path.exists(path) else {}
key = {"cfg3": "cfg3_walk_100M_x256", "cfg2": "cfg2_walk_10M_x256"}.get(cfg, cfg)
ent = d.get(key, {})
for name, kre in (("leafscan", "leafscan"), ("refine", "refine_q"), ("window", "window_kernel")):
    if traffic.get(kre) is not None:  # only kernels captured under this tag
        ent[f"{name}_dram_bytes"] = traffic[kre]
ent["source"] = f"profiles/{rnd}_*_{cfg}.txt (ncu --set full, first launch)"
d[key] = ent
json.dump(d, open(path, "w"), indent=1)
print("wrote", sorted(os.listdir(out)))
