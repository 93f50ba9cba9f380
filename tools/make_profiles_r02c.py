"""Write the round-2c profile summaries under profiles/ from gpurun_out/r02c_* (tools/profile_round2c.sh).

python tools/make_profiles_r02c.py
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import ncu_summary as ns  # noqa: E402

GO, OUT, T = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles"), "r02c"


def run(*a):
    return subprocess.run([sys.executable, *a], capture_output=True, text=True).stdout


def dram(rep, idx=0):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2 + idx]

    def get(k):
        i = h.index(k)
        return float(v[i].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u[i], 1)
    return get("dram__bytes_read.sum") + get("dram__bytes_write.sum")


def summary(rep, name, how):
    txt = f"# {how}\n# report: {os.path.basename(rep)}\n\n" + ns.report(rep) + "\n"
    txt += "\n# warp states per issue slot (smsp__average_warps_issue_stalled_*_per_issue_active)\n"
    txt += run(os.path.join(ROOT, "tools", "ncu_stalls.py"), rep)
    txt += "\n# basic blocks by warp instructions executed (offset, length x executions = share)\n"
    txt += run(os.path.join(ROOT, "tools", "ncu_sass_counts.py"), rep)
    txt += "\n# hottest source lines (warp stall samples)\n" + run(os.path.join(ROOT, "tools", "ncu_lines.py"), rep, "14")
    with open(os.path.join(OUT, name), "w") as f:
        f.write(txt)


for c in (1, 2, 3, 4, 5):
    src = os.path.join(GO, f"{T}_bench_cfg{c}.json")
    if os.path.exists(src) and os.path.getsize(src):
        shutil.copy(src, os.path.join(OUT, f"{T}_bench_cfg{c}.json"))
for c in (3, 5):
    p = os.path.join(GO, f"{T}_launches_cfg{c}.csv")
    if os.path.exists(p):
        with open(os.path.join(OUT, f"{T}_launches_cfg{c}.txt"), "w") as f:
            f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches)\n")
            f.write(f"# command: python bench.py --config {c} --steps 2 --warmup 3 --no-cpu-baseline (build + query batches)\n")
            f.write(ns.launches(p) + "\n")
p = os.path.join(GO, f"{T}_build_launches_cfg2.csv")
if os.path.exists(p):
    with open(os.path.join(OUT, f"{T}_build_cfg2.txt"), "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none: python tools/time_build.py --config 2 --reps 1\n")
        f.write(ns.launches(p) + "\n\n# python tools/time_build.py --config 2 --reps 3 (CUDA events, no profiler)\n")
        f.write(open(os.path.join(GO, f"{T}_build_cfg2.txt")).read())
        b3 = os.path.join(GO, f"{T}_build_cfg3.txt")
        if os.path.exists(b3):
            f.write("\n# python tools/time_build.py --config 3 --reps 1\n" + open(b3).read())
SCAN = "ncu --set full --clock-control none --import-source on -k regex:{k} -s 2 -c 1 python tools/sweep_env.py --config {c} --steps 2 --opt first_band=-1 (third launch: a full scan, first band off)"
traffic = {}
for c in (3, 2, 5):
    rep = os.path.join(GO, f"{T}_itemscan{c}.ncu-rep")
    if os.path.exists(rep):
        summary(rep, f"{T}_itemscan_cfg{c}.txt", SCAN.format(k="itemscan", c=c))
        traffic[c] = dram(rep)
rep = os.path.join(GO, f"{T}_nodescan3.ncu-rep")
if os.path.exists(rep):
    summary(rep, f"{T}_nodescan_cfg3.txt", SCAN.format(k="nodescan", c=3))
    traffic["n3"] = dram(rep)
for k, name in (("window3", "window_kernel"), ("candcheck3", "candcheck")):
    rep = os.path.join(GO, f"{T}_{k}.ncu-rep")
    if os.path.exists(rep):
        summary(rep, f"{T}_{name}_cfg3.txt",
                f"ncu --set full --clock-control none --import-source on -k regex:{name} -s 1 -c 1 python tools/sweep_env.py --config 3 --steps 2 --opt first_band=-1")
rep = os.path.join(GO, f"{T}_refine3.ncu-rep")
if os.path.exists(rep):
    with open(os.path.join(OUT, f"{T}_refine_cfg3.txt"), "w") as f:
        f.write("# ncu --set full --clock-control none --import-source on -k regex:'refine_q|filter' -s 3 -c 3 python tools/sweep_env.py "
                "--config 3 --steps 2 --opt first_band=-1 (pass 1, filter, pass 2 of one call)\n\n" + ns.report(rep) + "\n")
    traffic["r1"], traffic["r2"] = dram(rep, 0), dram(rep, 2)
rep = os.path.join(GO, f"{T}_build2.ncu-rep")
if os.path.exists(rep):
    with open(os.path.join(OUT, f"{T}_summarise_cfg2.txt"), "w") as f:
        f.write("# ncu --set full --clock-control none --import-source on -k regex:'summarise_tma|superkd' -c 2 python tools/time_build.py --config 2 --reps 1\n\n")
        f.write(ns.report(rep) + "\n\n# warp states per issue slot\n" + run(os.path.join(ROOT, "tools", "ncu_stalls.py"), rep))
        f.write("\n# hottest source lines (warp stall samples; first kernel)\n" + run(os.path.join(ROOT, "tools", "ncu_lines.py"), rep, "12"))
path = os.path.join(OUT, "ncu_traffic.json")
d = json.load(open(path)) if os.path.exists(path) else {}
names = {3: "cfg3_walk_100M_x256", 2: "cfg2_walk_10M_x256"}  # (cfg5 is captured with the first band off: not the bench's launch)
for c, nm in names.items():
    if c in traffic:
        e = d.setdefault(nm, {})
        e["leafscan_dram_bytes"] = traffic[c] + (traffic.get("n3", 0) if c == 3 else 0)
        e["itemscan_dram_bytes"] = traffic[c]
        e["source"] = f"profiles/{T}_itemscan_cfg{c}.txt (ncu --set full); refine from profiles/{T}_refine_cfg3.txt or r02"
if "r1" in traffic:
    e = d["cfg3_walk_100M_x256"]
    e["refine_pass1_dram_bytes"], e["refine_pass2_dram_bytes"] = traffic["r1"], traffic["r2"]
    e["refine_dram_bytes"] = traffic["r1"] + traffic["r2"]
if "n3" in traffic:
    d["cfg3_walk_100M_x256"]["nodescan_dram_bytes"] = traffic["n3"]
json.dump(d, open(path, "w"), indent=1)
print(sorted(x for x in os.listdir(OUT) if x.startswith(T)))
