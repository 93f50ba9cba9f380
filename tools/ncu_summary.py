"""Summarise ncu outputs: a launch list (CSV of gpu__time_duration) and/or a --set full report.

python tools/ncu_summary.py --launches gpurun_out/X_launches.csv
python tools/ncu_summary.py --report gpurun_out/X_prof.ncu-rep
"""
import argparse
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__occupancy_limit_shared_mem",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "smsp__inst_executed_op_shared_ld.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard", "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
    "smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct", "smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct",
    "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct", "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
    "smsp__warp_issue_stalled_wait_per_warp_active.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    tot = 0.0
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")[:70]
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
        tot += v
    out = [f"{'kernel':70s} {'launches':>8s} {'total_us':>12s} {'share':>6s}"]
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:70s} {c:8d} {v:12.1f} {100 * v / tot:5.1f}%")
    qk = ("qprep", "window", "scanprep", "nodescan", "itemscan", "leafscan", "lbscan", "candcheck", "filter", "refine", "finalize")
    qagg = {k: cv for k, cv in agg.items() if any(x in k for x in qk)}
    qtot = sum(v for _, v in qagg.values()) or 1
    out.append("")
    out.append("# query step only (kernels of isax_nn1; the build kernels above run once)")
    out.append(f"{'kernel':70s} {'launches':>8s} {'total_us':>12s} {'share':>6s}")
    for k, (c, v) in sorted(qagg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:70s} {c:8d} {v:12.1f} {100 * v / qtot:5.1f}%")
    return "\n".join(out)


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        out.append(f"kernel: {r[h.index('Kernel Name')]}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                out.append(f"  {k} = {r[i]} {units[i]}")
    return "\n".join(out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--report")
    a = ap.parse_args()
    if a.launches:
        print(launches(a.launches))
    if a.report:
        print(report(a.report))


def details(path):
    """Section name / metric / value lines of the details page (stall reasons, occupancy, ...)."""
    raw = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    si, mi, ui, vi = h.index("Section Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    return "\n".join(f"  [{r[si]}] {r[mi]} = {r[vi]} {r[ui]}" for r in rows[1:] if len(r) > vi)


def stalls(path, top=25):
    """Per-source-line warp stall samples (needs -lineinfo and --import-source)."""
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    return raw[:20000]
