#!/usr/bin/env python
"""bench.py: exact 1-NN queries/sec of the iSAX path on BASELINE.json's workloads.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl isax|reference]

What one step is: one batch of Q queries answered end to end by
the query path a6-a10 (query PAA/SAX/LUT, window BSF, full LB scan plus compaction, refine,
finalise) on an index built before the timed region. The build (a1-a5) is timed on its own
and reported under "build". At N=1 the workload is config 3 (100M x 256, the metric's
config). `value` is queries/s over all ranks. For N>1 every rank holds a replica of the
index and answers its own query batch, with no data-path collective (weak scaling;
DESIGN.md "Multi-GPU").

Extra keys: roofline (the dominant kernel, lbscan, timed live with CUDA events on its
stream), cpu_baseline (the oracle on this host's cores, on a bounded sample), e2e (the same
metric through isax_nn1 with host buffers, copies included), gpu_launches and clocks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "exact 1-NN queries/sec on 100M×256 fp32 series; scan/refine HBM GB/s vs peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3, help="BASELINE.json config 1..5 (3 = the metric's)")
    ap.add_argument("--impl", default="isax", choices=["isax", "reference"])
    ap.add_argument("--queries", type=int, default=0, help="override Q per step")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="budget of the oracle cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--stats-out", default="")
    ap.add_argument("--opt", action="append", default=[],
                    help="index option key=value (isax_opts field, e.g. probe_L=128); default: the library's")
    return ap.parse_args()


# ------------------------------------------------------------------------------------ clocks
REASONS = ["gpu_idle", "applications_clocks_setting", "sw_power_cap", "hw_slowdown", "sync_boost",
           "sw_thermal_slowdown", "hw_thermal_slowdown", "hw_power_brake_slowdown"]


class ClockSampler:
    """nvidia-smi sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, dev: int):
        self.dev = dev
        self.rows = []
        self.proc = None

    def start(self):
        q = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active"
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        for r in self.rows:
            p = [x.strip() for x in r.split(",")]
            if len(p) < 4:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
                mask = int(p[3], 16)
            except ValueError:
                continue
            for b, name in enumerate(REASONS):
                if mask & (1 << b) and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ------------------------------------------------------------------------------------ oracle
def cpu_baseline(wl, q_dev, budget_s: float, rank: int, series: int = 0):
    """The oracle (C7 brute force, oracle/oracle.c, OpenMP on all host cores) on a bounded sample.

    Sample: the first S dataset series (streamed from the device generator in 1M-series chunks,
    copied to host; copies excluded from the timing) against the first 4 queries. S is `series`
    if given, else it grows chunk by chunk until the oracle has spent ~budget_s seconds.
    queries/s for the whole workload = 4 / (t * N / S).
    """
    import torch

    import datagen
    from oracle import clib

    qh = q_dev[:4].cpu().numpy()
    qy, _, _, _, _ = clib.summarise(qh, want_paa=False)
    sc = clib.NN1Scan(qy, K=32)
    chunk = 1 << 20
    buf = torch.empty((chunk, wl.n), dtype=torch.float32, device="cuda")
    host = torch.empty((chunk, wl.n), dtype=torch.float32, pin_memory=True)
    t_or, S = 0.0, 0
    limit = min(series, wl.N) if series else wl.N
    while S < limit and (series or t_or < budget_s):
        c = min(chunk, limit - S)
        datagen.series(wl, S, c, out=buf[:c])
        host[:c].copy_(buf[:c])
        t0 = time.perf_counter()
        sc.feed(S, host[:c].numpy())
        t_or += time.perf_counter() - t0
        S += c
    qps = 4.0 / (t_or * wl.N / S)
    return {"value": qps, "unit": "queries/s", "cores": clib.num_threads(), "kind": "oracle", "series": S,
            "seconds": t_or,
            "sample": f"brute-force exact 1-NN (oracle C7) of 4 queries over the first {S} of {wl.N} series "
                      f"({t_or:.2f} s); scaled to the full collection"}


# ------------------------------------------------------------------------------------ main
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch

    import datagen

    wl = datagen.WORKLOADS[args.config]
    if args.impl == "reference":
        return run_reference(args, wl, world, rank, local)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2009_01614_b200 import isax

    from paper_2009_01614_b200 import dist as pdist

    Q = args.queries or wl.Q
    opts = {k: (float(v) if "." in v else int(v)) for k, v in (o.split("=", 1) for o in args.opt)}
    wlq = pdist.rank_workload(wl, rank)  # replicas: every rank answers its own queries
    # ---- build (a1-a5), timed on its own
    free, _ = torch.cuda.mem_get_info()
    raw_bytes = wl.N * wl.n * 4
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if 2 * raw_bytes + (8 << 30) < free:
        x = datagen.series(wl, 0, wl.N)
        torch.cuda.synchronize()
        ev0.record()
        ix = isax.Index.build(x, **opts)
        ev1.record()
        torch.cuda.synchronize()
        build_mode = "device-resident input"
        del x
        torch.cuda.empty_cache()
    else:
        fptr, ctx = datagen.fill_callback(wl)
        ev0.record()
        ix = isax.Index.build_stream(wl.N, wl.n, fptr, ctx, **opts)
        ev1.record()
        torch.cuda.synchronize()
        build_mode = "streamed input (generator fill callback, 2 passes; generation time included)"
    build_s = ev0.elapsed_time(ev1) / 1e3
    q, src = datagen.queries(wlq, Q)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    # ---- warmup
    for _ in range(max(args.warmup, 0)):
        ids, dist_ = ix.nn1(q)
    torch.cuda.synchronize()
    # ---- timed: K steps on the device, bracketed by barrier + synchronize
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # each step is one isax_nn1_async call on preallocated device buffers (the C ABI entry point
    # with its arguments marshalled once, so Python overhead stays out of the device timeline)
    ids = torch.empty(Q, dtype=torch.int64, device="cuda")
    dist_ = torch.empty(Q, dtype=torch.float32, device="cuda")
    step = ix.nn1_bound(q, ids, dist_, stream.cuda_stream)
    e_start.record(stream)
    for _ in range(args.steps):
        step()
    e_end.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    if dist:
        dist.barrier()
    ms = pdist.max_over_ranks(e_start.elapsed_time(e_end), device="cuda")
    value = pdist.aggregate_qps(Q, args.steps, world, ms)
    # ---- per-kernel times and counters: a separate pass of the same steps (stats() is host
    # work, kept out of the timed region). The library times its first batch with CUDA events
    # on the stream its kernels run on.
    keys = ["lbscan", "candcheck", "refine", "refine1", "filter", "refine2", "window", "qprep"]
    kms = {k: [] for k in keys}
    cand, refined, abandoned, skipped, winrows, rounds, scan_b, ref_b, pairs, launches = [], [], [], [], [], [], [], [], [], 0
    ref1_b, ref2_b, lookups_dev = [], [], []
    for _ in range(args.steps):
        ids, dist_ = ix.nn1(q)
        st = ix.stats()
        for k in keys:
            kms[k].append(st["ms_first_batch"][k])
        cand.append(sum(st["candidates"]))
        refined.append(sum(st["refined"]))
        abandoned.append(sum(st["abandoned"]))
        skipped.append(sum(st.get("skipped", [0])))
        winrows.append(sum(st["window_rows"]))
        rounds.append(max(st["rounds"]))
        launches += st.get("launches", 0)
        scan_b.append(st["scan_bytes_first_launch"])
        ref_b.append(st["refine_bytes_first_launch"])
        ref1_b.append(st["refine1_bytes_first_launch"])
        ref2_b.append(st["refine2_bytes_first_launch"])
        pairs.append(st["leaf_pairs_first_launch"])
        lookups_dev.append(st.get("scan_lookups_first_launch", 0))
    # ---- e2e through isax_nn1 with host (pinned) buffers, copies inside the timed region
    qh = torch.empty((Q, wl.n), dtype=torch.float32, pin_memory=True)
    qh.copy_(q)
    oid = torch.empty(Q, dtype=torch.int64, pin_memory=True)
    odist = torch.empty(Q, dtype=torch.float32, pin_memory=True)
    ix.nn1_host(qh.numpy(), oid.numpy(), odist.numpy())
    if dist:
        dist.barrier()
    e2e_steps = max(1, min(args.steps, 10))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        ix.nn1_host(qh.numpy(), oid.numpy(), odist.numpy())
    e2e_s = pdist.max_over_ranks(time.perf_counter() - t0, device="cuda")
    assert (oid.numpy() == ids.cpu().numpy()).all(), "host and device paths disagree"
    # ---- roofline of the dominant kernel (leafscan) and of the HBM-bound kernels
    # medians over the stats pass: the adaptive first-band policy (R15) re-times its other mode
    # now and then, and such a call's first launch is not the step's typical launch
    med = statistics.median
    hbm, peak_src = peaks()
    sm_mhz = clocks.get("sm_mhz") or 1965.0
    lb_ms = med(kms["lbscan"])
    bms = st.get("build_ms") or {}
    rf_ms = med(kms["refine"])
    nq1 = min(Q, st.get("batch_Q", 1024))  # queries of the first batch (the timed launches)
    leaf_size, super_size = st.get("leaf_size", 64), st.get("super_size", 1024)
    supers = (wl.N + super_size - 1) // super_size
    # algorithmic LUT lookups of the first scan launch, counted by the scan kernels themselves: 16
    # per node bound computed (hyper-node, super-node, leaf, 8-row cell; only under surviving
    # parents) and 16 per member of every (cell, query) pair that survived its cell bound. (The
    # round-2b kernel, -DISAX_SCAN_V1, does not count: 16 per super-node per query plus 16 per
    # member of every surviving (leaf, query) pair is used then.)
    lookups = float(med(lookups_dev)) or 16.0 * supers * nq1 + 16.0 * leaf_size * med(pairs)
    lk_peak = 148 * 32 * sm_mhz * 1e6  # one conflict-free 32-lane LDS wavefront per clock per SM
    lk_rate = lookups / (lb_ms / 1e3)
    scan_bytes = med(scan_b) + 4.0 * med(cand) * nq1 / Q
    traffic, tr = None, {}
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f).get(wl.name, {})
        traffic = tr.get("leafscan_dram_bytes")
    except Exception:
        pass
    roofline = {"kernel": "itemscan_kernel<16> (+ nodescan_kernel<16>, scanprep_kernel: the scan stage)", "bound": "alu", "achieved": round(lk_rate / 1e12, 4),
                "peak": round(lk_peak / 1e12, 4), "unit": "T LUT lookups/s", "frac": round(lk_rate / lk_peak, 4),
                "traffic": traffic,
                "peak_rule": "148 SMs x 32 lanes x SM clock (one conflict-free shared-memory wavefront per clock per SM); "
                             "DESIGN.md sec. 6",
                "lookups_per_launch": lookups, "launch_ms": round(lb_ms, 4),
                "hbm_view": {"bytes_per_launch": scan_bytes, "achieved": round(scan_bytes / (lb_ms / 1e3) / 1e9, 1),
                             "peak": hbm, "unit": "GB/s", "frac": round(scan_bytes / (lb_ms / 1e3) / 1e9 / hbm, 4),
                             "peak_source": peak_src}}
    rbytes = med(ref_b)
    r1b, r2b = med(ref1_b), med(ref2_b)
    r1_ms, f_ms, r2_ms = (med(kms[k]) for k in ("refine1", "filter", "refine2"))

    def gbs(b, ms_):
        return round(b / (ms_ / 1e3) / 1e9, 1) if ms_ > 0 else None
    # window: every row of the main window and of the kept probe windows is read once (4n B each);
    # the rows per query are the library's count (probe windows inside the main window or repeated
    # are dropped by qprep)
    wr = st.get("window_rows") or []
    win_rows = statistics.mean(wr[:nq1]) if wr else (
        min(st["window_L"], wl.N) + st.get("probe_windows", 15) * min(st.get("probe_L", 256), wl.N))
    wbytes = float(nq1) * win_rows * 4 * wl.n
    wn_ms = med(kms["window"])
    kernels = {
        "refine_q_kernel": {"bound": "hbm", "bytes_per_launch": rbytes, "launch_ms": round(rf_ms, 4),
                            "achieved": round(rbytes / (rf_ms / 1e3) / 1e9, 1), "peak": hbm, "unit": "GB/s",
                            "frac": round(rbytes / (rf_ms / 1e3) / 1e9 / hbm, 4),
                            "bytes_rule": "2n B per half row read (n float32 per row), counted by the kernel; "
                                          "launch_ms spans pass 1, filter_kernel and pass 2 (R14)",
                            "pass1": {"bytes": r1b, "ms": round(r1_ms, 4), "achieved": gbs(r1b, r1_ms),
                                      "frac": round(gbs(r1b, r1_ms) / hbm, 4) if r1_ms > 0 else None},
                            "filter_ms": round(f_ms, 4),
                            "traffic": {"pass1": tr.get("refine_pass1_dram_bytes"), "pass2": tr.get("refine_pass2_dram_bytes"),
                                        "source": "profiles/ncu_traffic.json (ncu dram read + write per launch)"},
                            "pass2": {"bytes": r2b, "ms": round(r2_ms, 4), "achieved": gbs(r2b, r2_ms),
                                      "frac": round(gbs(r2b, r2_ms) / hbm, 4) if r2_ms > 0 else None}},
        "window_kernel": {"bound": "hbm", "bytes_per_launch": wbytes, "launch_ms": round(wn_ms, 4),
                          "achieved": round(wbytes / (wn_ms / 1e3) / 1e9, 1), "peak": hbm, "unit": "GB/s",
                          "frac": round(wbytes / (wn_ms / 1e3) / 1e9 / hbm, 4),
                          "bytes_rule": "4n B per window row refined (main window and kept probe windows, the library's count); the windows of one "
                                        "query overlap (and near-duplicate queries share rows), so L2 serves part of "
                                        "it and frac can pass 1"},
        "ms_first_batch": {k: round(med(v), 4) for k, v in kms.items()},
    }
    # single-query latency: one query per call on the device path, after warm-up
    q1 = q[:1].contiguous()
    for _ in range(3):
        ix.nn1(q1)
    torch.cuda.synchronize()
    lat = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ix.nn1(q1)
        b.record(stream)
        b.synchronize()
        lat.append(a.elapsed_time(b))
    out = {
        "metric": METRIC, "value": round(value, 2), "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": wl.name, "N": wl.N, "n": wl.n, "w": 16, "card": 256, "queries_per_step": Q,
                   "queries": f"{min(Q, wl.q_walks)} random walks + {max(0, Q - wl.q_walks)} noisy copies (sigma {wl.sigma})",
                   "parallelism": f"replicas x{world} (each rank: own query batch)",
                   "l2": "inputs larger than L2 (SAX array 16N B, stored rows 4nN B)" if wl.N * 16 > 126e6
                   else "working set fits in L2 (small config)",
                   "source": wl.cite, "index_opts": opts or "library defaults"},
        "roofline": roofline,
        "kernels": kernels,
        "e2e": {"value": round(Q * e2e_steps * world / e2e_s, 2), "unit": "queries/s",
                "h2d_bytes_per_step": Q * wl.n * 4, "d2h_bytes_per_step": Q * 12,
                "how": "isax_nn1 on pinned host buffers, wall clock, copies inside"},
        "latency": {"q1_ms_median": round(statistics.median(lat), 4), "ms_per_query_in_batch": round(ms / args.steps / Q, 5),
                    "how": "isax_nn1_async with Q = 1, CUDA events on the stream, median of 20 calls"},
        "gpu_launches": launches,
        "clocks": clocks,
        "build": {"seconds": round(build_s, 3), "mode": build_mode, "N": wl.N, "n": wl.n,
                  "input_GBps": round(raw_bytes / build_s / 1e9, 1), "index_device_bytes": ix.device_bytes,
                  "stage_ms": bms,
                  # the summarise kernel reads every row once (4n B per series) and writes 48 B per series
                  "summarise": ({"ms": round(bms["summarise"], 3), "bytes": raw_bytes + 48 * wl.N,
                                 "achieved": round((raw_bytes + 48 * wl.N) / (bms["summarise"] / 1e3) / 1e9, 1),
                                 "peak": hbm, "unit": "GB/s",
                                 "frac": round((raw_bytes + 48 * wl.N) / (bms["summarise"] / 1e3) / 1e9 / hbm, 4),
                                 "bound": "hbm (the sequential fp64 chains of R3 and the float-to-double conversions "
                                          "limit it below the copy rate; DESIGN.md sec. 6)"}
                                if bms.get("summarise") else None)},
        "stats": {"candidates_per_query": med(cand) / Q,
                  "refined_per_query": med(refined) / Q,
                  "abandoned_per_query": med(abandoned) / Q,
                  "skipped_per_query": med(skipped) / Q,
                  "window_rows_per_query": med(winrows) / Q,
                  "rounds_max": max(rounds),
                  "note": "candidates = refined to the end + abandoned + skipped by the second band's bound; "
                          "window rows are counted apart"},
    }
    if rank == 0 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(wl, q, args.cpu_seconds, rank)
    if args.stats_out and rank == 0:
        with open(args.stats_out, "w") as f:
            json.dump(st, f)  # the last batch of the per-kernel pass (the Q = 1 calls came after)
    ix.close()
    if rank == 0:
        print(json.dumps(out))
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args, wl, world, rank, local):
    """--impl reference: the oracle (no reference implementation exists), timed on host cores.

    Every step is the same bounded sample of the workload: the oracle's brute force (C7) of 4
    queries over the first S series, S fixed by the first warm-up step (about 2 s of oracle work).
    ms_per_step is that step's measured wall time (oracle only; generating and copying the
    sample's series is excluded); value is the workload's queries/s the sample implies,
    4 / (t_step * N / S)."""
    if rank != 0:
        return
    import torch

    import datagen

    torch.cuda.set_device(local)
    q, _ = datagen.queries(wl, args.queries or wl.Q)
    per_step = 2.0
    first = cpu_baseline(wl, q, per_step, rank)  # calibrates S (counted as a warm-up step)
    S = first["series"]
    for _ in range(max(0, args.warmup - 1)):
        cpu_baseline(wl, q, per_step, rank, series=S)
    vals, secs, last = [], [], None
    for _ in range(args.steps):
        last = cpu_baseline(wl, q, per_step, rank, series=S)
        vals.append(last["value"])
        secs.append(last["seconds"])
    v = args.steps * 4 / (sum(secs) * wl.N / S)
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "queries/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(secs) / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": wl.name, "N": wl.N, "n": wl.n, "w": 16, "card": 256,
                      "step": f"oracle C7 brute force of 4 queries over the first {S} of {wl.N} series; "
                              "value = 4 / (ms_per_step * N / S)"},
           "cpu_baseline": {"kind": "oracle", "cores": last["cores"], "sample": last["sample"], "value": v,
                            "unit": "queries/s"},
           "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
