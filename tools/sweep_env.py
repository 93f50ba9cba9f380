#!/usr/bin/env python
"""A/B of library settings read from the environment, on one index built once.

python tools/sweep_env.py --config 3 --var ISAX_BAND0 --values 0 0.25 0.5
For each value: set the variable, 3 warm-up calls, 20 timed calls (CUDA events on the stream),
then one stats pass. Prints q/s, per-stage ms of the first batch and the counters.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--var", default="ISAX_BAND0")
    ap.add_argument("--values", nargs="+", default=["0"])
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--opt", action="append", default=[])
    a = ap.parse_args()
    import torch

    import datagen
    from paper_2009_01614_b200 import isax

    wl = datagen.WORKLOADS[a.config]
    opts = {k: int(v) for k, v in (o.split("=", 1) for o in a.opt)}
    free, _ = torch.cuda.mem_get_info()
    if 2 * wl.N * wl.n * 4 + (8 << 30) < free:
        x = datagen.series(wl, 0, wl.N)
        ix = isax.Index.build(x, **opts)
        del x
        torch.cuda.empty_cache()
    else:
        fptr, ctx = datagen.fill_callback(wl)
        ix = isax.Index.build_stream(wl.N, wl.n, fptr, ctx, **opts)
    q, _ = datagen.queries(wl)
    Q = q.shape[0]
    ids = torch.empty(Q, dtype=torch.int64, device="cuda")
    dist = torch.empty(Q, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    step = ix.nn1_bound(q, ids, dist, stream.cuda_stream)
    ref_ids = None
    for v in a.values:
        os.environ[a.var] = v
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        got = ids.cpu().numpy().copy()
        if ref_ids is None:
            ref_ids = got
        same = bool((got == ref_ids).all())
        kms = {k: [] for k in ("qprep", "window", "lbscan", "candcheck", "refine", "total")}
        for _ in range(5):
            step()
            st = ix.stats()
            for k in kms:
                kms[k].append(st["ms_first_batch"][k])
        out = {"var": a.var, "value": v, "qps": round(Q / ms * 1e3), "ms_step": round(ms, 4), "ids_same": same,
               "ms_first_round": {k: round(statistics.median(x), 4) for k, x in kms.items()},
               "cand_pq": round(sum(st["candidates"]) / Q), "refined_pq": round(sum(st["refined"]) / Q),
               "skipped_pq": round(sum(st["skipped"]) / Q), "leaf_pairs_pq": round(sum(st["leaves_alive"]) / Q),
               "rounds_max": max(st["rounds"]), "launches": st["launches"],
               "first_band": st.get("first_band"), "first_band_improved": st.get("first_band_improved")}
        print(json.dumps(out), flush=True)
    os.environ.pop(a.var, None)
    ix.close()


if __name__ == "__main__":
    main()
