#!/usr/bin/env python
"""Every query of BASELINE.json configs 1-5 against the oracle, with the artifacts committed.

    python tools/parity_full.py --configs 1 2 3 4 5 --out profiles/parity_r02

For each config: the index is built exactly as bench.py builds it (device input when it fits,
else the streamed two-pass build), the config's whole query batch is answered in one
isax_nn1_async call (the bench's launch configuration) twice (the adaptive policy runs the first
call with the first band and the second without, R15), and the oracle's streamed brute force
(C7, oracle/oracle.c + exact rational tie resolution) answers the same queries over all N
series generated from the same seeds. It writes <out>_cfgK.json with one row per query:
[query, gpu id, oracle id, gpu dist, oracle dist], the count of equal ids and the largest
relative distance error (bar: ids equal, dist within 1e-5 relative; north_star).
Test infrastructure (it runs the oracle): never imported by the product.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[1, 2, 3, 4, 5])
    ap.add_argument("--out", default="gpurun_out/parity")
    ap.add_argument("--head", default=os.environ.get("ISAX_HEAD", "unknown"))
    args = ap.parse_args()
    import numpy as np
    import torch

    import datagen
    from oracle import clib
    from paper_2009_01614_b200 import isax
    from tests.gpu_util import oracle_nn1_streamed

    torch.cuda.set_device(0)
    for cfg in args.configs:
        wl = datagen.WORKLOADS[cfg]
        free, _ = torch.cuda.mem_get_info()
        t0 = time.perf_counter()
        if 2 * wl.N * wl.n * 4 + (8 << 30) < free:
            x = datagen.series(wl, 0, wl.N)
            ix = isax.Index.build(x)
            del x
            torch.cuda.empty_cache()
            mode = "device input"
        else:
            fptr, ctx = datagen.fill_callback(wl)
            ix = isax.Index.build_stream(wl.N, wl.n, fptr, ctx)
            mode = "streamed input"
        q, src = datagen.queries(wl)
        # the library's adaptive policy (R15) runs its first call with the first band and its
        # second without: both are compared with the oracle
        ids, dist = ix.nn1(q)
        torch.cuda.synchronize()
        st = ix.stats()
        ids, dist = ids.cpu().numpy(), dist.cpu().numpy()
        ids2, dist2 = ix.nn1(q)
        torch.cuda.synchronize()
        st2 = ix.stats()
        ids2, dist2 = ids2.cpu().numpy(), dist2.cpu().numpy()
        modes = [st.get("first_band"), st2.get("first_band")]
        t_gpu = time.perf_counter() - t0
        ix.close()
        torch.cuda.empty_cache()
        qh = q.cpu().numpy()
        t1 = time.perf_counter()
        ids_or, dist_or, _ = oracle_nn1_streamed(wl, qh, K=256)
        t_or = time.perf_counter() - t1
        err = np.abs(dist.astype(np.float64) - dist_or) / np.maximum(np.abs(dist_or), 1e-3)
        err2 = np.abs(dist2.astype(np.float64) - dist_or) / np.maximum(np.abs(dist_or), 1e-3)
        eq = int((ids == ids_or).sum())
        eq2 = int((ids2 == ids_or).sum())
        rows = [[int(j), int(ids[j]), int(ids2[j]), int(ids_or[j]), float(dist[j]), float(dist2[j]), float(dist_or[j])]
                for j in range(len(ids))]
        rep = {"config": cfg, "workload": wl.name, "N": wl.N, "n": wl.n, "Q": int(len(ids)), "head": args.head,
               "build": mode, "bar": "ids equal (ties to the lowest id); dist within 1e-5 relative (north_star)",
               "first_band_per_call": modes,
               "ids_equal": eq, "ids_equal_call2": eq2, "ids_total": int(len(ids)),
               "max_rel_dist_err": float(max(err.max(), err2.max())),
               "dist_within_1e-5": int((err <= 1e-5).sum()), "dist_within_1e-5_call2": int((err2 <= 1e-5).sum()),
               "rounds_max": int(max(st["rounds"])), "rounds_max_call2": int(max(st2["rounds"])),
               "oracle": {"kind": "C7 brute force over all N (oracle/oracle.c, OpenMP) + exact rational near-tie resolution",
                          "cores": clib.num_threads(), "seconds": round(t_or, 1)},
               "gpu_seconds_incl_build": round(t_gpu, 1),
               "columns": ["query", "gpu_id_call1", "gpu_id_call2", "oracle_id", "gpu_dist_call1", "gpu_dist_call2",
                           "oracle_dist"], "rows": rows}
        path = f"{args.out}_cfg{cfg}.json"
        os.makedirs(os.path.dirname(path) or ".", exist_ok=True)
        with open(path, "w") as f:
            json.dump(rep, f)
        print(f"cfg{cfg}: ids {eq}/{len(ids)} (first band {modes[0]}), {eq2}/{len(ids)} (first band {modes[1]}) equal, "
              f"max rel dist err {max(err.max(), err2.max()):.3g}, oracle {t_or:.0f} s", flush=True)


if __name__ == "__main__":
    main()
