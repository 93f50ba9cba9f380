#!/usr/bin/env python
"""Single-query latency breakdown on a BASELINE config: python tools/latency_q1.py --config 3
Prints the median device time of Q = 1 calls and the per-stage device times of the last ones."""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    a = ap.parse_args()
    import torch

    import datagen
    from paper_2009_01614_b200 import isax

    wl = datagen.WORKLOADS[a.config]
    free, _ = torch.cuda.mem_get_info()
    if 2 * wl.N * wl.n * 4 + (8 << 30) < free:
        x = datagen.series(wl, 0, wl.N)
        ix = isax.Index.build(x)
        del x
    else:
        fptr, ctx = datagen.fill_callback(wl)
        ix = isax.Index.build_stream(wl.N, wl.n, fptr, ctx)
    q, _ = datagen.queries(wl)
    for qi in (0, q.shape[0] - 1):
        q1 = q[qi:qi + 1].contiguous()
        for _ in range(5):
            ix.nn1(q1)
        torch.cuda.synchronize()
        lat, stages = [], []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ix.nn1(q1)
            e1.record()
            torch.cuda.synchronize()
            lat.append(e0.elapsed_time(e1))
            stages.append(ix.stats()["ms_first_batch"])
        med = {k: round(statistics.median(s[k] for s in stages), 4) for k in stages[0]}
        st = ix.stats()
        print(f"cfg{a.config} query {qi}: median {statistics.median(lat):.4f} ms; stages {med}; candidates {st['candidates']}, "
              f"leaf pairs {st['leaves_alive']}, first_band {st.get('first_band')}", flush=True)
    ix.close()


if __name__ == "__main__":
    main()
