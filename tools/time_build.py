#!/usr/bin/env python
"""Time isax_build on a BASELINE config (device events), and check the words against a reference
build: python tools/time_build.py --config 2 [--reps 3]. Prints build ms, input GB/s and the
summarise kernel's share when run under a launch list."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch

    import datagen
    from paper_2009_01614_b200 import isax

    wl = datagen.WORKLOADS[a.config]
    free, _ = torch.cuda.mem_get_info()
    dev_input = 2 * wl.N * wl.n * 4 + (8 << 30) < free
    x = datagen.series(wl, 0, wl.N) if dev_input else None
    best = None
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        if dev_input:
            ix = isax.Index.build(x)
        else:
            fptr, ctx = datagen.fill_callback(wl)
            ix = isax.Index.build_stream(wl.N, wl.n, fptr, ctx)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
        print("  stages (device ms):", ix.stats().get("build_ms"), flush=True)
        ix.close()
        torch.cuda.empty_cache()
    gb = wl.N * wl.n * 4 / 1e9
    print(f"cfg{a.config} build {'device input' if dev_input else 'streamed (generation included)'}: "
          f"{best:.1f} ms, {gb / (best / 1e3):.1f} GB/s of input")


if __name__ == "__main__":
    main()
