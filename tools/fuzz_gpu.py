#!/usr/bin/env python
"""Randomised parity runs on the GPU (test infrastructure: it runs the oracle).

    python tools/fuzz_gpu.py --seconds 150 [--seed 1]

Each trial draws a collection (N, n, kind), a query batch (size, share of noisy copies, noise) and
index options at random, builds the index through the C ABI, answers the batch, and compares every
id and distance with the oracle's brute force on the same bytes (tests/gpu_util.py). It prints one
line per trial and exits non-zero at the first mismatch, with the trial's parameters.
"""
import argparse
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=120.0)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--only", type=int, default=0, help="draw every trial of the seed but run only this one (to reproduce)")
    ap.add_argument("--opt", action="append", default=[], help="with --only: override an index option, key=value")
    a = ap.parse_args()
    import numpy as np
    import torch

    import datagen
    from paper_2009_01614_b200 import isax
    from tests.gpu_util import assert_nn_parity, oracle_nn1

    rnd = random.Random(a.seed)
    t0, trial = time.time(), 0
    while time.time() - t0 < a.seconds and (not a.only or trial < a.only):
        trial += 1
        n = rnd.choice([64, 128, 128, 256, 256, 256, 512])
        N = rnd.choice([rnd.randint(1, 40), rnd.randint(900, 1100), rnd.randint(2_000, 40_000), rnd.randint(40_000, 400_000)])
        if rnd.random() < 0.06:  # now and then several hyper-nodes and many super-nodes
            N = rnd.randint(400_000, 3_000_000)
        if N * n > 400_000_000:
            N = 400_000_000 // n
        kind = rnd.choice(["walk", "walk", "sines"])
        Q = rnd.choice([1, 2, 3, 5, 8, 15, 16, 17, 31, 33, 64, 100, 257])
        noisy = rnd.choice([0, 0, Q // 2, Q])
        sigma = rnd.choice([0.02, 0.1, 0.5])
        opts = {}
        if rnd.random() < 0.3:
            opts["batch_Q"] = rnd.choice([1, 3, 16, 40, 100])
        if rnd.random() < 0.3:
            # (a capacity of 5 or 64 takes about 5 x candidates / capacity rounds, each a rescan: only
            # over small collections here, to keep a run short; 5 over 220K sines is 120K rounds)
            opts["cand_cap"] = rnd.choice([5, 7, 64, 1000, 50_000]) if N <= 50_000 else rnd.choice([300, 1000, 50_000])
        if rnd.random() < 0.4:
            opts["first_band"] = rnd.choice([-1.0, 0.02, 0.3, 0.9])
        if rnd.random() < 0.3:
            opts["window_L"] = rnd.choice([1, 100, 512, 1024, 2048, 4096])
        if rnd.random() < 0.3:
            opts["probe_bits"] = rnd.choice([0xFFFFFFFF, 1, 3, 5])
        if rnd.random() < 0.2:
            opts["probe_L"] = rnd.choice([1, 32, 64, 256, 1024])
        if rnd.random() < 0.1:
            opts["flags"] = 1
        if a.only and trial != a.only:
            rnd.random()  # (the duplicate draw below)
            continue
        for o in a.opt:
            k, v = o.split("=", 1)
            opts[k] = float(v) if "." in v else int(v)
        wl = datagen.Workload(f"fuzz{trial}", N, n, Q, kind, 1000 + trial, 5000 + trial, Q - noisy, noisy, sigma)
        x = datagen.series(wl, 0, N)
        q, _ = datagen.queries(wl)
        if rnd.random() < 0.15 and N > 50:  # exact copies and duplicates
            x = x.clone()
            q = q.clone()
            x[N // 2] = x[3]
            q[0] = x[N // 2]
            if N > 2000 and rnd.random() < 0.5:  # many exact ties: copies of one row, constant rows, a constant query
                g = torch.Generator().manual_seed(trial)
                k = rnd.choice([5, 40, 300, 700])
                idx = torch.randperm(N, generator=g)[:k].to(x.device)
                x[idx] = x[7].clone()
                cidx = torch.randperm(N, generator=g)[:rnd.choice([3, 60, 400])].to(x.device)
                x[cidx] = 2.5
                q[Q - 1] = x[7].clone()
                if Q > 2:
                    q[1] = -4.0
        ids_or, dist_or, _ = oracle_nn1(x.cpu().numpy(), q.cpu().numpy(), K=1200)  # (room for the tie trials' copies)
        desc = f"trial {trial}: N={N} n={n} {kind} Q={Q} noisy={noisy} sigma={sigma} opts={opts}"
        try:
            with isax.Index.build(x, **opts) as ix:
                for call in range(2):  # (the adaptive first band runs the second call in the other mode)
                    ids, dist = ix.nn1(q)
                    torch.cuda.synchronize()
                    assert_nn_parity(ids.cpu().numpy(), dist.cpu().numpy(), ids_or, dist_or)
                st = ix.stats()
        except Exception as e:  # noqa: BLE001
            print("FAIL", desc, "->", repr(e), flush=True)
            sys.exit(1)
        print("ok  ", desc, "rounds", max(st["rounds"]), flush=True)
        del x, q
    print(f"{trial} trials, all equal to the oracle")


if __name__ == "__main__":
    main()
