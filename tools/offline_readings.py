#!/usr/bin/env python
"""Reproduce the measurements behind DESIGN.md's readings and NEXT-3 decision (test infrastructure).

    python tools/offline_readings.py --out profiles/offline_readings_r02.json [--parts r5 r6b r14 next3]

Runs on a GPU box: the index is built by the library (its sorted layout is what the readings are
about), words and positions are exported, and the counting is done here in numpy from the
method's definitions (C6 LB with the u8 quantisation of R11b). Every part prints and stores the
numbers DESIGN.md quotes.

  r5     multi-probe approximate answer (R5): on 1M sines with 1000 noisy-copy queries (config 5's
         recipe, scaled), the fraction of queries whose window BSF already equals the final NN
         distance, and the candidates per query, with probes off and on.
  r6b    kd order inside super-nodes (R6b) against plain z order (C5): (leaf, query) pairs that
         survive the leaf bound and members tested, 4M walks, 24 walk queries, T = each query's
         final BSF (1 + 2^-12).
  r14    refinement order (R14): half-row reads per query to refine the LB-filtered candidates of
         2M walks, in one pass (sorted order), in two bands split at 0.55 T, and fully LB-sorted;
         early abandon after the first half and at the end (R8).
  next3  coarse-to-fine member test: on 4M walks, the fraction of members of alive
         leaves passing a coarse bound (8 lookups in per-query tables of the high nibbles of two
         segments) vs the full u8 test, and the fraction of (leaf, query) pairs where some lane
         passes each (a warp runs the full test when any lane passes the coarse one).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

DELTA = 2.0 ** -12
LEAF = 32


def build(wl, **opts):
    import torch

    import datagen
    from paper_2009_01614_b200 import isax

    x = datagen.series(wl, 0, wl.N)
    ix = isax.Index.build(x, **opts)
    del x
    torch.cuda.empty_cache()
    return ix


def lut_u8(lut_row, T):
    """R11b: e = floor(LUT * sc), sc = 254 / T rounded down, clamped at 255 (per segment, symbol)."""
    sc = np.float32(np.float32(254.0) / np.float32(T)) if T > 0 else np.float32(np.inf)
    e = np.floor(lut_row.astype(np.float32) * sc)
    e[lut_row <= 0] = 0
    return np.minimum(e, 255).astype(np.int32)


def member_e8(words_sorted, e8):
    """u8 sum of every member (words [N, 16] in sorted order) against one query's table e8 [16, 256]."""
    acc = np.zeros(len(words_sorted), np.int32)
    for s in range(16):
        acc += e8[s][words_sorted[:, s]]
    return acc


def leaf_node_e8(mn, mx, qsym, e8):
    """u8 node bound of every leaf: sum_s e8[s][clamp(q_s, min_s, max_s)] (R11)."""
    acc = np.zeros(len(mn), np.int32)
    for s in range(16):
        c = np.clip(qsym[s], mn[:, s], mx[:, s])
        acc += e8[s][c]
    return acc


def leaf_boxes(words_sorted):
    n = len(words_sorted) // LEAF * LEAF
    w = words_sorted[:n].reshape(-1, LEAF, 16)
    return w.min(axis=1), w.max(axis=1)


def part_r5(out):
    import torch

    import datagen

    wl = datagen.Workload("r5_sines_1M", 1_000_000, 256, 1000, "sines", 21, 22, 0, 1000, 0.05)
    res = {}
    q, _ = datagen.queries(wl)
    for name, opts in (("probes_off", dict(probe_bits=0xFFFFFFFF)), ("probes_on", dict())):
        # the window BSF of each query (round 0's threshold) against its final NN distance
        ix2 = build(wl, first_band=-1, **opts)
        ids, dist = ix2.nn1(q)
        torch.cuda.synchronize()
        st = ix2.stats()
        b0 = np.asarray(st["bsf0_d2"], np.float64)
        bf = np.asarray(st["bsf_final_d2"], np.float64)
        res[name] = {"nn_found_by_window": float(np.mean(b0 <= bf * (1 + 1e-7))),
                     "candidates_per_query_mean": float(np.mean(st["candidates"])),
                     "candidates_per_query_median": float(np.median(st["candidates"])),
                     "window_rows_per_query": float(np.mean(st["window_rows"]))}
        ix2.close()
    out["r5"] = {"workload": "1M sines x 256 (config 5 recipe, seed 21), 1000 noisy copies sigma 0.05 (seed 22)",
                 **res}
    print("r5", json.dumps(out["r5"]), flush=True)


def queries_and_T(ix, wl, Q):
    import torch

    import datagen

    q, _ = datagen.queries(wl, Q)
    ids, dist = ix.nn1(q)
    torch.cuda.synchronize()
    st = ix.stats()
    T = np.asarray(st["bsf_final_d2"], np.float64) * (1 + DELTA)
    dbg = ix.query_debug(q.cpu().numpy(), 0, 0)
    return q, T, dbg


def part_r6b(out):
    import datagen
    from oracle import ref

    wl = datagen.Workload("r6b_walk_4M", 4_000_000, 256, 24, "walk", 31, 32, 24, 0)
    ix = build(wl, first_band=-1)
    q, T, dbg = queries_and_T(ix, wl, 24)
    ex = ix.export(0, wl.N, sax=True, perm=True)
    ix.close()
    words = ex["sax"]
    kd = words[ex["perm"].astype(np.int64)]            # the library's layout (z order + kd in super-nodes)
    z = words[ref.canonical_order(words)]              # plain C5 z order
    res = {}
    for name, ws in (("z_order", z), ("kd_order", kd)):
        mn, mx = leaf_boxes(ws)
        pairs = 0
        for i in range(len(T)):
            e8 = lut_u8(dbg["lut"][i], T[i])
            pairs += int((leaf_node_e8(mn, mx, dbg["q_sax"][i].astype(np.int64), e8) <= 254).sum())
        res[name] = {"leaf_query_pairs": pairs, "members_tested": pairs * LEAF}
    res["kd_vs_z_members"] = res["kd_order"]["members_tested"] / res["z_order"]["members_tested"] - 1
    out["r6b"] = {"workload": "4M walks x 256 (seed 31), 24 walk queries (seed 32), T = final BSF (1 + 2^-12)", **res}
    print("r6b", json.dumps(out["r6b"]), flush=True)


def refine_reads(order, d2_half, d2_full, bsf0):
    """(half rows read, final BSF) to refine candidates in the given order with early abandon after
    the first half (partial > bsf (1 + delta)) and the BSF update on completion (R8)."""
    bsf = bsf0
    reads = 0
    for h, f in zip(d2_half[order], d2_full[order]):
        reads += 1
        if h > bsf * (1 + DELTA):
            continue
        reads += 1
        if f < bsf:
            bsf = f
    return reads, bsf


def part_r14(out):
    import datagen
    from oracle import ref

    wl = datagen.Workload("r14_walk_2M", 2_000_000, 256, 24, "walk", 41, 42, 24, 0)
    x = datagen.series(wl, 0, wl.N).cpu().numpy()
    ix = build(wl, first_band=-1)
    import torch

    q, _ = datagen.queries(wl, 24)
    ids, dist = ix.nn1(q)
    torch.cuda.synchronize()
    st = ix.stats()
    dbg = ix.query_debug(q.cpu().numpy(), 0, 0)
    ex = ix.export(0, wl.N, sax=True, perm=True)
    ix.close()
    from oracle import clib

    y, _, _, _, _ = clib.summarise(x, want_paa=False)
    qy, _, _, qm, _ = clib.summarise(q.cpu().numpy())
    words = ex["sax"]
    perm = ex["perm"].astype(np.int64)
    single, two, sorted_ = [], [], []
    for i in range(len(qy)):
        T = st["bsf0_d2"][i] * (1 + DELTA)
        lb = ref.lb2(qm[i], words[perm], wl.n)
        w0, w1 = st["window"][2 * i], st["window"][2 * i + 1]
        lb[w0:w1] = np.inf
        cand = np.nonzero(lb <= T)[0]
        rows = y[perm[cand]].astype(np.float64)
        d = rows - qy[i].astype(np.float64)[None]
        half = (d[:, :wl.n // 2] ** 2).sum(1)
        full = (d * d).sum(1)
        b0 = st["bsf0_d2"][i]
        single.append(refine_reads(np.arange(len(cand)), half, full, b0)[0])
        # two bands (R14): LB^2 <= 0.55 T first, in list (position) order; then the rest, minus those
        # whose LB^2 already exceeds the BSF the first band left (filter_kernel), in list order
        lbc = lb[cand]
        lo = np.nonzero(lbc <= 0.55 * T)[0]
        r1, b1 = refine_reads(lo, half, full, b0)
        hi = np.nonzero((lbc > 0.55 * T) & (lbc <= b1 * (1 + DELTA)))[0]
        r2, _ = refine_reads(hi, half, full, b1)
        two.append(r1 + r2)
        # MESSI's order: ascending LB^2, stopping at the first LB^2 above the BSF
        srt = np.argsort(lbc, kind="stable")
        bsf, r = b0, 0
        for j in srt:
            if lbc[j] > bsf * (1 + DELTA):
                break
            rr, bsf = refine_reads(np.array([j]), half, full, bsf)
            r += rr
        sorted_.append(r)
    out["r14"] = {"workload": "2M walks x 256 (seed 41), 24 walk queries (seed 42), window BSF as the start",
                  "half_rows_per_query": {"one_pass_sorted_position_order": float(np.mean(single)),
                                          "two_bands_split_0.55T": float(np.mean(two)),
                                          "full_lb_sort_stop_at_bsf": float(np.mean(sorted_))}}
    print("r14", json.dumps(out["r14"]), flush=True)


def coarse_tables(lut_row, T):
    """NEXT-3 coarse bound: for segment pairs (2k, 2k+1), a 256-entry u8 table indexed by the high
    nibbles of both symbols, entry = the u8 entries (R11b) of the two segments' smallest LUT values
    over the nibble cells, added. Each term is <= the member's own u8 entry, so the coarse sum never
    exceeds the full u8 sum (a member the coarse test prunes, the full test prunes too)."""
    e8 = lut_u8(lut_row, T)
    cell_min = e8.reshape(16, 16, 16).min(axis=2)  # [segment][high nibble]
    return [cell_min[2 * k][:, None] + cell_min[2 * k + 1][None, :] for k in range(8)]


def part_next3(out):
    import datagen

    wl = datagen.Workload("next3_walk_4M", 4_000_000, 256, 24, "walk", 51, 52, 24, 0)
    ix = build(wl, first_band=-1)
    q, T, dbg = queries_and_T(ix, wl, 24)
    ex = ix.export(0, wl.N, sax=True, perm=True)
    ix.close()
    ws = ex["sax"][ex["perm"].astype(np.int64)]
    n = len(ws) // LEAF * LEAF
    ws = ws[:n]
    mn, mx = leaf_boxes(ws)
    hi4 = (ws >> 4).astype(np.int64)
    tot_members = full_pass = coarse_pass = 0
    pairs = pairs_full_any = pairs_coarse_any = 0
    for i in range(len(T)):
        e8 = lut_u8(dbg["lut"][i], T[i])
        alive = np.nonzero(leaf_node_e8(mn, mx, dbg["q_sax"][i].astype(np.int64), e8) <= 254)[0]
        if not len(alive):
            continue
        idx = (alive[:, None] * LEAF + np.arange(LEAF)[None]).ravel()
        full = member_e8(ws[idx], e8) <= 254
        ct = coarse_tables(dbg["lut"][i], T[i])
        c = np.zeros(len(idx), np.int32)
        for k in range(8):
            c += ct[k][hi4[idx, 2 * k], hi4[idx, 2 * k + 1]]
        coarse = c <= 254
        assert np.all(coarse[full]), "the coarse bound must not prune a member the full test keeps"
        tot_members += len(idx)
        full_pass += int(full.sum())
        coarse_pass += int(coarse.sum())
        pairs += len(alive)
        pairs_full_any += int(full.reshape(-1, LEAF).any(axis=1).sum())
        pairs_coarse_any += int(coarse.reshape(-1, LEAF).any(axis=1).sum())
    fa = pairs_coarse_any / pairs
    out["next3"] = {"workload": "4M walks x 256 (seed 51), 24 walk queries (seed 52), T = final BSF (1 + 2^-12)",
                    "members_of_alive_leaves": tot_members, "pass_full": full_pass / tot_members,
                    "pass_coarse": coarse_pass / tot_members, "pairs_any_lane_full": pairs_full_any / pairs,
                    "pairs_any_lane_coarse": fa,
                    "lookups_per_pair_with_prefilter": 8 + 16 * fa, "lookups_per_pair_now": 16}
    print("next3", json.dumps(out["next3"]), flush=True)


def part_early(out):
    """Early exit inside the member test: after k of the 16 lookups, the warp (32 members of one
    alive leaf, one query) stops if every lane's partial u8 sum already exceeds 254. Fraction of
    (leaf, query) pairs that stop at k, in segment order 0..15 and in a per-query order (segments
    by descending mean table entry), and the lookups per pair that implies."""
    import datagen

    wl = datagen.Workload("early_walk_4M", 4_000_000, 256, 24, "walk", 51, 52, 24, 0)
    ix = build(wl, first_band=-1)
    q, T, dbg = queries_and_T(ix, wl, 24)
    ex = ix.export(0, wl.N, sax=True, perm=True)
    ix.close()
    ws = ex["sax"][ex["perm"].astype(np.int64)]
    n = len(ws) // LEAF * LEAF
    ws = ws[:n]
    mn, mx = leaf_boxes(ws)
    ks = (2, 4, 6, 8, 10, 12, 14)
    stop = {o: np.zeros(len(ks)) for o in ("fixed", "by_query")}
    pairs = 0
    for i in range(len(T)):
        e8 = lut_u8(dbg["lut"][i], T[i])
        alive = np.nonzero(leaf_node_e8(mn, mx, dbg["q_sax"][i].astype(np.int64), e8) <= 254)[0]
        if not len(alive):
            continue
        idx = (alive[:, None] * LEAF + np.arange(LEAF)[None]).ravel()
        w = ws[idx].astype(np.int64)
        pairs += len(alive)
        for o, order in (("fixed", np.arange(16)), ("by_query", np.argsort(-e8.mean(axis=1), kind="stable"))):
            part = np.zeros(len(idx), np.int32)
            done = 0
            for j, s in enumerate(order):
                part += e8[s][w[:, s]]
                if j + 1 in ks:
                    stop[o][ks.index(j + 1)] += int((part.reshape(-1, LEAF) > 254).all(axis=1).sum())
                    done += 1
    res = {"workload": "4M walks x 256 (seed 51), 24 walk queries (seed 52), T = final BSF (1 + 2^-12)",
           "pairs": pairs, "k": list(ks)}
    for o in stop:
        f = stop[o] / pairs
        res[o + "_stopped_after_k"] = [round(float(v), 4) for v in f]
        # one exit test at k: k lookups for every pair, 16 - k more for the pairs that go on
        res[o + "_lookups_per_pair_one_test"] = {int(k): round(float(k + (16 - k) * (1 - f[j])), 2)
                                                 for j, k in enumerate(ks)}
    out["early"] = res
    print("early", json.dumps(res), flush=True)


def kd_refine(ws, size):
    """One more kd level (R6b) inside every block of `size` consecutive rows: stable sort by the
    segment with the largest symbol range (lowest on ties). The halves are the children."""
    w = ws.reshape(-1, size, 16)
    rng = w.max(axis=1).astype(np.int32) - w.min(axis=1)
    seg = rng.argmax(axis=1)                                    # first maximum: the lowest segment
    keys = np.take_along_axis(w, seg[:, None, None], axis=2)[:, :, 0]
    order = np.argsort(keys, axis=1, kind="stable")
    return np.take_along_axis(w, order[:, :, None], axis=1).reshape(-1, 16)


def boxes(ws, size):
    w = ws.reshape(-1, size, 16)
    return w.min(axis=1), w.max(axis=1)


def part_sub(out):
    """Sub-leaf boxes: under the (leaf, query) pairs that survive the 32-member leaf bound, the
    fraction of 16-member halves and 8-member quarters whose own box bound survives, in the
    library's layout as it is and after one / two more kd levels inside each leaf; and the members
    that pass the u8 test (the floor any box level can reach). 10M walks (config 2's shape)."""
    import datagen

    wl = datagen.Workload("sub_walk_10M", 10_000_000, 256, 24, "walk", 61, 62, 24, 0)
    ix = build(wl, first_band=-1)
    q, T, dbg = queries_and_T(ix, wl, 24)
    import torch
    st = ix.stats()
    T0 = np.asarray(st["bsf0_d2"], np.float64) * (1 + DELTA)   # the scan's own threshold (window BSF)
    ex = ix.export(0, wl.N, sax=True, perm=True)
    ix.close()
    ws0 = ex["sax"][ex["perm"].astype(np.int64)]
    n = len(ws0) // 1024 * 1024
    ws0 = ws0[:n]
    ws1 = kd_refine(ws0, 32)      # kd down to 16
    ws2 = kd_refine(ws1, 16)      # kd down to 8
    res = {}
    for name, ws in (("layout_now", ws0), ("kd_to_16", ws1), ("kd_to_8", ws2)):
        mn, mx = boxes(ws, 32)
        mn16, mx16 = boxes(ws, 16)
        mn8, mx8 = boxes(ws, 8)
        pairs = h16 = h8 = h8_under16 = memb = 0
        for i in range(len(T0)):
            e8 = lut_u8(dbg["lut"][i], T0[i])
            qs = dbg["q_sax"][i].astype(np.int64)
            alive = np.nonzero(leaf_node_e8(mn, mx, qs, e8) <= 254)[0]
            pairs += len(alive)
            i16 = (alive[:, None] * 2 + np.arange(2)[None]).ravel()
            a16 = leaf_node_e8(mn16[i16], mx16[i16], qs, e8) <= 254
            h16 += int(a16.sum())
            i8 = (alive[:, None] * 4 + np.arange(4)[None]).ravel()
            a8 = leaf_node_e8(mn8[i8], mx8[i8], qs, e8) <= 254
            h8 += int(a8.sum())
            idx = (alive[:, None] * LEAF + np.arange(LEAF)[None]).ravel()
            memb += int((member_e8(ws[idx], e8) <= 254).sum())
        res[name] = {"leaf_pairs": pairs, "members_under_leaves": pairs * 32,
                     "members_under_alive_16": h16 * 16, "members_under_alive_8": h8 * 8,
                     "frac_16": h16 * 16 / (pairs * 32), "frac_8": h8 * 8 / (pairs * 32),
                     "members_passing_u8": memb}
    out["sub"] = {"workload": "10M walks x 256 (seed 61), 24 walk queries (seed 62), T = window BSF (1 + 2^-12)", **res}
    print("sub", json.dumps(out["sub"]), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/offline_readings.json")
    ap.add_argument("--parts", nargs="+", default=["r5", "r6b", "r14", "next3", "early"])
    a = ap.parse_args()
    import torch

    torch.cuda.set_device(0)
    out = {"when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    for p in a.parts:
        t0 = time.time()
        {"r5": part_r5, "r6b": part_r6b, "r14": part_r14, "next3": part_next3, "early": part_early, "sub": part_sub}[p](out)
        out.setdefault("seconds", {})[p] = round(time.time() - t0, 1)
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
