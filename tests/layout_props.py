"""Property checks of the index's sorted layout and approximate-answer window (test infrastructure).

These check the GPU's permutation and window against properties, not against a re-implementation
of the kernels' rules (VERDICT r1 "un-mirror the oracle"). The only oracle parts used are C5 (the
canonical (key, id) order, oracle.ref.canonical_order, pinned in test_oracle_pins.py) and the
key definition (ref.isax_keys).

Layout (R6, R6b): the sorted positions are the C5 z order, except that every full block
of SUPER = 1024 positions (a super-node) is reordered by a kd split down to cells of CELL = 8 rows
(the 32-row leaves of the scan are four such cells):
  P1  perm is a bijection of the ids;
  P2  every full super-node holds exactly the ids of the same C5 block, and the partial last
      super-node is in C5 order;
  P3  inside a full super-node, every node of 1024, 512, ..., 16 rows (a contiguous, aligned half
      of its parent) has its two halves separated on the node's widest segment (the largest
      max - min symbol range over the node's rows, the lowest segment on ties):
      max over the left half <= min over the right half;
  P4  the splits are stable: inside every 8-row cell, the rows are in ascending order of
      (symbol on the split segment of the level-6 node, ..., symbol on the level-0 one, C5 rank),
      which is what successive stable sorts by those segments produce.
Window (R5): the main window covers whole super-nodes around the one whose z-order key range
holds the query key; so it contains the id of the largest key below key_q (the predecessor) and,
for windows of two or more super-nodes, the smallest key at or above it (the successor).
"""
from __future__ import annotations

import numpy as np

from oracle import ref

SUPER = 1024
LEAF = 8  # the kd cell: the smallest node of the kd order


def _widest(wn: np.ndarray) -> int:
    rng = wn.max(axis=0).astype(np.int64) - wn.min(axis=0).astype(np.int64)
    return int(np.argmax(rng))  # the first maximum: lowest segment on ties


def check_super_block(words_block: np.ndarray, zrank: np.ndarray):
    """P3 + P4 for one full super-node: words_block [1024, 16] in the GPU's order, zrank the C5 rank
    of each of those rows."""
    wb = np.asarray(words_block, dtype=np.int64)
    assert len(wb) == SUPER
    segs = {}  # (level, node start) -> split segment
    size, level = SUPER, 0
    while size > LEAF:
        for a in range(0, SUPER, size):
            node = wb[a:a + size]
            s = _widest(node)
            segs[(level, a)] = s
            left, right = node[: size // 2, s], node[size // 2:, s]
            assert left.max() <= right.min(), f"level {level} node {a}: halves not separated on segment {s}"
        size //= 2
        level += 1
    nlev = level
    for a in range(0, SUPER, LEAF):
        path = [segs[(lv, (a // (SUPER >> lv)) * (SUPER >> lv))] for lv in range(nlev)]
        keys = [tuple(int(wb[r, s]) for s in reversed(path)) + (int(zrank[r]),) for r in range(a, a + LEAF)]
        assert all(keys[k] < keys[k + 1] for k in range(LEAF - 1)), f"cell at {a}: not in stable split order"


def check_layout(perm: np.ndarray, words_by_id: np.ndarray, full_blocks=None):
    """P1-P4 for the whole permutation (or only the listed full super-node indices)."""
    perm = np.asarray(perm, dtype=np.int64)
    N = len(perm)
    assert np.array_equal(np.sort(perm), np.arange(N)), "perm is not a bijection"
    z = ref.canonical_order(words_by_id)
    zrank = np.empty(N, np.int64)
    zrank[z] = np.arange(N)
    nfull = N // SUPER
    blocks = range(nfull) if full_blocks is None else full_blocks
    for b in blocks:
        sl = slice(b * SUPER, (b + 1) * SUPER)
        assert np.array_equal(np.sort(perm[sl]), np.sort(z[sl])), f"super-node {b}: not the C5 block"
        check_super_block(words_by_id[perm[sl]], zrank[perm[sl]])
    assert np.array_equal(perm[nfull * SUPER:], z[nfull * SUPER:]), "partial last super-node not in C5 order"


def pred_succ(words_by_id: np.ndarray, qword):
    """ids of the C5-last row with key < key_q and the C5-first row with key >= key_q (None if none)."""
    z = ref.canonical_order(words_by_id)
    hi, lo = ref.isax_keys(words_by_id[z])
    qh, ql = ref.isax_keys(np.asarray([qword], dtype=np.uint8))
    kq = (int(qh[0]), int(ql[0]))
    keys = list(zip(hi.tolist(), lo.tolist()))
    import bisect

    c = bisect.bisect_left(keys, kq)  # first position with key >= key_q
    pred = int(z[c - 1]) if c > 0 else None
    succ = int(z[c]) if c < len(z) else None
    return pred, succ


def check_window(win, perm: np.ndarray, words_by_id: np.ndarray, qword, L: int):
    """The main window [w0, w1): min(L, N) rows, whole super-nodes (or clamped into [0, N)),
    holding the key predecessor (and for L >= 2048 the successor) of the query key."""
    w0, w1 = int(win[0]), int(win[1])
    N = len(perm)
    assert 0 <= w0 < w1 <= N
    assert w1 - w0 == min(L, N)
    if L >= SUPER and N > L:
        assert w0 % SUPER == 0 or w1 == N, (w0, w1)
    pred, succ = pred_succ(words_by_id, qword)
    ids = set(np.asarray(perm[w0:w1]).tolist())
    if L >= SUPER:
        if pred is not None:
            assert pred in ids, "key predecessor outside the window"
        if (L >= 2 * SUPER or pred is None) and succ is not None:
            assert succ in ids, "key successor outside the window"
