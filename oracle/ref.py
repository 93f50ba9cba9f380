"""Plain numpy / pure-Python oracle of the iSAX exact 1-NN path. TEST INFRASTRUCTURE ONLY.

See oracle/__init__.py for who may call this.

Each function restates a definition from the paper (PAPER.md = P:line) or from the reading
DESIGN.md records where the paper is silent (SPEC.md = S:line). There is
no blocking, fusion or reordering beyond what the definition states.

Precision (reading R3). Sums that decide an integer (z-norm moments, PAA means)
are fp64 and run strictly left to right over the points of one series. They are written as
an explicit Python loop over the point index, vectorised only across series, so every
series sees the same order. numpy's np.sum is pairwise, so it is NOT used for these sums.
Products are never fused into adds.
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np

from .breakpoints import breakpoints

W_DEFAULT = 16
CARD_DEFAULT = 256
SIGMA_EPS = 1e-12  # "if input standard deviation < 1e-12, output is the all-zero series"


# --------------------------------------------------------------------------------------
# C1 z-normalisation (north_star "z-norm then PAA"; R2/R3)
# --------------------------------------------------------------------------------------
def znorm(x: np.ndarray):
    """Z-normalise each row of x [N, n] (fp32).

    Returns (y fp32 [N,n], mu fp64 [N], sigma fp64 [N]), where
        mu    = (sum_i x_i) / n                 (fp64, left to right)
        sigma = sqrt((sum_i (x_i - mu)^2) / n)  (population std, fp64, left to right)
        y_i   = fp32_rne( fp64( (x_i - mu) / sigma ) )   (a true fp64 division)
    If sigma < 1e-12, then y = 0.
    """
    x = np.ascontiguousarray(x, dtype=np.float32)
    if x.ndim != 2:
        raise ValueError("x must be [N, n]")
    N, n = x.shape
    x64 = x.astype(np.float64)
    s = np.zeros(N, dtype=np.float64)
    for i in range(n):
        s = s + x64[:, i]
    mu = s / n
    s2 = np.zeros(N, dtype=np.float64)
    for i in range(n):
        t = x64[:, i] - mu
        s2 = s2 + t * t
    sigma = np.sqrt(s2 / n)
    flat = sigma < SIGMA_EPS
    safe = np.where(flat, 1.0, sigma)
    y = ((x64 - mu[:, None]) / safe[:, None]).astype(np.float32)
    y[flat] = 0.0
    return y, mu, sigma


# --------------------------------------------------------------------------------------
# C2 PAA ("the value of each segment is the mean of the corresponding points")
# --------------------------------------------------------------------------------------
def paa(y: np.ndarray, w: int = W_DEFAULT) -> np.ndarray:
    """Return the segment means m [N, w] (fp64) of the fp32 rows y [N, n]. w must divide n.

    m_s = (sum over the n/w points of segment s, fp64 left to right) / (n/w)
    """
    y = np.asarray(y, dtype=np.float32)
    N, n = y.shape
    if n % w:
        raise ValueError("w must divide n (S:71)")
    seg = n // w
    y64 = y.astype(np.float64)
    m = np.empty((N, w), dtype=np.float64)
    for s in range(w):
        acc = np.zeros(N, dtype=np.float64)
        for j in range(seg):
            acc = acc + y64[:, s * seg + j]
        m[:, s] = acc / seg
    return m


# --------------------------------------------------------------------------------------
# C4 SAX symbols (tie to the upper region, S:90 / S:136)
# --------------------------------------------------------------------------------------
def sax(m: np.ndarray, card: int = CARD_DEFAULT) -> np.ndarray:
    """Return the symbol of each mean: sym = #{k in 1..card-1 : beta_k <= m} (uint8).

    Symbol 0 is the lowest region. A mean exactly on a breakpoint goes to the region above it.
    """
    beta = np.asarray(breakpoints(card), dtype=np.float64)
    m = np.asarray(m, dtype=np.float64)
    return (beta <= m[..., None]).sum(axis=-1).astype(np.uint8)


def summarise(x: np.ndarray, w: int = W_DEFAULT, card: int = CARD_DEFAULT):
    """Return (y, mu, sigma, m, word) for the rows of x: C1, then C2, then C4 (north_star (a))."""
    y, mu, sigma = znorm(x)
    m = paa(y, w)
    return y, mu, sigma, m, sax(m, card)


# --------------------------------------------------------------------------------------
# C5 sort key and canonical order.
# the root subtree is "determined by the first bit of each of the w segments".
# DESIGN.md R6: plane-major bit interleave, so the top w bits are that root key.
# --------------------------------------------------------------------------------------
def isax_key_int(word) -> int:
    """Return the 128-bit key (a Python int) of one 16-segment, 8-bit word.

    Key bit (127 - 16p - s) is bit (7 - p) of symbol s, for planes p = 0..7 and segments
    s = 0..15. Bits are appended most significant first.
    """
    word = [int(c) for c in word]
    if len(word) != 16:
        raise ValueError("key defined for w=16, card=256")
    k = 0
    for p in range(8):
        for s in range(16):
            k = (k << 1) | ((word[s] >> (7 - p)) & 1)
    return k


def isax_keys(words: np.ndarray):
    """Return the keys of words [N,16] as (hi, lo) uint64 arrays. hi holds planes 0..3, lo planes 4..7."""
    words = np.asarray(words, dtype=np.uint64)
    N = words.shape[0]
    hi = np.zeros(N, dtype=np.uint64)
    lo = np.zeros(N, dtype=np.uint64)
    one = np.uint64(1)
    for p in range(8):
        for s in range(16):
            bit = (words[:, s] >> np.uint64(7 - p)) & one
            if p < 4:
                hi = (hi << one) | bit
            else:
                lo = (lo << one) | bit
    return hi, lo


def canonical_order(words: np.ndarray) -> np.ndarray:
    """Return perm with perm[pos] = id, ordered by ascending (key, id) (C5; R6)."""
    hi, lo = isax_keys(words)
    ids = np.arange(len(hi), dtype=np.int64)
    return np.lexsort((ids, lo, hi)).astype(np.int64)


# --------------------------------------------------------------------------------------
# C6 lower bound MINDIST_PAA_iSAX (formula S:117-125)
# --------------------------------------------------------------------------------------
def lb2(q_paa: np.ndarray, words: np.ndarray, n: int, card: int = CARD_DEFAULT) -> np.ndarray:
    """Return the squared lower bound between one query's PAA [w] and words [N, w] (fp64).

    LB^2 = (n/w) * sum_s max(0, lo(c_s) - m_s, m_s - hi(c_s))^2
    [lo, hi) is the region of symbol c_s; lo = -inf for symbol 0 and hi = +inf for the top symbol.
    """
    beta = np.asarray(breakpoints(card), dtype=np.float64)
    ext = np.concatenate([[-np.inf], beta, [np.inf]])
    words = np.asarray(words, dtype=np.int64)
    q = np.asarray(q_paa, dtype=np.float64)[None, :]
    lo = ext[words]
    hi = ext[words + 1]
    d = np.maximum(0.0, np.maximum(lo - q, q - hi))
    w = words.shape[1]
    return (n / w) * (d * d).sum(axis=1)


# --------------------------------------------------------------------------------------
# C7 Euclidean distance and exact 1-NN (ties to the lowest id per north_star)
# --------------------------------------------------------------------------------------
def ed2(q: np.ndarray, Y: np.ndarray) -> np.ndarray:
    """Return fp64 squared ED between one fp32 query [n] and the fp32 rows Y [N, n]."""
    d = Y.astype(np.float64) - np.asarray(q, dtype=np.float64)[None, :]
    return (d * d).sum(axis=1)


def ed2_exact(q, y) -> Fraction:
    """Return the exact squared ED between two fp32 vectors, as a rational."""
    tot = Fraction(0)
    for a, b in zip(np.asarray(q, dtype=np.float32).tolist(), np.asarray(y, dtype=np.float32).tolist()):
        d = Fraction(a) - Fraction(b)
        tot += d * d
    return tot


def euclidean_distance(a, b, abandon_at=None):
    """sqrt(sum (a_i-b_i)^2), or None (ABANDONED) once the running sum exceeds abandon_at^2."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError("length mismatch")
    lim = None if abandon_at is None else float(abandon_at) ** 2
    s = 0.0
    for x, y in zip(a.tolist(), b.tolist()):
        s += (x - y) * (x - y)
        if lim is not None and s > lim:
            return None
    return float(np.sqrt(s))


NEAR_REL = 1e-9  # fp64 d^2 of 256 terms is within ~3e-14 relative of the exact value


def resolve_exact(q, Y_rows: dict) -> tuple[int, Fraction]:
    """Return the lexicographic minimum of (exact d^2, id) over the candidates {id: fp32 row}."""
    best = None
    for i in sorted(Y_rows):
        d = ed2_exact(q, Y_rows[i])
        if best is None or d < best[1]:
            best = (i, d)
    return best


def nn1_bruteforce(Y: np.ndarray, Qy: np.ndarray):
    """Return the exact 1-NN of each z-normalised query among the z-normalised rows Y (C7).

    Returns (ids int64 [Q], d2 list of Fraction, dist fp64 [Q]), where dist = sqrt(exact d^2).
    Every id whose fp64 d^2 is within NEAR_REL of the minimum is re-evaluated exactly.
    """
    Y = np.asarray(Y, dtype=np.float32)
    ids, d2s, dist = [], [], []
    for q in np.asarray(Qy, dtype=np.float32):
        d = ed2(q, Y)
        mn = d.min()
        near = np.nonzero(d <= mn * (1 + NEAR_REL) + 1e-300)[0]
        i, e = resolve_exact(q, {int(j): Y[j] for j in near})
        ids.append(i)
        d2s.append(e)
        dist.append(float(np.sqrt(float(e))))
    return np.asarray(ids, dtype=np.int64), d2s, np.asarray(dist)


# --------------------------------------------------------------------------------------
# C8 ParIS-style index search, on the sorted order (a7 window; R5)
# --------------------------------------------------------------------------------------
def lower_bound_pos(sorted_hi, sorted_lo, key_hi, key_lo) -> int:
    """Return the first position whose key is >= (key_hi, key_lo), by plain bisection."""
    lo, hi = 0, len(sorted_hi)
    while lo < hi:
        mid = (lo + hi) // 2
        if (int(sorted_hi[mid]), int(sorted_lo[mid])) < (int(key_hi), int(key_lo)):
            lo = mid + 1
        else:
            hi = mid
    return lo


def window(pos: int, N: int, L: int) -> tuple[int, int]:
    """Return [start, end), the L sorted positions centred on pos and clamped into [0, N) (R5)."""
    if N <= L:
        return 0, N
    start = min(max(pos - L // 2, 0), N - L)
    return start, start + L


def nn1_index_search(x: np.ndarray, Qx: np.ndarray, w: int = W_DEFAULT, L: int = 1024):
    """ParIS query answering on raw rows x and raw queries Qx (both z-normalised here).

    The steps follow P:270-279:
    1. "computes an approximate answer by calculating BSF": the real distances over the
       leaf-sized window of the C5 sorted order centred at the query key's lower_bound position
       (the library's own window rule, R5, affects speed only and is not
       restated here).
    2. "lower bound distances between the query and the iSAX summary of each data series",
       for every series outside the window.
    3. "prune the series whose lower bound distance is larger than the approximate real
       distance" (strict, with fp64 slack NEAR_REL).
    4. The candidate list is consumed with early-abandoning real distances; the
       BSF is updated.
    5. Near ties are resolved exactly (lowest id).
    Returns (ids, stats), with stats = list of dicts (window, candidates, abandoned).
    """
    y, _, _, _, words = summarise(x, w)
    qy, _, _, qm, qwords = summarise(Qx, w)
    N, n = y.shape
    perm = canonical_order(words)
    khi, klo = isax_keys(words[perm])
    qhi, qlo = isax_keys(qwords)
    out, stats = [], []
    for qi in range(len(qy)):
        q = qy[qi].astype(np.float64)
        s0, s1 = window(lower_bound_pos(khi, klo, qhi[qi], qlo[qi]), N, L)
        win_ids = perm[s0:s1]
        d_win = ed2(qy[qi], y[win_ids])
        bsf = float(d_win.min())
        done = {int(i): float(d) for i, d in zip(win_ids, d_win)}
        inwin = np.zeros(N, dtype=bool)
        inwin[s0:s1] = True
        lbs = lb2(qm[qi], words[perm], n)
        cand = np.nonzero(~inwin & (lbs <= bsf * (1 + NEAR_REL)))[0]
        abandoned = 0
        for p in cand:
            i = int(perm[p])
            row = y[i].astype(np.float64)
            s = 0.0
            lim = bsf * (1 + NEAR_REL)
            ok = True
            for a, b in zip(q.tolist(), row.tolist()):
                s += (a - b) * (a - b)
                if s > lim:
                    ok = False
                    break
            if not ok:
                abandoned += 1
                continue
            done[i] = s
            bsf = min(bsf, s)
        near = {i: y[i] for i, d in done.items() if d <= bsf * (1 + NEAR_REL) + 1e-300}
        best, _ = resolve_exact(qy[qi], near)
        out.append(best)
        stats.append({"window": (s0, s1), "candidates": int(len(cand)), "abandoned": abandoned})
    return np.asarray(out, dtype=np.int64), stats
