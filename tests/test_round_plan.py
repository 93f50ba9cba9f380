"""The per-query plan of scan rounds (R9, R10; csrc/round_plan.h), driven on the CPU through
isax_debug_plan_round against a simulated scanner.

The scanner holds candidate bounds (LB^2) at sorted positions. A round keeps the candidates with
lo < LB^2 <= min(hi, T) at positions in [plo, phi); if they fit the capacity they are refined
(marked), else the round's 64-bin histogram goes to the plan. The checks: every candidate under
the final threshold is refined exactly once, and the plan terminates, also when many candidates
share one bound (the band cannot be split by value: positions are split) and when T = 0 (an exact
duplicate in the window).
"""
import numpy as np
import pytest

from paper_2009_01614_b200 import isax

HIST_BINS = 64
INF = np.float32(np.inf)


def run_plan(lb, pos, N, cap, T, max_rounds=20000):
    lb = np.asarray(lb, np.float32)
    pos = np.asarray(pos, np.int64)
    band = np.array([-1.0, INF], np.float32)
    rng = np.array([0, N], np.uint32)
    state = np.array([N, 0], np.uint32)
    T = np.float32(T)
    refined = np.zeros(len(lb), np.int64)
    for r in range(max_rounds):
        lo, hi = band
        tused = np.float32(min(hi, T))
        keep = (lb > lo) & (lb <= tused) & (pos >= rng[0]) & (pos < rng[1])
        cnt = int(keep.sum())
        hist = np.zeros(HIST_BINS, np.uint32)
        if cnt > cap:
            l0 = max(lo, np.float32(0))
            span = np.float32(tused - l0)
            x = (lb[keep] - l0) / span if span > 0 else np.zeros(cnt, np.float32)
            b = np.minimum((np.maximum(x, 0) * HIST_BINS).astype(np.int64), HIST_BINS - 1)
            hist = np.bincount(b, minlength=HIST_BINS).astype(np.uint32)
        else:
            refined[keep] += 1
        act = isax.plan_round(band, rng, state, cnt, cap, hist, False, tused, T, N)
        assert act != isax.PLAN_ERROR
        if act == isax.PLAN_DONE:
            return refined, r + 1
    raise AssertionError("the plan did not terminate")


def check(lb, pos, N, cap, T):
    refined, rounds = run_plan(lb, pos, N, cap, T)
    must = np.asarray(lb, np.float32) <= np.float32(T)
    assert np.all(refined[must] == 1), f"{int((refined[must] != 1).sum())} candidates not refined exactly once"
    assert np.all(refined[~must] == 0)
    return rounds


def test_fits_in_one_round():
    rng = np.random.default_rng(1)
    lb = rng.uniform(0, 10, 1000).astype(np.float32)
    assert check(lb, rng.integers(0, 10_000, 1000), 10_000, cap=5000, T=5.0) == 1


@pytest.mark.parametrize("cap", [7, 50, 300])
def test_bands_shrink_and_continue(cap):
    rng = np.random.default_rng(cap)
    lb = rng.exponential(2.0, 5000).astype(np.float32)
    rounds = check(lb, rng.integers(0, 100_000, 5000), 100_000, cap=cap, T=3.0)
    assert rounds >= 2


@pytest.mark.parametrize("value", [0.0, 1.25])
def test_many_equal_bounds_split_positions(value):
    """300 candidates share one bound (identical words): the histogram cannot split them, so the
    rounds split the sorted positions (halving, then doubling ranges)."""
    rng = np.random.default_rng(7)
    N = 50_000
    lb = np.concatenate([np.full(300, value, np.float32), rng.uniform(0, 3, 2000).astype(np.float32)])
    pos = np.concatenate([rng.integers(20_000, 21_000, 300), rng.integers(0, N, 2000)])
    check(lb, pos, N, cap=7, T=2.0)


def test_exact_duplicate_threshold_zero():
    """T = 0 (an exact duplicate in the window): only LB^2 = 0 candidates are kept; 40 of them
    against a capacity of 7."""
    rng = np.random.default_rng(3)
    N = 20_000
    lb = np.concatenate([np.zeros(40, np.float32), rng.uniform(0, 1, 500).astype(np.float32)])
    pos = np.concatenate([rng.integers(5000, 5100, 40), rng.integers(0, N, 500)])
    check(lb, pos, N, cap=7, T=0.0)


def test_near_overflow_starts_over():
    band = np.array([0.5, 2.0], np.float32)
    rng = np.array([100, 200], np.uint32)
    state = np.array([100, 2], np.uint32)
    act = isax.plan_round(band, rng, state, 3, 10, np.zeros(64, np.uint32), True, 2.0, 2.5, 1000)
    assert act == isax.PLAN_RESCAN
    assert band[0] == -1.0 and np.isinf(band[1]) and rng.tolist() == [0, 1000]


def test_band_a_few_ulps_wide_makes_progress():
    """Six candidates at the top of a band about 30 fp32 ulps wide against a capacity of 5: the
    histogram's shrunk edge (63/64 of the span) rounds back onto the band's upper end, so the plan
    must split positions instead of repeating the round (found on the GPU by tools/fuzz_gpu.py:
    cand_cap 5 over 220K sines)."""
    lo = np.float32(182.600998)
    ulp = np.spacing(lo)
    top = np.float32(lo + 30 * ulp)
    lb = np.concatenate([np.full(6, top, np.float32), np.float32(lo) - np.arange(1, 40, dtype=np.float32)])
    pos = np.arange(len(lb)) * 97 + 11
    N = 10_000
    refined, rounds = run_plan(lb, pos, N, cap=5, T=np.float32(top), max_rounds=5000)
    assert np.all(refined == 1) and rounds < 5000
