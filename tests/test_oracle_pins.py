"""Pins for the oracle (CPU only). They check the oracle against something other than itself.

* SPEC.md hand examples (tests/golden/spec_examples.json, each with its citation).
* Closed forms. A ramp series has known moments, PAA and symbols; the symbols come from
  Phi (mpmath.ncdf), not from the inverse used to build the table.
* Invariants: LB admissibility, LB(q, SAX(q)) = 0, monotonicity under refinement, prefix
  consistency, affine invariance of z-norm.
* Library routines: scipy.special.ndtri and statistics.NormalDist for the breakpoints.
* Brute force with exact rationals on tiny inputs.

Each pin is chosen so that a plausible slip fails it: a dropped term, a wrong sign or index,
a transposed operand, off-by-one regions, the wrong tie side, or a sample instead of a
population sigma.
"""
import math
import statistics
from fractions import Fraction

import mpmath
import numpy as np
import pytest
import scipy.special

from oracle import ref
from oracle.breakpoints import breakpoints, region


# ----------------------------------------------------------------------------- breakpoints
def test_breakpoints_golden(golden):
    for ex in golden["breakpoints"]:
        got = breakpoints(ex["card"])
        assert len(got) == ex["card"] - 1, ex["cite"]
        np.testing.assert_allclose(got, ex["beta"], atol=10 ** -ex["decimals"], err_msg=ex["cite"])


def test_breakpoints_correctly_rounded_against_phi():
    """beta_k is the double nearest to Phi^-1(k/256).

    Phi is checked at the half-ulp neighbours of beta_k with mpmath.ncdf, the forward CDF.
    The table itself comes from the inverse (erfinv), so this pin is independent of it.
    """
    b = breakpoints(256)
    with mpmath.workdps(50):
        for k, x in enumerate(b, start=1):
            p = mpmath.mpf(k) / 256
            if x == 0.0:
                assert k == 128
                continue
            lo = (mpmath.mpf(x) + mpmath.mpf(math.nextafter(x, -math.inf))) / 2
            hi = (mpmath.mpf(x) + mpmath.mpf(math.nextafter(x, math.inf))) / 2
            assert mpmath.ncdf(lo) <= p <= mpmath.ncdf(hi), k


def test_breakpoints_structure():
    b = np.array(breakpoints(256))
    assert b[127] == 0.0  # beta_128 = Phi^-1(1/2)
    np.testing.assert_array_equal(b, -b[::-1])  # symmetry
    assert np.all(np.diff(b) > 0)
    assert np.all(np.diff(b.astype(np.float32)) > 0)  # distinct even in fp32
    for card in (2, 4, 8, 16, 32, 64, 128):  # dyadic nesting
        np.testing.assert_array_equal(np.array(breakpoints(card)), b[(256 // card) - 1 :: 256 // card])


def test_breakpoints_vs_library_routines():
    b = np.array(breakpoints(256))
    k = np.arange(1, 256)
    nd = scipy.special.ndtri(k / 256.0)
    st = np.array([statistics.NormalDist().inv_cdf(kk / 256.0) for kk in k])
    ulp = np.spacing(np.abs(b)) + (b == 0) * 1e-300
    assert np.max(np.abs(nd - b) / ulp) <= 4
    assert np.max(np.abs(st - b) / ulp) <= 4
    assert b[63] == pytest.approx(-0.6744897501960817, abs=2e-16)
    assert b[-1] == pytest.approx(2.6600674686174597, abs=5e-16)


# ----------------------------------------------------------------------------- z-norm
def test_znorm_golden(golden):
    for ex in golden["znorm"]:
        y, _, _ = ref.znorm(np.array([ex["x"]], np.float32))
        np.testing.assert_array_equal(y[0], np.array(ex["y"], np.float32), err_msg=ex["cite"])


def test_znorm_ramp_closed_form():
    n = 256
    x = np.arange(n, dtype=np.float32)[None]
    y, mu, sigma = ref.znorm(x)
    assert mu[0] == 127.5
    # population sigma of 0..n-1 is sqrt((n^2-1)/12); a sample sigma would be sqrt(n(n+1)/12)
    assert sigma[0] == math.sqrt((n * n - 1) / 12.0)
    assert sigma[0] == pytest.approx(73.90027063549903, rel=1e-15)
    expect = ((np.arange(n) - 127.5) / math.sqrt((n * n - 1) / 12.0)).astype(np.float32)
    np.testing.assert_array_equal(y[0], expect)


def test_znorm_moments_and_affine_invariance():
    rng = np.random.default_rng(0)
    x = np.cumsum(rng.standard_normal((200, 256)), axis=1).astype(np.float32)
    y, _, _ = ref.znorm(x)
    y64 = y.astype(np.float64)
    assert np.all(np.abs(y64.mean(1)) < 1e-6)
    assert np.all(np.abs(y64.std(1) - 1) < 1e-6)
    y2, _, _ = ref.znorm((3.0 * x.astype(np.float64) + 7.0).astype(np.float32))
    assert np.max(np.abs(y2.astype(np.float64) - y64)) < 1e-5
    # idempotent up to fp32 rounding
    y3, _, _ = ref.znorm(y)
    assert np.max(np.abs(y3.astype(np.float64) - y64)) < 1e-6


def test_znorm_constant_and_tiny_sigma():
    x = np.full((2, 16), 5.0, np.float32)
    x[1, 3] += 1e-6  # sigma ~2.4e-7 > 1e-12, so the row is normalised, not zeroed
    y, _, s = ref.znorm(x)
    assert np.all(y[0] == 0) and s[0] == 0
    assert y[1, 3] > 3.0


# ----------------------------------------------------------------------------- PAA / SAX
def test_paa_golden(golden):
    for ex in golden["paa"]:
        m = ref.paa(np.array([ex["y"]], np.float32), ex["w"])
        np.testing.assert_array_equal(m[0], ex["m"], err_msg=ex["cite"])


def test_paa_piecewise_constant_and_constant():
    vals = np.linspace(-2, 2, 16).astype(np.float32)
    y = np.repeat(vals, 16)[None]
    np.testing.assert_array_equal(ref.paa(y, 16)[0], vals.astype(np.float64))
    y = np.full((1, 128), 0.25, np.float32)
    np.testing.assert_array_equal(ref.paa(y, 16)[0], np.full(16, 0.25))


def test_isax_golden(golden):
    for ex in golden["isax"]:
        assert int(ref.sax(np.array([ex["m"]]), ex["card"])[0]) == ex["sym"], ex["cite"]


def test_ramp_paa_and_word_closed_form():
    """Ramp x_t = t: m_s = (16 s + 7.5 - 127.5) / sigma, and symbol = floor(256 Phi(m_s))."""
    n = 256
    y, _, sigma, m, word = ref.summarise(np.arange(n, dtype=np.float32)[None])
    closed = (16 * np.arange(16) + 7.5 - 127.5) / sigma[0]
    np.testing.assert_allclose(m[0], closed, atol=1e-6)
    with mpmath.workdps(30):
        expect = [int(mpmath.floor(256 * mpmath.ncdf(c))) for c in closed]
        # the pin is only valid if no mean sits within 1e-6 of a region edge
        for c in closed:
            f = 256 * mpmath.ncdf(c)
            assert abs(f - mpmath.nint(f)) > 1e-4
    assert word[0].tolist() == expect == [13, 20, 29, 42, 57, 75, 95, 116, 139, 160, 180, 198, 213, 226, 235, 242]


def test_sax_constant_series_and_tie_goes_up():
    _, _, _, m, word = ref.summarise(np.full((1, 256), 3.0, np.float32))
    assert np.all(m == 0) and np.all(word == 128)  # mean 0 sits exactly on beta_128: upper region
    b = breakpoints(256)
    assert ref.sax(np.array([b[9]]))[0] == 10  # on beta_10 -> symbol 10
    assert ref.sax(np.array([math.nextafter(b[9], -math.inf)]))[0] == 9


def test_sax_monotone_and_prefix_consistent():
    rng = np.random.default_rng(1)
    m = np.sort(rng.standard_normal(20000) * 1.5)
    s = ref.sax(m).astype(int)
    assert np.all(np.diff(s) >= 0)
    for bits in range(1, 8):
        np.testing.assert_array_equal(ref.sax(m, 1 << bits), s >> (8 - bits))


def test_promote_golden(golden):
    """the low-card symbol is a bit prefix of the high-card symbol."""
    for ex in golden["promote"]:
        (ls, lb), (hs, hb) = ex["low"], ex["high"]
        assert ((hs >> (hb - lb)) == ls) == ex["expect"], ex["cite"]


# ----------------------------------------------------------------------------- key order
def test_key_top_bits_are_root_subtree_key():
    """the root subtree is set by the first bit of each of the w segments."""
    rng = np.random.default_rng(2)
    words = rng.integers(0, 256, (500, 16)).astype(np.uint8)
    hi, lo = ref.isax_keys(words)
    root = np.zeros(500, np.uint64)
    for s in range(16):
        root |= (words[:, s].astype(np.uint64) >> np.uint64(7)) << np.uint64(15 - s)
    np.testing.assert_array_equal(hi >> np.uint64(48), root)
    for i in range(20):
        assert ref.isax_key_int(words[i]) == (int(hi[i]) << 64) | int(lo[i])


def test_canonical_order_is_plane_lexicographic():
    """Ascending key order is lexicographic over the bit planes (plane 0 = top bits), then id."""
    rng = np.random.default_rng(3)
    words = rng.integers(0, 4, (400, 16)).astype(np.uint8) * 64  # many equal keys -> id ties
    perm = ref.canonical_order(words)

    def planes(w):
        return tuple(sum(((int(w[s]) >> (7 - p)) & 1) << (15 - s) for s in range(16)) for p in range(8))

    expect = sorted(range(400), key=lambda i: (planes(words[i]), i))
    assert perm.tolist() == expect


def test_lower_bound_window():
    """C8's approximate-answer window: L rows of the C5 order centred on the query key's
    lower_bound position, clamped into [0, N)."""
    keys_hi = np.array([0, 1, 1, 1, 5, 9], np.uint64)
    keys_lo = np.array([3, 0, 2, 2, 0, 0], np.uint64)
    assert ref.lower_bound_pos(keys_hi, keys_lo, 1, 2) == 2  # first key >= (1, 2)
    assert ref.lower_bound_pos(keys_hi, keys_lo, 1, 3) == 4
    assert ref.lower_bound_pos(keys_hi, keys_lo, 0, 0) == 0
    assert ref.lower_bound_pos(keys_hi, keys_lo, 10, 0) == 6
    assert ref.window(2, 6, 4) == (0, 4) and ref.window(5, 6, 4) == (2, 6) and ref.window(3, 10, 4) == (1, 5)
    assert ref.window(0, 3, 8) == (0, 3)


def test_layout_checker_detects_violations():
    """tests/layout_props.py (the GPU layout's property checker) accepts a block that satisfies
    P3/P4 trivially and rejects it after a cross-half swap or a within-leaf swap."""
    from tests import layout_props as lp

    wb = np.zeros((1024, 16), np.int64)
    wb[:, 0] = np.arange(1024) // 4  # one non-constant segment, ascending: every split is on it
    zr = np.arange(1024)
    lp.check_super_block(wb, zr)
    bad = wb.copy()
    bad[[10, 700]] = bad[[700, 10]]
    with pytest.raises(AssertionError):
        lp.check_super_block(bad, zr)
    zr2 = zr.copy()
    zr2[[4, 5]] = zr2[[5, 4]]  # equal symbols out of C5 order: the splits were not stable
    with pytest.raises(AssertionError):
        lp.check_super_block(wb, zr2)


# ----------------------------------------------------------------------------- LB / ED
def test_lb_golden(golden):
    for ex in golden["lb"]:
        v = ref.lb2(np.array(ex["q_paa"]), np.array([ex["word"]]), ex["n"], ex["card"])[0]
        assert math.sqrt(v) == pytest.approx(ex["lb"], abs=10 ** -ex["decimals"]), ex["cite"]


def test_lb_ramp_vs_zero_word_closed_form():
    """Ramp query against the all-128 word, region [0, beta_129): d_s = -m_s for m_s < 0, else m_s - beta_129."""
    n = 256
    _, _, sigma, m, _ = ref.summarise(np.arange(n, dtype=np.float32)[None])
    b129 = breakpoints(256)[128]
    d = np.where(m[0] < 0, -m[0], m[0] - b129)
    expect = 16 * np.sum(d * d)
    got = ref.lb2(m[0], np.full((1, 16), 128, np.uint8), n)[0]
    assert got == pytest.approx(expect, rel=1e-14)
    assert math.sqrt(got) == pytest.approx(15.901110294454368, rel=1e-7)
    # admissible against ED to the all-zero series (which summarises to the all-128 word)
    y, _, _ = ref.znorm(np.arange(n, dtype=np.float32)[None])
    assert got <= ref.ed2(y[0], np.zeros((1, n), np.float32))[0]


def test_lb_of_own_word_is_zero_and_admissible():
    rng = np.random.default_rng(4)
    for n, card in [(256, 256), (128, 256), (256, 16), (256, 4), (256, 2)]:
        x = np.cumsum(rng.standard_normal((300, n)), axis=1).astype(np.float32)
        y, _, _, m, word = ref.summarise(x, 16, card)
        q = rng.standard_normal((20, n)).cumsum(1).astype(np.float32)
        qy, _, _, qm, qw = ref.summarise(q, 16, card)
        for i in range(20):
            assert ref.lb2(qm[i], qw[i : i + 1], n, card)[0] == 0.0
            lbs = ref.lb2(qm[i], word, n, card)
            eds = ref.ed2(qy[i], y)
            assert np.all(lbs <= eds * (1 + 1e-9) + 1e-12), (n, card)


def test_lb_monotone_under_refinement():
    rng = np.random.default_rng(5)
    x = np.cumsum(rng.standard_normal((500, 256)), axis=1).astype(np.float32)
    _, _, _, m, w8 = ref.summarise(x)
    qm = ref.paa(ref.znorm(np.cumsum(rng.standard_normal((1, 256)), 1).astype(np.float32))[0])[0]
    prev = np.zeros(500)
    for bits in range(1, 9):
        lb = ref.lb2(qm, w8.astype(int) >> (8 - bits), 256, 1 << bits)
        assert np.all(lb >= prev - 1e-12)
        prev = lb


def test_ed_golden(golden):
    for ex in golden["ed"]:
        assert ref.euclidean_distance(ex["a"], ex["b"], ex["abandon_at"]) == ex["dist"], ex["cite"]
    a = np.random.default_rng(6).standard_normal(64)
    b = np.random.default_rng(7).standard_normal(64)
    assert ref.euclidean_distance(a, b, math.inf) == ref.euclidean_distance(a, b)


def test_ed2_exact_matches_rational_definition():
    q = np.array([0.1, -2.5, 3.0], np.float32)
    y = np.array([1e-8, 2.5, -3.0], np.float32)
    expect = sum((Fraction(float(a)) - Fraction(float(b))) ** 2 for a, b in zip(q, y))
    assert ref.ed2_exact(q, y) == expect
    assert float(expect) == pytest.approx(ref.ed2(q, y[None])[0], rel=1e-15)


# ----------------------------------------------------------------------------- exact 1-NN
def _exact_nn(qy, Y):
    best = None
    for i in range(len(Y)):
        d = ref.ed2_exact(qy, Y[i])
        if best is None or d < best[1]:
            best = (i, d)
    return best


def test_nn1_bruteforce_equals_exact_rational_scan():
    rng = np.random.default_rng(8)
    x = np.cumsum(rng.standard_normal((60, 32)), axis=1).astype(np.float32)
    x[17] = x[5]  # duplicate: the tie must go to id 5
    Y, _, _ = ref.znorm(x)
    q = np.vstack([x[17], np.cumsum(rng.standard_normal((5, 32)), 1)]).astype(np.float32)
    qy, _, _ = ref.znorm(q)
    ids, d2, dist = ref.nn1_bruteforce(Y, qy)
    assert ids[0] == 5 and d2[0] == 0 and dist[0] == 0.0
    for j in range(len(qy)):
        i, e = _exact_nn(qy[j], Y)
        assert ids[j] == i and d2[j] == e


def test_nn1_single_series_and_near_tie():
    Y = np.zeros((1, 16), np.float32)
    ids, _, _ = ref.nn1_bruteforce(Y, np.ones((2, 16), np.float32))
    assert ids.tolist() == [0, 0]
    # two rows at fp32-adjacent distances: fp64 sees them within NEAR_REL, exact picks right one
    q = np.zeros(4, np.float32)
    a = np.array([1, 0, 0, 0], np.float32)
    b = np.array([np.nextafter(np.float32(1), np.float32(0)), 0, 0, 0], np.float32)
    ids, _, _ = ref.nn1_bruteforce(np.vstack([a, b]), q[None])
    assert ids[0] == 1


@pytest.mark.parametrize("N,L,n", [(1, 1024, 64), (37, 8, 64), (300, 32, 128), (300, 1024, 64), (500, 1, 64)])
def test_index_search_equals_bruteforce(N, L, n):
    """The north star: the oracle's index search equals brute force on tiny inputs (C8 == C7)."""
    rng = np.random.default_rng(N * 7 + L)
    x = np.cumsum(rng.standard_normal((N, n)), axis=1).astype(np.float32)
    if N > 10:
        x[N - 1] = x[3]
    q = np.cumsum(rng.standard_normal((6, n)), axis=1).astype(np.float32)
    if N > 10:
        q[0] = x[N - 1] * 2 + 1  # same shape after z-norm -> ties between ids 3 and N-1
    ids, stats = ref.nn1_index_search(x, q, 16, L)
    Y, _, _ = ref.znorm(x)
    qy, _, _ = ref.znorm(q)
    bf, _, _ = ref.nn1_bruteforce(Y, qy)
    np.testing.assert_array_equal(ids, bf)
    if N > 10:
        assert ids[0] == 3
    for st in stats:
        s0, s1 = st["window"]
        assert s1 - s0 == min(L, N) and 0 <= s0 and s1 <= N
        assert st["candidates"] + (s1 - s0) <= N  # SPEC.md:276 accounting identity (pruned = rest)
