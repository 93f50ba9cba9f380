"""The C oracle (oracle/oracle.c) computes the same definitions as the numpy oracle, bit for bit.

CPU only. The numpy oracle is pinned in test_oracle_pins.py, so agreeing with it pins the C
code too.
"""
import numpy as np
import pytest

from oracle import clib, ref


@pytest.mark.parametrize("n", [128, 256, 64])
def test_summarise_bit_exact_vs_numpy(n):
    rng = np.random.default_rng(n)
    x = np.cumsum(rng.standard_normal((700, n)), axis=1).astype(np.float32)
    x[5] = 2.5  # constant row
    x[6] *= 1e-3
    x[7] += 1e4
    a = ref.summarise(x)
    b = clib.summarise(x)
    for u, v in zip(a, b):
        np.testing.assert_array_equal(u, v)


def test_summarise_rejects_nonfinite():
    x = np.zeros((3, 64), np.float32)
    x[1, 7] = np.nan
    with pytest.raises(ValueError):
        clib.summarise(x)


@pytest.mark.parametrize("chunk", [1, 97, 5000])
def test_nn1_scan_matches_bruteforce(chunk):
    rng = np.random.default_rng(chunk)
    N, n = 3000, 128
    x = np.cumsum(rng.standard_normal((N, n)), axis=1).astype(np.float32)
    x[2999] = x[12]  # exact duplicate of id 12: the tie goes to 12
    q = np.cumsum(rng.standard_normal((7, n)), axis=1).astype(np.float32)
    q[0] = x[2999] * 2 + 1
    qy, _, _ = ref.znorm(q)
    Y, _, _ = ref.znorm(x)
    bf, d2, dist = ref.nn1_bruteforce(Y, qy)
    sc = clib.NN1Scan(qy, K=8)
    for s in range(0, N, chunk):
        sc.feed(s, x[s : s + chunk])
    ids, dd, e = sc.result()
    np.testing.assert_array_equal(ids, bf)
    assert ids[0] == 12
    assert e == d2
    np.testing.assert_array_equal(dd, dist)
