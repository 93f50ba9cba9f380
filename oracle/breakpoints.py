"""Oracle breakpoint table (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

PAPER.md:168 ("[iSAX Representation]", §Preliminaries) says iSAX "divides the (y-axis)
space in different regions by assigning a bit-wise symbol to each region". It gives no
breakpoint values. Reading R1 follows SPEC.md:77-85 and SURVEY §8(c) C3: the
breakpoints are the equiprobable quantiles of N(0,1).

    beta_k = correctly rounded fp64 of Phi^-1(k / card),   k = 1 .. card-1

Here Phi^-1(p) = sqrt(2) * erfinv(2p - 1), evaluated with mpmath at 60 significant digits.
The result is rounded to the nearest double via a 40-digit decimal string; Python's
float(str) rounds correctly. For card = 2^b the table is the subset beta^(256)_{k*256/card}
of the 8-bit table (dyadic nesting).
"""
from __future__ import annotations

import functools

import mpmath

MAX_CARD = 256


@functools.lru_cache(maxsize=None)
def breakpoints(card: int = MAX_CARD) -> tuple[float, ...]:
    """Return (beta_1, ..., beta_{card-1}) for an alphabet of `card` symbols (a power of 2)."""
    if card < 2 or card > MAX_CARD or card & (card - 1):
        raise ValueError("card must be a power of two in [2, 256]")
    out = []
    with mpmath.workdps(60):
        for k in range(1, card):
            p = mpmath.mpf(k) / card
            x = mpmath.sqrt(2) * mpmath.erfinv(2 * p - 1)
            out.append(float(mpmath.nstr(x, 40, strip_zeros=False)))
    return tuple(out)


def region(sym: int, card: int = MAX_CARD) -> tuple[float, float]:
    """Return the value interval [lo, hi) of symbol `sym`.

    Symbol 0 is the lowest region, with lo = -inf. The top symbol has hi = +inf.
    """
    b = breakpoints(card)
    lo = -float("inf") if sym == 0 else b[sym - 1]
    hi = float("inf") if sym == card - 1 else b[sym]
    return lo, hi
