"""ctypes wrapper for oracle/oracle.c. TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The shared library is compiled by `__graft_entry__.build()`, or on first use, with gcc:
-ffp-contract=off, no -ffast-math, OpenMP. The functions compute the same definitions as
oracle/ref.py (a test checks the two agree bit for bit) at benchmark sizes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import ref
from .breakpoints import breakpoints

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

CFLAGS = ["-std=c11", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC"]


def build(force: bool = False) -> str:
    """Compile liboracle.so if it is missing or older than oracle.c."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        L.orc_summarise.argtypes = [P, ctypes.c_int64, ctypes.c_int, ctypes.c_int, P, ctypes.c_int, P, P, P, P, P]
        L.orc_summarise.restype = ctypes.c_int64
        L.orc_nn1_scan.argtypes = [P, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, P, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_double, P, P, P, P, P]
        L.orc_nn1_scan.restype = ctypes.c_int64
        L.orc_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def num_threads() -> int:
    return int(lib().orc_num_threads())


def summarise(x: np.ndarray, w: int = 16, card: int = 256, want_y: bool = True, want_paa: bool = True):
    """Return (y|None, mu, sigma, m|None, word), the same as ref.summarise, for raw rows x [N, n]."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    N, n = x.shape
    if n % w:
        raise ValueError("w must divide n")
    beta = np.ascontiguousarray(breakpoints(card), dtype=np.float64)
    y = np.empty((N, n), np.float32) if want_y else None
    mu = np.empty(N, np.float64)
    sd = np.empty(N, np.float64)
    m = np.empty((N, w), np.float64) if want_paa else None
    sym = np.empty((N, w), np.uint8)
    bad = lib().orc_summarise(_p(x), N, n, w, _p(beta), card, _p(y), _p(mu), _p(sd), _p(m), _p(sym))
    if bad:
        raise ValueError(f"{bad} rows hold NaN/Inf")
    return y, mu, sd, m, sym


class NN1Scan:
    """Streaming brute-force exact 1-NN (C7) over raw chunks fed in id order.

    The queries must already be z-normalised (ref.znorm / summarise). feed(id0, raw_chunk)
    scans a chunk and caches the oracle z-normalised rows of every current near-tie entry.
    result() resolves the near ties exactly and returns (ids, dist).
    """

    def __init__(self, qy: np.ndarray, K: int = 32):
        self.qy = np.ascontiguousarray(qy, dtype=np.float32)
        self.Q, self.n = self.qy.shape
        self.K = K
        self.qt = np.ascontiguousarray(self.qy.T)
        self.best = np.full(self.Q, np.inf)
        self.cnt = np.zeros(self.Q, np.int32)
        self.ids = np.zeros((self.Q, K), np.int64)
        self.d2 = np.zeros((self.Q, K), np.float64)
        self.ovf = np.full(self.Q, np.inf)  # smallest d2 dropped for lack of room (oracle.c)
        self.rows = {}

    def feed(self, id0: int, xraw: np.ndarray):
        xraw = np.ascontiguousarray(xraw, dtype=np.float32)
        m, n = xraw.shape
        assert n == self.n
        bad = lib().orc_nn1_scan(_p(xraw), m, n, id0, _p(self.qt), self.Q, self.K, ref.NEAR_REL, _p(self.best),
                                 _p(self.cnt), _p(self.ids), _p(self.d2), _p(self.ovf))
        if bad:
            raise ValueError(f"{bad} rows hold NaN/Inf")
        live = set()
        for q in range(self.Q):
            for i in self.ids[q, : self.cnt[q]].tolist():
                live.add(i)
                if i not in self.rows and id0 <= i < id0 + m:
                    y, _, _, _, _ = summarise(xraw[i - id0 : i - id0 + 1], want_paa=False)
                    self.rows[i] = y[0]
        self.rows = {i: r for i, r in self.rows.items() if i in live}

    def result(self):
        lost = self.ovf <= self.best * (1 + ref.NEAR_REL) + 1e-300
        if lost.any():
            raise RuntimeError(f"oracle near-tie list overflow at queries {np.nonzero(lost)[0][:8]}; raise K")
        ids, dist, d2 = [], [], []
        for q in range(self.Q):
            cand = {int(i): self.rows[int(i)] for i in self.ids[q, : self.cnt[q]]}
            i, e = ref.resolve_exact(self.qy[q], cand)
            ids.append(i)
            d2.append(e)
            dist.append(float(np.sqrt(float(e))))
        return np.asarray(ids, np.int64), np.asarray(dist), d2
