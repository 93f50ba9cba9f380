"""Seeded synthetic inputs (harness). Both the CUDA path and the oracle read these bytes.

This module holds none of the method's arithmetic. See gen.cu for the recipes and
DESIGN.md "Input recipe". The device generator (libisaxgen.so) is the source for every GPU
test and for the benchmark; the oracle receives the same bytes by device-to-host copy.
`host.py` is a numpy stand-in for CPU-only oracle tests (different bits, same distributions).

WORKLOADS mirrors BASELINE.json "configs" 1-5.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libisaxgen.so")
_lib = None


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    N: int
    n: int
    Q: int
    data_kind: str  # "walk" | "sines"
    data_seed: int
    q_seed: int
    q_walks: int  # queries 0 .. q_walks-1 are independent random walks (seed q_seed)
    q_noisy: int  # the rest are dataset series + N(0, sigma^2) noise, re-z-normalised
    sigma: float = 0.0
    cite: str = ""


WORKLOADS = {
    1: Workload("cfg1_walk_100k_x256", 100_000, 256, 10, "walk", 1, 2, 10, 0, cite="BASELINE.json configs[0]"),
    2: Workload("cfg2_walk_10M_x256", 10_000_000, 256, 100, "walk", 3, 4, 100, 0, cite="BASELINE.json configs[1]"),
    3: Workload("cfg3_walk_100M_x256", 100_000_000, 256, 100, "walk", 5, 6, 50, 50, 0.1, cite="BASELINE.json configs[2]; PAPER.md:384, 509-511"),
    4: Workload("cfg4_walk_200M_x128", 200_000_000, 128, 100, "walk", 7, 8, 100, 0, cite="BASELINE.json configs[3]; SALD shape PAPER.md:384"),
    5: Workload("cfg5_sines_20M_x256", 20_000_000, 256, 1000, "sines", 9, 10, 0, 1000, 0.05, cite="BASELINE.json configs[4]"),
}


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} missing: run `python -m paper_2009_01614_b200.build` (or __graft_entry__.build())")
        L = ctypes.CDLL(_LIB_PATH)
        P, U64, U32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32
        L.isaxgen_walk.argtypes = [P, U64, U64, U32, U64, P]
        L.isaxgen_sines.argtypes = [P, U64, U64, U32, U64, P]
        L.isaxgen_noisy.argtypes = [P, U32, U32, ctypes.c_int, U64, U64, U64, ctypes.c_double, P, P]
        L.isaxgen_fill.argtypes = [P, U64, U64, P, P]
        for f in (L.isaxgen_walk, L.isaxgen_sines, L.isaxgen_noisy, L.isaxgen_fill):
            f.restype = ctypes.c_int
        _lib = L
    return _lib


class GenCtx(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("n", ctypes.c_uint32), ("seed", ctypes.c_uint64)]


def _stream():
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def series(wl: Workload, first_id: int, count: int, out=None):
    """Raw dataset series first_id .. first_id+count-1 of workload wl, as a CUDA fp32 tensor [count, n]."""
    import torch

    if out is None:
        out = torch.empty((count, wl.n), dtype=torch.float32, device="cuda")
    fn = lib().isaxgen_walk if wl.data_kind == "walk" else lib().isaxgen_sines
    rc = fn(ctypes.c_void_p(out.data_ptr()), first_id, count, wl.n, wl.data_seed, _stream())
    if rc:
        raise RuntimeError(f"isaxgen failed rc={rc}")
    return out


def queries(wl: Workload, Q: int | None = None):
    """Raw queries of wl as a CUDA fp32 tensor [Q, n], plus the source ids of noisy copies (-1 for walks)."""
    import torch

    Q = wl.Q if Q is None else Q
    nw = min(Q, wl.q_walks)
    nn = Q - nw
    out = torch.empty((Q, wl.n), dtype=torch.float32, device="cuda")
    src = torch.full((Q,), -1, dtype=torch.int64, device="cuda")
    if nw:
        rc = lib().isaxgen_walk(ctypes.c_void_p(out.data_ptr()), 0, nw, wl.n, wl.q_seed, _stream())
        if rc:
            raise RuntimeError(f"isaxgen_walk failed rc={rc}")
    if nn:
        kind = 0 if wl.data_kind == "walk" else 1
        rc = lib().isaxgen_noisy(ctypes.c_void_p(out[nw:].data_ptr()), nn, wl.n, kind, wl.data_seed, wl.N, wl.q_seed,
                                 wl.sigma, ctypes.c_void_p(src[nw:].data_ptr()), _stream())
        if rc:
            raise RuntimeError(f"isaxgen_noisy failed rc={rc}")
    return out, src


def fill_callback(wl: Workload):
    """(function pointer, ctx) usable as isax_build_stream's fill/ctx. Keep ctx alive during the build."""
    ctx = GenCtx(0 if wl.data_kind == "walk" else 1, wl.n, wl.data_seed)
    fptr = ctypes.cast(lib().isaxgen_fill, ctypes.c_void_p)
    return fptr, ctx
