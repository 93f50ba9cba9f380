"""Thin Python binding of libisax.so (include/isax.h). It only marshals arguments.

Every step of the method runs in the library's sm_100a kernels. torch supplies device memory
and the current CUDA stream. There is no CPU fallback: if libisax.so is missing, importing
this module raises.
"""
from __future__ import annotations

import ctypes
import json
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# ISAX_LIB: an alternative build of the same library (A/B measurement of kernel variants)
LIB_PATH = os.environ.get("ISAX_LIB") or os.path.join(_HERE, "libisax.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing. Build it with `python -m paper_2009_01614_b200.build`; "
                      "there is no CPU fallback.")

_lib = ctypes.CDLL(LIB_PATH)
_P, _U64, _U32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32

ISAX_OK = 0
ERRORS = {-1: "ISAX_E_INVAL", -2: "ISAX_E_EMPTY", -3: "ISAX_E_UNSUPPORTED", -4: "ISAX_E_NOMEM", -5: "ISAX_E_CUDA",
          -6: "ISAX_E_NONFINITE", -7: "ISAX_E_CALLBACK", -8: "ISAX_E_IO"}


class Opts(ctypes.Structure):
    _fields_ = [("window_L", ctypes.c_uint32), ("slack_log2", ctypes.c_int32), ("batch_Q", ctypes.c_uint32),
                ("cand_cap", ctypes.c_uint32), ("flags", ctypes.c_uint32), ("probe_bits", ctypes.c_uint32),
                ("probe_L", ctypes.c_uint32), ("first_band", ctypes.c_float)]


def _sig(name, args, res=ctypes.c_int):
    f = getattr(_lib, name)
    f.argtypes = args
    f.restype = res
    return f


isax_build = _sig("isax_build", [_P, _U64, _U32, _U32, _U32, _P, ctypes.POINTER(_P)])
isax_build_stream = _sig("isax_build_stream", [_U64, _U32, _U32, _U32, _P, _P, _U64, _P, ctypes.POINTER(_P)])
isax_nn1 = _sig("isax_nn1", [_P, _P, _U32, _P, _P])
isax_nn1_async = _sig("isax_nn1_async", [_P, _P, _U32, _P, _P, _P])
isax_export = _sig("isax_export", [_P, _U64, _U64, _P, _P, _P])
isax_query_debug = _sig("isax_query_debug", [_P, _P, _U32, _P, _P, _P, _U64, _U64, _P, _P])
isax_debug_candidates = _sig("isax_debug_candidates", [_P, _U32, _P, _U64, ctypes.POINTER(_U64)])
isax_stats = _sig("isax_stats", [_P, ctypes.c_char_p, ctypes.c_size_t])
isax_debug_plan_round = _sig("isax_debug_plan_round", [_P, _P, _P, _U32, _U32, _P, ctypes.c_int, ctypes.c_float,
                                                       ctypes.c_float, _U32])
isax_info = _sig("isax_info", [_P, ctypes.POINTER(_U64), ctypes.POINTER(_U32), ctypes.POINTER(_U32),
                               ctypes.POINTER(_U32), ctypes.POINTER(_U64)])
isax_debug_bounds = _sig("isax_debug_bounds", [ctypes.c_int])
isax_save = _sig("isax_save", [_P, ctypes.c_char_p])
isax_load = _sig("isax_load", [ctypes.c_char_p, _P, ctypes.POINTER(_P)])
isax_free = _sig("isax_free", [_P], None)
isax_last_error = _sig("isax_last_error", [], ctypes.c_char_p)
isax_version = _sig("isax_version", [], ctypes.c_char_p)


class IsaxError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        self.name = ERRORS.get(code, str(code))
        msg = (isax_last_error() or b"").decode()
        super().__init__(f"{where}: {self.name}: {msg}")


def _check(rc: int, where: str):
    if rc != ISAX_OK:
        raise IsaxError(rc, where)


def _ptr(a):
    """Device or host address of a torch tensor or numpy array (must be contiguous)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"]
        return ctypes.c_void_p(a.ctypes.data)
    assert a.is_contiguous()
    return ctypes.c_void_p(a.data_ptr())


FLAG_FLAT_SCAN = 1  # include/isax.h ISAX_FLAG_FLAT_SCAN
PROBES_NONE = 0xFFFFFFFF  # include/isax.h ISAX_PROBES_NONE


def _opts(window_L=0, slack_log2=0, batch_Q=0, cand_cap=0, flags=0, probe_bits=0, probe_L=0, first_band=0.0):
    return Opts(window_L, slack_log2, batch_Q, cand_cap, flags, probe_bits, probe_L, first_band)


class Index:
    """An iSAX index on the current CUDA device (isax_build / isax_build_stream)."""

    def __init__(self, handle: int, keep=None):
        self._h = ctypes.c_void_p(handle)
        self._keep = keep
        N, n, w, c, b = _U64(), _U32(), _U32(), _U32(), _U64()
        _check(isax_info(self._h, ctypes.byref(N), ctypes.byref(n), ctypes.byref(w), ctypes.byref(c), ctypes.byref(b)),
               "isax_info")
        self.N, self.n, self.w, self.card, self.device_bytes = N.value, n.value, w.value, c.value, b.value

    # -- construction --------------------------------------------------------------------------
    @classmethod
    def build(cls, series, w: int = 16, card: int = 256, **opts):
        """series: torch tensor (CUDA or CPU) or numpy array, fp32 [N, n], raw values."""
        if isinstance(series, np.ndarray):
            series = np.ascontiguousarray(series, dtype=np.float32)
        else:
            import torch

            if series.dtype != torch.float32:
                raise TypeError(f"series must be float32, got {series.dtype}")
            series = series.contiguous()
        if series.ndim != 2:
            raise ValueError(f"series must be [N, n], got shape {tuple(series.shape)}")
        N, n = series.shape
        h = _P()
        o = _opts(**opts)
        _check(isax_build(_ptr(series), N, n, w, card, ctypes.byref(o), ctypes.byref(h)), "isax_build")
        return cls(h.value)

    @classmethod
    def build_stream(cls, N: int, n: int, fill_ptr, ctx, chunk: int = 0, w: int = 16, card: int = 256, **opts):
        """fill_ptr: an isax_fill_fn C function pointer; ctx: a ctypes object passed by reference."""
        h = _P()
        o = _opts(**opts)
        _check(isax_build_stream(N, n, w, card, fill_ptr, ctypes.cast(ctypes.pointer(ctx), _P), chunk, ctypes.byref(o),
                                 ctypes.byref(h)), "isax_build_stream")
        return cls(h.value, keep=ctx)

    @classmethod
    def load(cls, path: str, **opts):
        """isax_load: an index saved by save(), onto the current CUDA device."""
        h = _P()
        o = _opts(**opts)
        _check(isax_load(os.fsencode(path), ctypes.byref(o), ctypes.byref(h)), "isax_load")
        return cls(h.value)

    def save(self, path: str):
        """isax_save: the whole index (rows, words, permutation, node summaries) to a file."""
        _check(isax_save(self._h, os.fsencode(path)), "isax_save")

    # -- queries -------------------------------------------------------------------------------
    def nn1_bound(self, queries, out_id, out_dist, stream):
        """A zero-argument callable that runs isax_nn1_async on fixed device buffers (the C ABI call
        itself, with its arguments marshalled once): for tight serving or timing loops."""
        args = (self._h, _ptr(queries), ctypes.c_uint32(queries.shape[0]), _ptr(out_id), _ptr(out_dist),
                ctypes.c_void_p(stream))
        fn = isax_nn1_async

        def call():
            rc = fn(*args)
            if rc != ISAX_OK:
                raise IsaxError(rc, "isax_nn1_async")
        return call

    def nn1(self, queries, out_id=None, out_dist=None, stream=None):
        """Exact 1-NN of raw queries [Q, n].

        CUDA tensor in -> isax_nn1_async on `stream` (default: torch's current stream), with
        CUDA outputs. numpy / CPU tensor in -> isax_nn1 (synchronous, host outputs).
        Returns (ids int64 [Q], dist fp32 [Q]).
        """
        import torch

        if isinstance(queries, np.ndarray):
            queries = torch.from_numpy(np.ascontiguousarray(queries, dtype=np.float32))
        queries = queries.contiguous()
        Q = queries.shape[0]
        assert queries.dtype == torch.float32 and queries.shape[1] == self.n
        dev = queries.device
        if out_id is None:
            out_id = torch.empty(Q, dtype=torch.int64, device=dev, pin_memory=False)
        if out_dist is None:
            out_dist = torch.empty(Q, dtype=torch.float32, device=dev)
        if dev.type == "cuda":
            s = torch.cuda.current_stream().cuda_stream if stream is None else stream
            _check(isax_nn1_async(self._h, _ptr(queries), Q, _ptr(out_id), _ptr(out_dist), ctypes.c_void_p(s)),
                   "isax_nn1_async")
        else:
            _check(isax_nn1(self._h, _ptr(queries), Q, _ptr(out_id), _ptr(out_dist)), "isax_nn1")
        return out_id, out_dist

    def nn1_host(self, queries_host, out_id_host, out_dist_host):
        """isax_nn1 on caller-provided host buffers (pinned or pageable); used by the e2e bench."""
        Q = queries_host.shape[0]
        _check(isax_nn1(self._h, _ptr(queries_host), Q, _ptr(out_id_host), _ptr(out_dist_host)), "isax_nn1")

    # -- inspection ----------------------------------------------------------------------------
    def export(self, first_id: int = 0, count: int | None = None, sax: bool = True, perm: bool = False,
               stored: bool = False):
        """Return dict with 'sax' [count, w] u8 (by id), 'perm' [N] u32, 'stored' [count, n] fp32 (by position)."""
        count = self.N - first_id if count is None else count
        out = {}
        a_sax = np.empty((count, self.w), np.uint8) if sax else None
        a_perm = np.empty(self.N, np.uint32) if perm else None
        a_st = np.empty((count, self.n), np.float32) if stored else None
        _check(isax_export(self._h, first_id, count, _ptr(a_sax), _ptr(a_perm), _ptr(a_st)), "isax_export")
        if sax:
            out["sax"] = a_sax
        if perm:
            out["perm"] = a_perm
        if stored:
            out["stored"] = a_st
        return out

    def query_debug(self, queries, first_pos: int = 0, count: int = 0):
        """Return dict: q_paa [Q,w] f64, q_sax [Q,w] u8, lut [Q,w,card] f32, lb2 [Q,count] f32, win [Q,2] u32."""
        q = np.ascontiguousarray(queries, dtype=np.float32)
        Q = q.shape[0]
        r = {"q_paa": np.empty((Q, self.w)), "q_sax": np.empty((Q, self.w), np.uint8),
             "lut": np.empty((Q, self.w, self.card), np.float32), "win": np.empty((Q, 2), np.uint32)}
        lb = np.empty((Q, count), np.float32) if count else None
        _check(isax_query_debug(self._h, _ptr(q), Q, _ptr(r["q_paa"]), _ptr(r["q_sax"]), _ptr(r["lut"]), first_pos,
                                count, _ptr(lb), _ptr(r["win"])), "isax_query_debug")
        if count:
            r["lb2"] = lb
        return r

    def candidates(self, q: int):
        """Sorted positions of query q's candidate list in the last nn1 call (isax_debug_candidates)."""
        cnt = _U64()
        _check(isax_debug_candidates(self._h, q, None, 0, ctypes.byref(cnt)), "isax_debug_candidates")
        out = np.empty(cnt.value, np.uint32)
        _check(isax_debug_candidates(self._h, q, _ptr(out), cnt.value, ctypes.byref(cnt)), "isax_debug_candidates")
        return out

    def stats(self) -> dict:
        need = isax_stats(self._h, None, 0)
        if need < 0:
            _check(need, "isax_stats")
        buf = ctypes.create_string_buffer(need + 1)
        isax_stats(self._h, buf, need + 1)
        return json.loads(buf.value.decode())

    def close(self):
        if self._h is not None and self._h.value:
            isax_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


PLAN_DONE, PLAN_AGAIN, PLAN_RESCAN, PLAN_ERROR = 0, 1, 2, -1


def plan_round(band, pos, state, cand_cnt: int, cap: int, hist, near_ovf: bool, tused: float, bsf_lim: float, N: int):
    """One step of the per-query round plan (isax_debug_plan_round; host logic, no device).

    band: float32[2] (lo, hi], pos: uint32[2] [plo, phi), state: uint32[2] (next range length,
    first-bin overflows), all updated in place; hist: uint32[64]. Returns the action code."""
    for a, dt in ((band, np.float32), (pos, np.uint32), (state, np.uint32)):
        assert isinstance(a, np.ndarray) and a.dtype == dt and a.shape == (2,)
    hist = np.ascontiguousarray(hist, dtype=np.uint32)
    assert hist.shape == (64,)
    return isax_debug_plan_round(_ptr(band), _ptr(pos), _ptr(state), cand_cnt, cap, _ptr(hist), int(near_ovf),
                                 float(tused), float(bsf_lim), N)


def version() -> str:
    return isax_version().decode()
