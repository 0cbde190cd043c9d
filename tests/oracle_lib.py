"""ctypes access to the parity checkers (TEST INFRASTRUCTURE).

* ``oracle/liboracle.so``           — the C restatement (oracle/alignplot_oracle.c)
* ``oracle/_ref/libalignplot_ref.so`` — the unmodified reference library (oracle/Makefile)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm load these.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_int, c_int32, c_int64, c_size_t, c_uint, c_uint64, c_void_p

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libalignplot_ref.so")

_or = None
_ref = None


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


def oracle():
    global _or
    if _or is None:
        if not os.path.exists(ORACLE_SO):
            import subprocess
            subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), os.path.join(ROOT, "oracle", "liboracle.so")],
                           check=True, capture_output=True)
        L = ctypes.CDLL(ORACLE_SO)
        L.or_window_grid_dims.argtypes = [c_size_t] * 4 + [POINTER(c_size_t)] * 2
        L.or_validate.argtypes = [c_size_t, c_size_t, c_size_t, c_size_t, c_uint, c_uint, c_int]
        L.or_blowup.argtypes = [c_void_p, c_size_t, c_void_p]
        L.or_recover_score.argtypes = [c_size_t, c_size_t, c_size_t]
        L.or_recover_score.restype = c_int32
        L.or_comb_strip.argtypes = [c_void_p, c_size_t, c_void_p, c_size_t, c_void_p, c_void_p]
        L.or_comb_strip.restype = None
        L.or_llcs_query.argtypes = [c_void_p, c_size_t, c_void_p, c_size_t, c_size_t, c_size_t, POINTER(c_size_t)]
        L.or_window_llcs_from_events.argtypes = [c_void_p, c_size_t, c_size_t, c_size_t, c_void_p]
        L.or_plot_rows.argtypes = [c_void_p, c_size_t, c_void_p, c_size_t, c_size_t, c_size_t, c_uint,
                                   c_size_t, c_size_t, c_uint, c_void_p]
        L.or_apply_threshold.argtypes = [c_void_p, c_size_t, c_size_t, c_int32, c_void_p, c_void_p, c_void_p, c_size_t]
        L.or_apply_threshold.restype = c_size_t
        L.or_ref_llcs.argtypes = [c_void_p, c_size_t, c_void_p, c_size_t]
        L.or_ref_llcs.restype = c_size_t
        L.or_ref_align_score_half.argtypes = [c_void_p, c_size_t, c_void_p, c_size_t]
        L.or_ref_align_score_half.restype = c_int32
        _or = L
    return _or


def u8(a) -> np.ndarray:
    if isinstance(a, (bytes, bytearray)):
        return np.frombuffer(bytes(a), dtype=np.uint8).copy()
    if isinstance(a, str):
        return np.frombuffer(a.encode("latin-1"), dtype=np.uint8).copy()
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint8))


def grid_dims(m, n, w, h):
    r, c = c_size_t(), c_size_t()
    rc = oracle().or_window_grid_dims(m, n, w, h, ctypes.byref(r), ctypes.byref(c))
    return rc, r.value, c.value


def comb_strip(xw, y):
    """Bottom-event starts (and right-exit starts) of the scalar comb."""
    xw, y = u8(xw), u8(y)
    bs = np.empty(y.size, dtype=np.int32)
    rs = np.empty(xw.size, dtype=np.int32)
    oracle().or_comb_strip(_p(xw), xw.size, _p(y), y.size, _p(bs), _p(rs))
    return bs, rs


def window_llcs(starts, window_cols, stride=1):
    starts = np.ascontiguousarray(starts, dtype=np.int32)
    n = starts.size
    if stride == 0 or window_cols == 0 or window_cols > n:
        out = np.empty(1, dtype=np.uint64)
    else:
        out = np.empty((n - window_cols) // stride + 1, dtype=np.uint64)
    rc = oracle().or_window_llcs_from_events(_p(starts), n, window_cols, stride, _p(out))
    return rc, out


def plot_rows(x, y, w, h, r, row_begin=0, row_end=None, workers=8):
    """Oracle grid (int32 half-units) for rows [row_begin, row_end)."""
    x, y = u8(x), u8(y)
    rc, rows, cols = grid_dims(x.size, y.size, w, h)
    if rc:
        return rc, None
    re = rows if row_end is None else min(row_end, rows)
    out = np.zeros((max(re - row_begin, 0), cols), dtype=np.int32)
    rc = oracle().or_plot_rows(_p(x), x.size, _p(y), y.size, w, h, r, row_begin, re, workers, _p(out))
    return rc, out


def ref_llcs(a, b):
    a, b = u8(a), u8(b)
    return oracle().or_ref_llcs(_p(a), a.size, _p(b), b.size)


def ref_align_score_half(a, b):
    a, b = u8(a), u8(b)
    return oracle().or_ref_align_score_half(_p(a), a.size, _p(b), b.size)


# ---- the reference library itself (oracle/_ref) ----------------------------
def ref_available() -> bool:
    return os.path.exists(REF_SO)


def reflib():
    global _ref
    if _ref is None:
        L = ctypes.CDLL(REF_SO)
        L.ref_compute_plot.argtypes = [c_void_p, c_size_t, c_void_p, c_size_t, c_size_t, c_size_t, c_uint, c_int,
                                       c_uint, c_void_p, c_size_t, POINTER(c_size_t), POINTER(c_size_t),
                                       c_char_p, c_size_t]
        L.ref_lane_window_llcs.argtypes = [c_void_p, c_size_t, c_void_p, c_size_t, c_size_t, c_uint, c_uint,
                                           c_void_p, c_char_p, c_size_t]
        L.ref_comb_strip.argtypes = [c_void_p, c_size_t, c_void_p, c_size_t, c_void_p]
        _ref = L
    return _ref


SEA8, SEA16 = 4, 3


def ref_compute_plot(x, y, w, h, r, mode=SEA8, workers=8):
    """Reference compute_plot (int32 grid) on the full inputs; returns (rc, grid 2-D or None, err)."""
    x, y = u8(x), u8(y)
    rc0, rows, cols = grid_dims(x.size, y.size, w, h) if (w and h) else (1, 0, 0)
    cap = max(rows * cols, 1)
    out = np.zeros(cap, dtype=np.int32)
    rr, cc = c_size_t(), c_size_t()
    err = ctypes.create_string_buffer(512)
    rc = reflib().ref_compute_plot(_p(x), x.size, _p(y), y.size, w, h, r, mode, workers, _p(out), cap,
                                   ctypes.byref(rr), ctypes.byref(cc), err, 512)
    if rc:
        return rc, None, err.value.decode()
    return 0, out[: rr.value * cc.value].reshape(rr.value, cc.value), ""


def ref_plot_rows(x, y, w, h, r, row_begin, row_end, mode=SEA8, workers=8):
    """Reference grid rows [row_begin, row_end) via compute_plot on the x slice."""
    x = u8(x)
    xs = x[row_begin * h: (row_end - 1) * h + w]
    return ref_compute_plot(xs, y, w, h, r, mode, workers)
