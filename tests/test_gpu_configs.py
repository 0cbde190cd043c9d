"""GPU parity at the five BASELINE.json configs' full sizes against the reference library itself.

The checker is ``oracle/_ref`` -- the unmodified reference ``compute_plot`` (runner.cpp:78-131)
compiled from /root/reference by oracle/Makefile -- run on row blocks of each config's plot
(SURVEY.md §8c/§8d): engine sea8 for C1-C4, sea16 for C5 (sea8 rejects w = 256,
model.cpp:53-56), all host cores.  Thresholded lists are compared with apply_threshold
(scoring.cpp:30-39) of the reference rows, element by element.

  C1, C2  full grids
  C3      full grid in row blocks, and the full thresholded lists (t_half 192 = the config's
          WLCS >= 96, which uniform DNA almost never reaches, and 176 for ~1e6 hits)
  C4, C5  4096 evenly spaced rows (64 blocks of 64): dense scores, and the full-plot
          thresholded list restricted to those rows
"""
import os

import numpy as np
import pytest

import oracle_lib as ol
from paper_0909_2000_b200 import alignplot as ap
from paper_0909_2000_b200 import datagen

pytestmark = pytest.mark.gpu

CORES = os.cpu_count() or 8


def cfg(c, t=None):
    return ap.PlotConfig(window_w=c.w, step_h=c.h, blowup_r=c.r, threshold_half=t, mode=ap.Mode.cuda)


def ref_mode(c):
    return ol.SEA8 if c.w <= 254 else ol.SEA16


def ref_rows(x, y, c, rb, re):
    rc, g, err = ol.ref_plot_rows(x, y, c.w, c.h, c.r, rb, re, ref_mode(c), CORES)
    assert rc == 0, err
    return g


def list_rows(lst, rb, re):
    """The part of a row-major (rows, cols, halves) list in grid rows [rb, re)."""
    r, k, h = lst
    i0, i1 = np.searchsorted(r, rb), np.searchsorted(r, re)
    return r[i0:i1].astype(np.int64) - rb, k[i0:i1].astype(np.int64), h[i0:i1].astype(np.int16).astype(np.int32)


def assert_list_matches(lst, g, rb, re, t, what):
    gr, gc, gh = list_rows(lst, rb, re)
    er, ec = np.nonzero(g >= t)
    assert gr.size == er.size, (what, rb, gr.size, er.size)
    assert np.array_equal(gr, er) and np.array_equal(gc, ec) and np.array_equal(gh, g[er, ec]), (what, rb)


@pytest.fixture(scope="module", autouse=True)
def _need_reference():
    assert ol.ref_available(), "oracle/_ref/libalignplot_ref.so missing: run make (it travels with the repo)"


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_full_grid_vs_reference(name):
    """C1 (2000^2, LCS) and C2 (16384^2 alignment score, 530 MB of uint16) whole grids."""
    c = datagen.CONFIGS[name]
    x, y = datagen.make_inputs(name)
    got = ap.plot_dense_u16(x, y, cfg(c))
    rows = got.shape[0]
    blk = 2048
    for rb in range(0, rows, blk):
        re = min(rows, rb + blk)
        g = ref_rows(x, y, c, rb, re)
        assert np.array_equal(got[rb:re].astype(np.int32), g), (name, rb)


def test_c3_full_grid_and_lists_vs_reference():
    """C3 (65409^2 LCS, w = 128): every row block of the dense grid, and the two full-plot
    thresholded lists (one call each; they run with the tail split of the last wave)."""
    c = datagen.CONFIGS["C3"]
    x, y = datagen.make_inputs("C3")
    rows = (x.size - c.w) // c.h + 1
    lists = {t: ap.plot_threshold_arrays(x, y, cfg(c), t) for t in (c.t_half, 176)}
    assert lists[176][0].size > 100000
    blk = 1024
    for rb in range(0, rows, blk):
        re = min(rows, rb + blk)
        g = ref_rows(x, y, c, rb, re)
        got = ap.plot_dense_u16(x, y, cfg(c), rb, re)
        assert np.array_equal(got.astype(np.int32), g), rb
        for t, lst in lists.items():
            assert_list_matches(lst, g, rb, re, t, f"C3 t={t}")
    for t, lst in lists.items():   # nothing outside the grid
        assert lst[0].size == 0 or int(lst[0][-1]) < rows


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_sampled_rows_vs_reference(name):
    """C4 (262081^2 alignment score, sigma = 20) and C5 (1048321^2 LCS, w = 256): 4096 evenly
    spaced rows -- dense scores and the config's full thresholded list on those rows."""
    c = datagen.CONFIGS[name]
    x, y = datagen.make_inputs(name)
    rows = (x.size - c.w) // c.h + 1
    lst = ap.plot_threshold_arrays(x, y, cfg(c), c.t_half)
    assert lst[0].size > 1000
    key = lst[0].astype(np.int64) * (1 << 32) + lst[1]
    assert np.all(np.diff(key) > 0)   # strictly row-major
    blk, nblk = 64, 64
    starts = np.linspace(0, rows - blk, nblk).astype(np.int64)
    checked = 0
    for rb in starts:
        rb = int(rb)
        re = rb + blk
        g = ref_rows(x, y, c, rb, re)
        got = ap.plot_dense_u16(x, y, cfg(c), rb, re)
        assert np.array_equal(got.astype(np.int32), g), (name, rb)
        assert_list_matches(lst, g, rb, re, c.t_half, name)
        checked += int(np.count_nonzero(g >= c.t_half))
    assert checked > 0


def test_c4_count_only_beyond_2_pow_32():
    """A count-only query (cap = 0) with a threshold below every score on the full C4 plot: the
    count is rows * cols = 262081^2 = 68,686,450,561 > 2^32, exact through the 64-bit scan, and no
    list is staged (a uint32 scan would wrap).  Through the device API and the host API
    (which then reports AP_CAPACITY with the exact count)."""
    import ctypes

    import torch

    from paper_0909_2000_b200 import _native
    c = datagen.CONFIGS["C4"]
    x, y = datagen.make_inputs("C4")
    rows, cols = (x.size - c.w) // c.h + 1, y.size - c.w + 1
    L = _native.lib()
    cc = ap._cfg(cfg(c, -100))
    count = ctypes.c_uint64()
    ctx = ctypes.c_void_p()
    assert L.ap_ctx_create(0, ctypes.byref(ctx)) == 0
    try:
        dx, dy = torch.from_numpy(x.copy()).cuda(), torch.from_numpy(y.copy()).cuda()
        rc = L.ap_ctx_plot_threshold_device(ctx, dx.data_ptr(), x.size, dy.data_ptr(), y.size, ctypes.byref(cc),
                                            ctypes.byref(count), None, None, None, 0, None)
        assert rc == _native.AP_CAPACITY and count.value == rows * cols > 2 ** 32
    finally:
        L.ap_ctx_destroy(ctx)
    count2 = ctypes.c_uint64()
    rc = L.ap_plot_threshold(x.ctypes.data, x.size, y.ctypes.data, y.size, ctypes.byref(cc), ctypes.byref(count2),
                             None, None, None, 0)
    assert rc == _native.AP_CAPACITY and count2.value == rows * cols
    # and the config's own threshold, count-only, equals the length of its list
    cc = ap._cfg(cfg(c, c.t_half))
    rc = L.ap_plot_threshold(x.ctypes.data, x.size, y.ctypes.data, y.size, ctypes.byref(cc), ctypes.byref(count2),
                             None, None, None, 0)
    assert rc == _native.AP_CAPACITY and count2.value == ap.plot_threshold_arrays(x, y, cfg(c), c.t_half)[0].size
