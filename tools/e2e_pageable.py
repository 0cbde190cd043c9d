#!/usr/bin/env python3
"""Dense host API (ap_plot_dense) end to end into pinned vs pageable (numpy) host buffers, and the
bare D2H of the same bytes both ways: how much a caller without pinned memory loses.

  python tools/e2e_pageable.py [--config C2] [--reps 5]
"""
import argparse
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_0909_2000_b200 import _native, datagen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    c = datagen.CONFIGS[a.config]
    x, y = datagen.make_inputs(a.config)
    L = _native.lib()
    cfg = _native.ApConfig(window_w=c.w, step_h=c.h, blowup_r=c.r, has_threshold=0, threshold_half=0,
                           n_devices=1, row_begin=0, row_end=0)
    rows, cols = (x.size - c.w) // c.h + 1, y.size - c.w + 1
    nbytes = rows * cols * 2
    pinned = torch.empty(rows * cols, dtype=torch.int16).pin_memory()
    pageable = np.empty(rows * cols, dtype=np.uint16)
    pageable[:] = 1   # touch the pages
    xa, ya = np.ascontiguousarray(x), np.ascontiguousarray(y)

    def run(ptr):
        rc = L.ap_plot_dense(xa.ctypes.data, x.size, ya.ctypes.data, y.size, ctypes.byref(cfg), ptr)
        assert rc == 0, _native.last_error()

    for name, ptr in (("pinned", pinned.data_ptr()), ("pageable", pageable.ctypes.data)):
        run(ptr)
        t0 = time.perf_counter()
        for _ in range(a.reps):
            run(ptr)
        dt = (time.perf_counter() - t0) / a.reps
        print(f"{a.config} ap_plot_dense into {name}: {dt * 1e3:.2f} ms/plot ({nbytes / dt / 1e9:.1f} GB/s of plot)")
    assert np.array_equal(pinned.numpy().view(np.uint16), pageable)
    d = torch.empty(rows * cols, dtype=torch.int16, device="cuda")
    for name, dst in (("pinned", pinned), ("pageable", torch.from_numpy(pageable.view(np.int16)))):
        dst.copy_(d)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(a.reps):
            dst.copy_(d)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / a.reps
        print(f"bare D2H of {nbytes / 1e6:.0f} MB into {name}: {dt * 1e3:.2f} ms ({nbytes / dt / 1e9:.1f} GB/s)")


if __name__ == "__main__":
    main()
