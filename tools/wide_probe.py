#!/usr/bin/env python3
"""Large-window path timing: seeded DNA / protein strips with blown windows above 1024,
through the device API (kernel time = ap_ctx_last_kernel_ms), comb cells/s and the ALU-op rate.

  python tools/wide_probe.py [--rows 1184] [--n 40000]
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_0909_2000_b200 import _native, datagen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1184)
    ap.add_argument("--n", type=int, default=40000)
    a = ap.parse_args()
    L = _native.lib()
    ctx = ctypes.c_void_p()
    assert L.ap_ctx_create(0, ctypes.byref(ctx)) == 0
    for w, r, alpha in ((2048, 1, datagen.DNA), (20000, 1, datagen.DNA), (4096, 2, datagen.DNA),
                        (2048, 1, datagen.PROTEIN)):
        x = datagen.uniform(7, 0, w + a.rows - 1, alpha)
        y = datagen.uniform(7, 1, a.n, alpha)
        rows, cols = a.rows, y.size - w + 1
        cfg = _native.ApConfig(window_w=w, step_h=1, blowup_r=r, has_threshold=0, threshold_half=0, n_devices=1,
                               row_begin=0, row_end=0)
        dx, dy = torch.from_numpy(x.copy()).cuda(), torch.from_numpy(y.copy()).cuda()
        out = torch.empty(rows * cols, dtype=torch.int16, device="cuda")
        for rep in range(2):
            rc = L.ap_ctx_plot_dense_device(ctx, dx.data_ptr(), x.size, dy.data_ptr(), y.size, ctypes.byref(cfg),
                                            out.data_ptr(), None)
            assert rc == 0, _native.last_error()
        ms = L.ap_ctx_last_kernel_ms(ctx)
        cells = rows * (w * r) * (y.size * r)
        kern = (L.ap_ctx_last_kernel(ctx) or b"").decode()
        ops = 1.0 if kern.endswith(",packed>") else 2.0 if ",table" in kern else 3.0
        frac = cells * ops / (ms / 1e3) / (148 * 63.41 * 1.965e9)
        print(f"w={w} r={r} sigma={alpha.size} rows={rows} n={y.size} kernel={kern} {ms:.2f} ms "
              f"{cells / (ms / 1e3):.3e} comb cells/s, ALU-op frac {frac:.3f}", flush=True)
    L.ap_ctx_destroy(ctx)


if __name__ == "__main__":
    main()
