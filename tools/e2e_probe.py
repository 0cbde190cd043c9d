#!/usr/bin/env python3
"""Where the dense end-to-end time goes (C2 by default): the host API call with pinned
buffers, versus device compute followed by one D2H, versus the D2H alone.

  python tools/e2e_probe.py [--config C2] [--reps 5]
"""
import argparse
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

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
    hx = torch.from_numpy(x.copy()).pin_memory()
    hy = torch.from_numpy(y.copy()).pin_memory()
    hout = torch.empty(rows * cols, dtype=torch.int16).pin_memory()
    dx, dy = hx.cuda(), hy.cuda()
    dout = torch.empty(rows * cols, dtype=torch.int16, device="cuda")
    ctx = ctypes.c_void_p()
    assert L.ap_ctx_create(0, ctypes.byref(ctx)) == 0
    s = torch.cuda.Stream()

    def host_api():
        assert L.ap_plot_dense(hx.data_ptr(), x.size, hy.data_ptr(), y.size, ctypes.byref(cfg), hout.data_ptr()) == 0

    hout8 = torch.empty(rows * cols, dtype=torch.uint8).pin_memory()

    def host_api_u8():
        assert L.ap_plot_dense_u8(hx.data_ptr(), x.size, hy.data_ptr(), y.size, ctypes.byref(cfg),
                                  hout8.data_ptr()) == 0

    def dev_then_copy():
        assert L.ap_ctx_plot_dense_device(ctx, dx.data_ptr(), x.size, dy.data_ptr(), y.size, ctypes.byref(cfg),
                                          dout.data_ptr(), s.cuda_stream) == 0
        with torch.cuda.stream(s):
            hout.copy_(dout, non_blocking=True)
        s.synchronize()

    def dev_only():
        assert L.ap_ctx_plot_dense_device(ctx, dx.data_ptr(), x.size, dy.data_ptr(), y.size, ctypes.byref(cfg),
                                          dout.data_ptr(), s.cuda_stream) == 0
        s.synchronize()

    def copy_only():
        with torch.cuda.stream(s):
            hout.copy_(dout, non_blocking=True)
        s.synchronize()

    s2 = torch.cuda.Stream()
    dout2 = torch.empty_like(dout)
    hout2 = torch.empty_like(hout).pin_memory()

    def d2h_chunked(k=16):
        n = hout.numel()
        with torch.cuda.stream(s):
            for i in range(k):
                hout[i * n // k:(i + 1) * n // k].copy_(dout[i * n // k:(i + 1) * n // k], non_blocking=True)
        s.synchronize()

    def d2h_during_compute():
        # the D2H of one buffer while the comb kernel writes another (streams overlap)
        assert L.ap_ctx_plot_dense_device(ctx, dx.data_ptr(), x.size, dy.data_ptr(), y.size, ctypes.byref(cfg),
                                          dout2.data_ptr(), s.cuda_stream) == 0
        with torch.cuda.stream(s2):
            hout.copy_(dout, non_blocking=True)
        s2.synchronize()
        s.synchronize()

    for name, fn in (("d2h_16_chunks", d2h_chunked), ("d2h_while_comb", d2h_during_compute),
                     ("host_api", host_api), ("host_api_u8", host_api_u8), ("device_then_d2h", dev_then_copy), ("device_only", dev_only),
                     ("d2h_only", copy_only)):
        fn()
        t = []
        for _ in range(a.reps):
            t0 = time.perf_counter()
            fn()
            t.append((time.perf_counter() - t0) * 1e3)
        print(f"{name:16s} ms: min {min(t):.3f} median {sorted(t)[len(t) // 2]:.3f}")
    L.ap_ctx_destroy(ctx)


if __name__ == "__main__":
    main()
