#!/usr/bin/env python3
"""Kernel time of one thresholded LCS plot of random sigma-letter strings (device API):
  python tools/sigma_step.py --sigma 20 --w 128 --m 32768"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_0909_2000_b200 import _native  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sigma", type=int, default=20)
    ap.add_argument("--w", type=int, default=128)
    ap.add_argument("--m", type=int, default=32768)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--r", type=int, default=1)
    a = ap.parse_args()
    rng = np.random.default_rng(a.sigma * 1000 + a.w)
    x = rng.integers(1, a.sigma + 1, a.m).astype(np.uint8)
    y = rng.integers(1, a.sigma + 1, a.m).astype(np.uint8)
    L = _native.lib()
    ctx = ctypes.c_void_p()
    assert L.ap_ctx_create(0, ctypes.byref(ctx)) == 0
    cfg = _native.ApConfig(window_w=a.w, step_h=1, blowup_r=a.r, has_threshold=1, threshold_half=2 * a.w - 8,
                           n_devices=1, row_begin=0, row_end=0)
    dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    cap = 1 << 20
    r_ = torch.empty(cap, dtype=torch.int32, device="cuda")
    c_ = torch.empty(cap, dtype=torch.int32, device="cuda")
    h_ = torch.empty(cap, dtype=torch.int16, device="cuda")
    cnt = ctypes.c_uint64()
    for _ in range(a.reps):
        rc = L.ap_ctx_plot_threshold_device(ctx, dx.data_ptr(), x.size, dy.data_ptr(), y.size, ctypes.byref(cfg),
                                            ctypes.byref(cnt), r_.data_ptr(), c_.data_ptr(), h_.data_ptr(), cap, None)
        assert rc in (0, _native.AP_CAPACITY), _native.last_error()
        torch.cuda.synchronize()
        print(f"sigma={a.sigma} w={a.w} r={a.r} m={a.m} {(L.ap_ctx_last_kernel(ctx) or b'').decode()} "
              f"kernel_ms={L.ap_ctx_last_kernel_ms(ctx):.3f} hits={cnt.value}", flush=True)
    L.ap_ctx_destroy(ctx)


if __name__ == "__main__":
    main()
