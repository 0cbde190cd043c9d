#!/usr/bin/env python3
"""One or more plot steps of a config through the device API, for ncu / launch lists.

  python tools/prof_step.py --config C3 [--rows N] [--reps 2]

--rows limits the grid rows (row_end) so an ncu --set full replay stays short.
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_0909_2000_b200 import _native, datagen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--rows", type=int, default=0)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    c = datagen.CONFIGS[a.config]
    x, y = datagen.make_inputs(a.config)
    L = _native.lib()
    ctx = ctypes.c_void_p()
    assert L.ap_ctx_create(0, ctypes.byref(ctx)) == 0
    rows = (x.size - c.w) // c.h + 1
    re = min(rows, a.rows) if a.rows else 0
    cfg = _native.ApConfig(window_w=c.w, step_h=c.h, blowup_r=c.r, has_threshold=int(c.t_half is not None),
                           threshold_half=c.t_half or 0, n_devices=1, row_begin=0, row_end=re)
    nrows = re or rows
    dx = torch.from_numpy(x.copy()).cuda()
    dy = torch.from_numpy(y.copy()).cuda()
    cols = y.size - c.w + 1
    cnt = ctypes.c_uint64()
    if c.t_half is None:
        out = torch.empty(nrows * cols, dtype=torch.int16, device="cuda")
    else:
        cap = 1 << 20
        r_ = torch.empty(cap, dtype=torch.int32, device="cuda")
        c_ = torch.empty(cap, dtype=torch.int32, device="cuda")
        h_ = torch.empty(cap, dtype=torch.int16, device="cuda")
    for _ in range(a.reps):
        if c.t_half is None:
            rc = L.ap_ctx_plot_dense_device(ctx, dx.data_ptr(), x.size, dy.data_ptr(), y.size, ctypes.byref(cfg),
                                            out.data_ptr(), None)
        else:
            rc = L.ap_ctx_plot_threshold_device(ctx, dx.data_ptr(), x.size, dy.data_ptr(), y.size, ctypes.byref(cfg),
                                                ctypes.byref(cnt), r_.data_ptr(), c_.data_ptr(), h_.data_ptr(), cap, None)
        assert rc in (0, _native.AP_CAPACITY), _native.last_error()
        torch.cuda.synchronize()
        print(f"{a.config} rows={nrows} kernel_ms={L.ap_ctx_last_kernel_ms(ctx):.3f} hits={cnt.value}", flush=True)
    L.ap_ctx_destroy(ctx)


if __name__ == "__main__":
    main()
