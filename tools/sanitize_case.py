#!/usr/bin/env python3
"""Small dense + threshold runs of every kernel family for compute-sanitizer (one tool per call)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0909_2000_b200 import alignplot as ap  # noqa: E402

rng = np.random.default_rng(3)
x = rng.integers(1, 5, 300).astype(np.uint8)
y = np.concatenate([x[20:200], rng.integers(1, 5, 150)]).astype(np.uint8)
for w, h, r in ((40, 1, 1), (50, 2, 2), (64, 1, 2), (20, 3, 1)):
    c = ap.PlotConfig(window_w=w, step_h=h, blowup_r=r, mode=ap.Mode.cuda)
    g = ap.plot_dense_u16(x, y, c)
    t = int(np.quantile(g, 0.9))
    rr, cc, hh = ap.plot_threshold_arrays(x, y, c, t)
    assert rr.size == int((g >= t).sum())
xb = rng.integers(1, 61, 300).astype(np.uint8)   # large alphabet -> computed-mask kernel
yb = rng.integers(1, 61, 400).astype(np.uint8)
ap.plot_dense_u16(xb, yb, ap.PlotConfig(window_w=121, step_h=5, blowup_r=2, mode=ap.Mode.cuda))
print("sanitize case ok")
# repeated calls: the speculative alphabet plan + fused code-stream kernel, and a plan re-run
for s in (4, 4, 20, 4):
    xs = rng.integers(1, s + 1, 500).astype(np.uint8)
    ys = rng.integers(1, s + 1, 600).astype(np.uint8)
    ap.plot_dense_u16(xs, ys, ap.PlotConfig(window_w=48, step_h=1, blowup_r=2, mode=ap.Mode.cuda))
    ap.plot_dense_u8(xs, ys, ap.PlotConfig(window_w=48, step_h=1, blowup_r=1, mode=ap.Mode.cuda))
# fp16-key kernels across several rebases, and a streamed host plot of several row blocks
xl = rng.integers(1, 5, 2600).astype(np.uint8)
yl = rng.integers(1, 5, 3000).astype(np.uint8)
ap.plot_dense_u16(xl, yl, ap.PlotConfig(window_w=100, step_h=1, blowup_r=2, mode=ap.Mode.cuda))
ap.plot_dense_u16(xl, yl, ap.PlotConfig(window_w=128, step_h=1, blowup_r=1, mode=ap.Mode.cuda))
print("sanitize case (extended) ok")
# the large-window path (w*r > 1024): band comb across 3 warps + prefix-sum extraction
xw = rng.integers(1, 5, 1300).astype(np.uint8)
yw = np.concatenate([xw[50:1250], rng.integers(1, 5, 300)]).astype(np.uint8)
cw = ap.PlotConfig(window_w=1100, step_h=7, blowup_r=1, mode=ap.Mode.cuda)
gw = ap.plot_dense_u16(xw, yw, cw)
tw = int(np.quantile(gw, 0.9))
assert ap.plot_threshold_arrays(xw, yw, cw, tw)[0].size == int((gw >= tw).sum())
ap.plot_dense_u16(xw, yw, ap.PlotConfig(window_w=550, step_h=9, blowup_r=2, mode=ap.Mode.cuda))
print("sanitize case (large window) ok")
