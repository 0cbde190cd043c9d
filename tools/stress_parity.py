#!/usr/bin/env python3
"""Randomised parity stress (one-off, not part of the suite): many random plots through the
host API -- dense uint16 and thresholded lists -- against the CPU oracle, with shapes that reach
the tail-split, multi-segment, fp16-key and computed-mask paths.

  python tools/stress_parity.py [--n 400] [--seed 1]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle_lib as ol  # noqa: E402
from paper_0909_2000_b200 import alignplot as ap  # noqa: E402


def main():
    a = argparse.ArgumentParser()
    a.add_argument("--n", type=int, default=400)
    a.add_argument("--seed", type=int, default=1)
    a.add_argument("--big", action="store_true", help="large windows (W up to 1024) and long y, few rows")
    a.add_argument("--wide", action="store_true", help="blown windows 1025..8000 (the large-window path), few rows")
    a.add_argument("--dual", action="store_true",
                   help="LCS plots with h = 1 and the dual-pair kernel's windows (AP_DUAL=1 lifts its size gate)")
    args = a.parse_args()
    if args.dual:
        os.environ["AP_DUAL"] = "1"
    rng = np.random.default_rng(args.seed)
    t0 = time.time()
    cells = 0
    for it in range(args.n):
        r = 1 + int(rng.integers(0, 2))
        if args.dual:
            r, h = 1, 1
            w = int(rng.choice([32, 64, 64, 80, 96, 100, 100, 120, 128, 128, 160, 192, 200, 240, 256, 256, 300, 320, 384, 512,
                               768, 1024]))
            sigma = int(rng.choice([2, 4, 4, 20, 60]))
            m = int(rng.integers(w, w + 300))
            n = int(rng.integers(w, w + (40000 if it % 8 == 0 else 3000)))
        elif args.wide:
            w = int(rng.integers(1025, 8001)) // r
            h = int(rng.choice([1, 1, 3]))
            sigma = int(rng.choice([2, 4, 4, 20]))
            m = int(rng.integers(w, w + 12))
            n = int(rng.integers(w, w + 5000))
        elif args.big:
            w = int(rng.integers(300, 1025 if r == 1 else 513))
            h = int(rng.choice([1, 1, 2]))
            sigma = int(rng.choice([4, 4, 20]))
            m = int(rng.integers(w, w + 24))
            n = int(rng.integers(w, w + 40000))
        else:
            w = int(rng.integers(1, 300 if r == 1 else 150))
            h = int(rng.choice([1, 1, 1, 2, 3, 5, 7]))
            sigma = int(rng.choice([2, 4, 4, 20, 60, 200]))
            m = int(rng.integers(w, w + 600))
            n = int(rng.integers(w, w + 3000))
        x = rng.integers(1, sigma + 1, m).astype(np.uint8)
        if rng.random() < 0.5:   # planted homology
            y = np.concatenate([rng.integers(1, sigma + 1, n // 3), x[: min(m, n // 2)],
                                rng.integers(1, sigma + 1, n // 3)]).astype(np.uint8)
        else:
            y = rng.integers(1, sigma + 1, n).astype(np.uint8)
        if y.size < w:
            continue
        rc, want = ol.plot_rows(x, y, w, h, r)
        assert rc == 0
        c = ap.PlotConfig(window_w=w, step_h=h, blowup_r=r, mode=ap.Mode.cuda)
        got = ap.plot_dense_i32(x, y, c)
        assert np.array_equal(got, want), ("dense", it, w, h, r, m, y.size, sigma)
        t = int(np.quantile(want, 0.9))
        rr, cc, hh = ap.plot_threshold_arrays(x, y, c, t)
        er, ec = np.nonzero(want >= t)
        assert np.array_equal(rr, er) and np.array_equal(cc, ec) and np.array_equal(hh, want[er, ec]), \
            ("threshold", it, w, h, r, m, y.size, sigma)
        cells += want.size
    print(f"stress parity ok: {args.n} random plots, {cells} grid entries, {time.time() - t0:.1f} s")


if __name__ == "__main__":
    main()
