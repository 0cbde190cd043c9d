"""GPU parity: the CUDA engine (through the C ABI) vs the oracle and the reference's golden outputs.

Bit-exact comparison (integer work).  Full grids at sizes the oracle finishes
in seconds; sampled rows (row_begin/row_end) at the BASELINE configs' full
sizes; thresholded lists compared element by element with apply_threshold.
"""
import numpy as np
import pytest

import golden_util as gu
import oracle_lib as ol
from paper_0909_2000_b200 import alignplot as ap
from paper_0909_2000_b200 import datagen

pytestmark = pytest.mark.gpu


def cfg(w, h, r, t=None, n_devices=1):
    return ap.PlotConfig(window_w=w, step_h=h, blowup_r=r, threshold_half=t, mode=ap.Mode.cuda,
                         n_devices=n_devices)


def gpu_grid(x, y, w, h, r, row_begin=0, row_end=0):
    return ap.plot_dense_u16(x, y, cfg(w, h, r), row_begin, row_end).astype(np.int32)


@pytest.mark.parametrize("name", ["runner_engines.json", "runner_modes.json"])
def test_reference_grids(name):
    for case in gu.load(name)["cases"]:
        g = gpu_grid(gu.unhex(case["x"]), gu.unhex(case["y"]), case["w"], case["h"], case["r"])
        assert g.shape == (case["rows"], case["cols"])
        assert np.array_equal(g.reshape(-1), np.array(case["grid"], dtype=np.int32))


def test_reference_acceptance1_540_instances():
    bad = []
    for i, case in enumerate(gu.load("acceptance1.json")["cases"]):
        g = gpu_grid(gu.unhex(case["x"]), gu.unhex(case["y"]), case["w"], case["h"], case["r"])
        if gu.grid_hash(g) != int(case["hash"]):
            bad.append((i, case["w"], case["h"], case["r"]))
    assert not bad, bad[:10]


def test_reference_acceptance7():
    (case,) = gu.load("acceptance7.json")["cases"]
    g = gpu_grid(gu.unhex(case["x"]), gu.unhex(case["y"]), case["w"], case["h"], case["r"])
    assert gu.grid_hash(g) == int(case["hash"])


def test_compute_plot_matches_oracle_random_shapes():
    rng = np.random.default_rng(2024)
    for it in range(60):
        w = int(rng.integers(1, 130))
        r = 1 + it % 2
        m, n = int(rng.integers(w, w + 400)), int(rng.integers(w, w + 700))
        sigma = [2, 4, 20, 60][it % 4]
        x = rng.integers(1, sigma + 1, m).astype(np.uint8)
        y = rng.integers(1, sigma + 1, n).astype(np.uint8)
        h = int(rng.integers(1, 6))
        rc, want = ol.plot_rows(x, y, w, h, r)
        assert rc == 0
        got = gpu_grid(x, y, w, h, r)
        assert np.array_equal(got, want), (it, w, h, r, m, n, sigma)


def test_config_c1_full_grid():
    c = datagen.CONFIGS["C1"]
    x, y = datagen.make_inputs("C1")
    rc, want = ol.plot_rows(x, y, c.w, c.h, c.r)
    got = gpu_grid(x, y, c.w, c.h, c.r)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("name,rows", [("C2", [0, 1, 2, 3, 4097, 8000, 16284]),
                                       ("C3", [0, 1, 31337, 65407, 65408]),
                                       ("C4", [0, 5, 131071, 262080]),
                                       ("C5", [0, 524287, 1048320])])
def test_configs_sampled_rows(name, rows):
    c = datagen.CONFIGS[name]
    x, y = datagen.make_inputs(name)
    for rb in rows:
        re = rb + 2 if name in ("C2", "C3") else rb + 1
        rc, want = ol.plot_rows(x, y, c.w, c.h, c.r, rb, re)
        assert rc == 0
        got = gpu_grid(x, y, c.w, c.h, c.r, rb, re)
        assert np.array_equal(got, want), (name, rb)


def test_threshold_matches_apply_threshold():
    rng = np.random.default_rng(77)
    for it in range(20):
        w = int(rng.integers(4, 80))
        r = 1 + it % 2
        m, n = int(rng.integers(w, 600)), int(rng.integers(w, 900))
        x = rng.integers(1, 5, m).astype(np.uint8)
        y = x[rng.integers(0, m, n)] if it % 3 == 0 else rng.integers(1, 5, n).astype(np.uint8)
        h = 1 + it % 3
        rc, grid = ol.plot_rows(x, y, w, h, r)
        t = int(np.quantile(grid, 0.97))
        rr, cc = np.nonzero(grid >= t)
        gr, gc, gh = ap.plot_threshold_arrays(x, y, cfg(w, h, r), t)
        assert np.array_equal(gr, rr) and np.array_equal(gc, cc)
        assert np.array_equal(gh, grid[rr, cc])


def test_threshold_planted_homology():
    # x and y share long blocks, so thresholded hits are dense along diagonals
    rng = np.random.default_rng(5)
    x = rng.integers(1, 5, 3000).astype(np.uint8)
    y = np.concatenate([rng.integers(1, 5, 400), x[500:1500], rng.integers(1, 5, 300), x[2000:2600]]).astype(np.uint8)
    w, h, r = 64, 1, 1
    rc, grid = ol.plot_rows(x, y, w, h, r)
    t = 2 * 60
    rr, cc = np.nonzero(grid >= t)
    assert rr.size > 1000
    gr, gc, gh = ap.plot_threshold_arrays(x, y, cfg(w, h, r), t)
    assert np.array_equal(gr, rr) and np.array_equal(gc, cc) and np.array_equal(gh, grid[rr, cc])


def test_errors_before_device_work():
    with pytest.raises(ap.EmptyPlotError):
        ap.compute_plot(ap.Sequence("x", [1, 2, 1]), ap.Sequence("y", [2, 1, 2]), cfg(10, 1, 1))
    with pytest.raises(ap.ConfigError):
        ap.compute_plot(ap.Sequence("x", [1, 2, 1]), ap.Sequence("y", [2, 1, 2]), cfg(2, 1, 7))
    with pytest.raises(ap.ConfigError):
        ap.plot_dense_u16(np.array([1, 0, 2], np.uint8), np.array([1, 2, 2], np.uint8), cfg(2, 1, 1))


def test_window_equals_input():
    x = np.array([1, 2, 3, 1, 2], np.uint8)
    g = gpu_grid(x, x, 5, 1, 1)
    assert g.shape == (1, 1) and g[0, 0] == 10
    g = gpu_grid(x, x, 5, 1, 2)
    assert g[0, 0] == 10


def test_cpp_shim_reference_cases():
    """The reference's own test cases, written against the C++ drop-in header, run on the GPU."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "tests", "cpp", "test_shim")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", root, "tests/cpp/test_shim"], check=True)
    res = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr


def test_pgm_fused_matches_host_quantisation():
    from paper_0909_2000_b200 import writers as wr
    rng = np.random.default_rng(31)
    for w, h, r, t in ((30, 1, 1, None), (25, 2, 2, 20), (64, 1, 1, 100)):
        x = rng.integers(1, 5, 400).astype(np.uint8)
        y = np.concatenate([x[100:300], rng.integers(1, 5, 200)]).astype(np.uint8)
        c = cfg(w, h, r, t)
        rc, want = ol.plot_rows(x, y, w, h, r)
        g = ap.PlotGrid(want.shape[0], want.shape[1], w, h, values=want.reshape(-1))
        assert wr.plot_pgm(x, y, c) == wr.pgm_header(*want.shape) + wr.pgm_pixels(g, t).tobytes()


def test_cli_matches_reference_cli_bytes():
    """The CLI (python -m paper_0909_2000_b200) reproduces the reference CLI's output bytes
    (tests/golden/cli, made by the reference library through oracle/ref_cli.cpp)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    gdir = os.path.join(root, "tests", "golden", "cli")
    index = json.load(open(os.path.join(gdir, "index.json")))
    for case in index["cases"]:
        args = [sys.executable, "-m", "paper_0909_2000_b200", "--x", os.path.join(gdir, "x.fa"), "--y",
                os.path.join(gdir, "y.fa"), "--window", str(case["window"]), "--step", str(case["step"]),
                "--format", case["format"]]
        if case["lcs_only"]:
            args.append("--lcs-only")
        if case["dense"]:
            args.append("--dense")
        if case["threshold"] is not None:
            args += ["--threshold", str(case["threshold"])]
        out = subprocess.run(args, capture_output=True, cwd=root, timeout=300)
        assert out.returncode == 0, out.stderr.decode()
        want = open(os.path.join(gdir, case["file"]), "rb").read()
        assert out.stdout == want, case["name"]


GENERIC_SHAPES = ["4,32,2", "4,32,4", "8,8,2", "8,16,2", "8,16,4", "8,24,2", "8,32,2", "8,32,4", "16,8,2",
                  "16,16,2", "16,16,4", "16,24,2", "16,32,2", "16,32,4", "32,8,2", "32,16,2", "32,16,4",
                  "32,24,2", "32,32,2", "32,32,4"]


@pytest.mark.parametrize("shape", [s + ",0,0" for s in GENERIC_SHAPES] + [s + ",0,1" for s in GENERIC_SHAPES] +
                         ["4,32,2,1", "8,16,4,1", "16,16,4,1", "32,8,2,1"])
def test_forced_generic_shapes(shape, monkeypatch):
    """Every instantiated generic (L, R, K) shape, forced with AP_SHAPE, is bit-exact:
    table masks with integer keys (",0,0") and with fp16 keys (",0,1"), and the
    computed-mask variant (",1", exercised with a 60-letter alphabet)."""
    monkeypatch.setenv("AP_SHAPE", shape)
    monkeypatch.setenv("AP_NO_R2", "1")
    rng = np.random.default_rng(sum(map(ord, shape)))
    L, R, K = map(int, shape.split(",")[:3])
    sigma = 60 if shape.count(",") == 3 else 4
    for r in (1, 2):
        w = max(2, min((L * R) // r - 3, 200))
        x = rng.integers(1, sigma + 1, w + 150).astype(np.uint8)
        y = rng.integers(1, sigma + 1, w + 700).astype(np.uint8)
        rc, want = ol.plot_rows(x, y, w, 2, r)
        assert np.array_equal(gpu_grid(x, y, w, 2, r), want), (shape, r)


DUAL_SHAPES = ["4,32,1", "4,32,2", "8,32,1", "8,32,2", "8,16,1", "8,16,2", "16,16,1", "16,16,2", "8,8,1", "8,8,2",
               "4,16,2", "4,8,2", "4,24,2", "8,24,2", "16,24,2", "32,24,2", "16,32,2", "32,32,2",
               # lane groups that do not tile the warp (idle phantom group)
               "5,20,1", "10,20,1", "5,16,2", "5,24,2", "5,32,2", "10,32,2", "15,20,1", "10,24,2"]


def _dual_hf_ok(s):   # fp16 keys need W + L*K <= 768 (kHfMaxSpan)
    L, R, K = map(int, s.split(","))
    return L * R + L * K <= 768


def last_kernel_name(x, y, w, h, r):
    """Name of the comb kernel a dense device-API plot of (x, y) launches (ap_ctx_last_kernel)."""
    import ctypes

    import torch

    from paper_0909_2000_b200 import _native
    L = _native.lib()
    ctx = ctypes.c_void_p()
    assert L.ap_ctx_create(0, ctypes.byref(ctx)) == 0
    c = _native.ApConfig(window_w=w, step_h=h, blowup_r=r, has_threshold=0, threshold_half=0, n_devices=1,
                         row_begin=0, row_end=0)
    dx, dy = torch.from_numpy(x.copy()).cuda(), torch.from_numpy(y.copy()).cuda()
    rows, cols = (x.size - w) // h + 1, y.size - w + 1
    out = torch.empty(rows * cols, dtype=torch.int16, device="cuda")
    rc = L.ap_ctx_plot_dense_device(ctx, dx.data_ptr(), x.size, dy.data_ptr(), y.size, ctypes.byref(c),
                                    out.data_ptr(), None)
    assert rc == 0, _native.last_error()
    name = (L.ap_ctx_last_kernel(ctx) or b"").decode()
    L.ap_ctx_destroy(ctx)
    return name, out.cpu().numpy().astype(np.uint16).astype(np.int32).reshape(rows, cols)


@pytest.mark.parametrize("shape", [s + ",0,0,1" for s in DUAL_SHAPES] + [s + ",0,1,1" for s in DUAL_SHAPES if _dual_hf_ok(s)])
def test_forced_dual_shapes(shape, monkeypatch):
    """Every instantiated dual-pair shape (two strip pairs per lane group sharing one mask table,
    ap_dual_kernels.cuh), integer and fp16 keys, dense and thresholded, for row counts of every
    residue mod 4 (a group holds grid rows 4g .. 4g+3)."""
    monkeypatch.setenv("AP_SHAPE", shape)
    monkeypatch.setenv("AP_DUAL", "1")
    L, R, K = map(int, shape.split(",")[:3])
    w = L * R
    rng = np.random.default_rng(sum(map(ord, shape)))
    for extra in range(4):
        x = rng.integers(1, 5, w + 70 + extra).astype(np.uint8)
        y = np.concatenate([rng.integers(1, 5, 300), x[5:w + 40], rng.integers(1, 5, 400)]).astype(np.uint8)
        if extra == 0:
            name, grid = last_kernel_name(x, y, w, 1, 1)
            assert name.startswith("combd<%d,%d,%d," % (L, R, K)), name
        rc, want = ol.plot_rows(x, y, w, 1, 1)
        assert rc == 0
        assert np.array_equal(gpu_grid(x, y, w, 1, 1), want), (shape, extra)
        t = int(np.quantile(want, 0.97))
        rr, cc = np.nonzero(want >= t)
        gr, gc, gh = ap.plot_threshold_arrays(x, y, cfg(w, 1, 1), t)
        assert np.array_equal(gr, rr) and np.array_equal(gc, cc) and np.array_equal(gh, want[rr, cc]), (shape, extra)


@pytest.mark.parametrize("w,sigma", [(64, 4), (128, 4), (256, 4), (128, 20), (256, 2), (100, 4), (200, 4), (100, 20),
                                     (320, 4)])
def test_dual_kernel_long_y_and_row_ranges(w, sigma, monkeypatch):
    """The dual-pair kernel as the default plan picks it (AP_DUAL=1 lifts the problem-size gate):
    a y long enough for interior chunks and fp16-key rebases with planted homology, odd row
    ranges, bytes of x absent from y, dense and thresholded."""
    monkeypatch.setenv("AP_DUAL", "1")
    rng = np.random.default_rng(w + sigma)
    x = rng.integers(1, sigma + 1, w + 22).astype(np.uint8)
    x[w // 2] = 200   # absent from y
    parts = []
    while sum(p.size for p in parts) < 40000:
        parts.append(rng.integers(1, sigma + 1, int(rng.integers(50, 2500))).astype(np.uint8))
        blk = x[int(rng.integers(0, 20)):][:w + 10].copy()
        blk[blk == 200] = 1
        flip = rng.random(blk.size) < 0.06
        blk[flip] = rng.integers(1, sigma + 1, int(flip.sum()))
        parts.append(blk)
    y = np.concatenate(parts)
    name, grid = last_kernel_name(x, y, w, 1, 1)
    assert name.startswith("combd<"), name
    rc, want = ol.plot_rows(x, y, w, 1, 1)
    assert rc == 0 and np.array_equal(grid, want)
    assert np.array_equal(gpu_grid(x, y, w, 1, 1), want)
    for rb, re in ((1, 2), (3, 10), (5, 23), (22, 23)):
        assert np.array_equal(gpu_grid(x, y, w, 1, 1, rb, re), want[rb:re]), (rb, re)
    for t in (int(np.quantile(want, 0.999)), int(want.max())):
        rr, cc = np.nonzero(want >= t)
        gr, gc, gh = ap.plot_threshold_arrays(x, y, cfg(w, 1, 1), t)
        assert np.array_equal(gr, rr) and np.array_equal(gc, cc) and np.array_equal(gh, want[rr, cc]), t


def test_dual_kernel_output_kinds(monkeypatch):
    """uint8 / int32 half-units and the fused PGM raster (with and without a threshold) through
    the dual-pair kernel equal the uint16 plot and the host-side quantisation."""
    from paper_0909_2000_b200 import writers as wr
    monkeypatch.setenv("AP_DUAL", "1")
    rng = np.random.default_rng(64)
    x = rng.integers(1, 5, 700).astype(np.uint8)
    y = np.concatenate([x[100:400], rng.integers(1, 5, 500)]).astype(np.uint8)
    name, _ = last_kernel_name(x, y, 64, 1, 1)
    assert name.startswith("combd<"), name
    rc, want = ol.plot_rows(x, y, 64, 1, 1)
    c = cfg(64, 1, 1)
    assert np.array_equal(ap.plot_dense_u8(x, y, c).astype(np.int32), want)
    assert np.array_equal(ap.plot_dense_i32(x, y, c), want)
    assert np.array_equal(ap.plot_dense_i32(x, y, c, 5, 42), want[5:42])
    g = ap.PlotGrid(want.shape[0], want.shape[1], 64, 1, values=want.reshape(-1))
    for t in (None, 90):
        assert wr.plot_pgm(x, y, cfg(64, 1, 1, t)) == wr.pgm_header(*want.shape) + wr.pgm_pixels(g, t).tobytes()


@pytest.mark.parametrize("ndev", [2, 3])
def test_dual_kernel_row_shards(ndev, monkeypatch):
    """Row shards (one GPU standing in for ndev devices) through the dual-pair kernel: shard
    boundaries cut groups of four rows anywhere, each shard uploads its own x halo."""
    monkeypatch.setenv("AP_DUAL", "1")
    monkeypatch.setenv("AP_SHARDS_PER_DEVICE", str(ndev))
    rng = np.random.default_rng(70 + ndev)
    x = rng.integers(1, 5, 64 + 201).astype(np.uint8)
    y = np.concatenate([x[30:230], rng.integers(1, 5, 400)]).astype(np.uint8)
    rc, want = ol.plot_rows(x, y, 64, 1, 1)
    many = ap.plot_dense_u16(x, y, cfg(64, 1, 1, n_devices=ndev)).astype(np.int32)
    assert np.array_equal(many, want)
    t = int(np.quantile(want, 0.97))
    rr, cc = np.nonzero(want >= t)
    gr, gc, gh = ap.plot_threshold_arrays(x, y, cfg(64, 1, 1, n_devices=ndev), t)
    assert np.array_equal(gr, rr) and np.array_equal(gc, cc) and np.array_equal(gh, want[rr, cc])


@pytest.mark.parametrize("w", [64, 100])
def test_dual_kernel_tiny_plots(w, monkeypatch):
    """Edge sizes through the dual-pair kernel: 1-5 grid rows (groups with missing strips and a
    missing second pair), a single-column and a two-column y."""
    monkeypatch.setenv("AP_DUAL", "1")
    rng = np.random.default_rng(w)
    for rows in (1, 2, 3, 4, 5):
        for ncols in (1, 2, 37):
            x = rng.integers(1, 5, w + rows - 1).astype(np.uint8)
            y = np.concatenate([x[:w // 2], rng.integers(1, 5, w - w // 2 + ncols - 1)]).astype(np.uint8)
            rc, want = ol.plot_rows(x, y, w, 1, 1)
            assert rc == 0 and want.shape == (rows, ncols)
            assert np.array_equal(gpu_grid(x, y, w, 1, 1), want), (rows, ncols)
            t = int(want.max())
            rr, cc = np.nonzero(want >= t)
            gr, gc, gh = ap.plot_threshold_arrays(x, y, cfg(w, 1, 1), t)
            assert np.array_equal(gr, rr) and np.array_equal(gc, cc) and np.array_equal(gh, want[rr, cc])
    name, _ = last_kernel_name(x, y, w, 1, 1)
    assert name.startswith("combd<"), name


def test_dual_kernel_gate_and_streamed_blocks(monkeypatch):
    """Small plots keep the single-pair kernel (too few pair groups to fill the GPU), large ones
    take the dual-pair kernel; the streamed host plot (row blocks whose mask words reach into
    the next block's x characters) equals the one-launch device plot and the oracle."""
    rng = np.random.default_rng(99)
    x = rng.integers(1, 5, 2600).astype(np.uint8)
    y = np.concatenate([x[300:1200], rng.integers(1, 5, 1500)]).astype(np.uint8)
    name, _ = last_kernel_name(x[:400], y[:600], 64, 1, 1)
    assert name.startswith("comb<"), name
    monkeypatch.setenv("AP_DUAL", "1")
    name, grid = last_kernel_name(x, y, 64, 1, 1)
    assert name.startswith("combd<"), name
    rc, want = ol.plot_rows(x, y, 64, 1, 1)
    assert rc == 0 and np.array_equal(grid, want)
    assert np.array_equal(gpu_grid(x, y, 64, 1, 1), want)
    # a 120-letter alphabet's table (> 90 KB per warp) keeps the single-pair kernel
    x60 = rng.integers(1, 121, 500).astype(np.uint8)
    y60 = np.concatenate([x60[100:300], rng.integers(1, 121, 300)]).astype(np.uint8)
    name, grid = last_kernel_name(x60, y60, 64, 1, 1)
    assert name.startswith("comb<"), name
    rc, want = ol.plot_rows(x60, y60, 64, 1, 1)
    assert rc == 0 and np.array_equal(grid, want)
    monkeypatch.delenv("AP_DUAL")
    big_x = rng.integers(1, 5, 70000).astype(np.uint8)
    big_y = rng.integers(1, 5, 9000).astype(np.uint8)
    name, grid = last_kernel_name(big_x, big_y, 64, 1, 1)
    assert name.startswith("combd<"), name
    for rb in (0, 33333, 69935):
        rc, wr = ol.plot_rows(big_x, big_y, 64, 1, 1, rb, rb + 2)
        assert np.array_equal(grid[rb:rb + 2], wr), rb


@pytest.mark.parametrize("shape", ["8,4,1", "8,4,2", "16,4,1", "16,4,2", "32,4,1", "32,4,2"])
def test_forced_r2_dual_shapes(shape, monkeypatch):
    """The r = 2 dual-pair kernel (comb2d_kernel: two strip pairs per lane group, one linear mask
    table per warp), w = 4 L, every row-count residue mod 4, dense and thresholded, a 20-letter
    and a 4-letter alphabet."""
    monkeypatch.setenv("AP_SHAPE2", shape + ",0,1")
    monkeypatch.setenv("AP_DUAL", "1")
    L, RR, K = map(int, shape.split(","))
    w = 4 * L
    rng = np.random.default_rng(L * 10 + K)
    for extra in range(4):
        sigma = 20 if extra % 2 else 4
        x = rng.integers(1, sigma + 1, w + 90 + extra).astype(np.uint8)
        y = np.concatenate([rng.integers(1, sigma + 1, 200), x[5:w + 60], rng.integers(1, sigma + 1, 300)]).astype(np.uint8)
        if extra == 0:
            name, grid = last_kernel_name(x, y, w, 1, 2)
            assert name.startswith("comb2d<%d,4,%d," % (L, K)), name
        rc, want = ol.plot_rows(x, y, w, 1, 2)
        assert rc == 0
        assert np.array_equal(gpu_grid(x, y, w, 1, 2), want), (shape, extra)
        t = int(np.quantile(want, 0.97))
        rr, cc = np.nonzero(want >= t)
        gr, gc, gh = ap.plot_threshold_arrays(x, y, cfg(w, 1, 2), t)
        assert np.array_equal(gr, rr) and np.array_equal(gc, cc) and np.array_equal(gh, want[rr, cc]), (shape, extra)


@pytest.mark.parametrize("w,sigma", [(64, 20), (32, 4), (128, 4)])
def test_r2_dual_kernel_long_y_and_row_ranges(w, sigma, monkeypatch):
    """comb2d_kernel (opt-in: AP_SHAPE2=L,4,K,0,1) on a y long enough for interior chunks and a
    key rebase (> 28K blown columns) with planted homology, odd row ranges, a byte of x absent
    from y, dense and thresholded."""
    monkeypatch.setenv("AP_DUAL", "1")
    monkeypatch.setenv("AP_SHAPE2", "%d,4,2,0,1" % (w // 4))
    rng = np.random.default_rng(w + sigma + 1)
    x = rng.integers(1, sigma + 1, w + 22).astype(np.uint8)
    x[w // 2] = 200
    parts = []
    while sum(p.size for p in parts) < 20000:
        parts.append(rng.integers(1, sigma + 1, int(rng.integers(50, 2500))).astype(np.uint8))
        blk = x[int(rng.integers(0, 20)):][:w + 10].copy()
        blk[blk == 200] = 1
        flip = rng.random(blk.size) < 0.06
        blk[flip] = rng.integers(1, sigma + 1, int(flip.sum()))
        parts.append(blk)
    y = np.concatenate(parts)
    name, grid = last_kernel_name(x, y, w, 1, 2)
    assert name.startswith("comb2d<"), name
    rc, want = ol.plot_rows(x, y, w, 1, 2)
    assert rc == 0 and np.array_equal(grid, want)
    assert np.array_equal(gpu_grid(x, y, w, 1, 2), want)
    for rb, re in ((1, 2), (3, 10), (5, 23), (22, 23)):
        assert np.array_equal(gpu_grid(x, y, w, 1, 2, rb, re), want[rb:re]), (rb, re)
    for t in (int(np.quantile(want, 0.999)), int(want.max())):
        rr, cc = np.nonzero(want >= t)
        gr, gc, gh = ap.plot_threshold_arrays(x, y, cfg(w, 1, 2), t)
        assert np.array_equal(gr, rr) and np.array_equal(gc, cc) and np.array_equal(gh, want[rr, cc]), t


R2_SHAPES = ["4,25,5", "4,25,1", "10,10,2", "10,10,1", "5,20,4", "5,20,1", "8,8,2", "8,8,4", "16,8,4",
             "32,8,4", "8,16,4", "16,16,4", "32,16,4", "16,4,2", "32,4,2", "16,10,2", "8,20,4", "32,5,1",
             "32,4,1", "16,4,1"]


@pytest.mark.parametrize("shape", [s + ",0" for s in R2_SHAPES] +
                         [s + ",1" for s in R2_SHAPES if int(s.split(",")[1]) >= 8])
def test_forced_r2_shapes(shape, monkeypatch):
    """Every instantiated r = 2 (L, RR, K) shape, forced with AP_SHAPE2, is bit-exact (dense and
    threshold), with integer keys (,0) and -- for the RR >= 8 shapes -- fp16 keys (,1; rebased
    every few hundred columns, so these short strips already cross several rebases)."""
    monkeypatch.setenv("AP_SHAPE2", shape)
    L, RR, K, _ = map(int, shape.split(","))
    w = RR * min(L, max(1, 100 // RR))
    rng = np.random.default_rng(RR * 131 + L)
    x = rng.integers(1, 5, w + 120).astype(np.uint8)
    y = np.concatenate([x[10:w + 60], rng.integers(1, 5, 600)]).astype(np.uint8)
    rc, want = ol.plot_rows(x, y, w, 1, 2)
    assert np.array_equal(gpu_grid(x, y, w, 1, 2), want), shape
    t = int(np.quantile(want, 0.95))
    rr, cc = np.nonzero(want >= t)
    gr, gc, gh = ap.plot_threshold_arrays(x, y, cfg(w, 1, 2), t)
    assert np.array_equal(gr, rr) and np.array_equal(gc, cc) and np.array_equal(gh, want[rr, cc]), shape


@pytest.mark.parametrize("shape,w", [("32,16,4,1", 288), ("16,10,2,1", 160), ("10,10,2,1", 100)])
def test_forced_r2_fp16_keys_long(shape, w, monkeypatch):
    """fp16-key r = 2 kernel at the largest span it accepts (w = 288: W + 2*VB = 720, rebased
    every 176 blown columns) and at C2's shape, over a long y with planted homology."""
    monkeypatch.setenv("AP_SHAPE2", shape)
    rng = np.random.default_rng(w)
    x = rng.integers(1, 5, w + 90).astype(np.uint8)
    y = np.concatenate([rng.integers(1, 5, 1500), x[20:w + 60], rng.integers(1, 5, 2500)]).astype(np.uint8)
    rc, want = ol.plot_rows(x, y, w, 1, 2)
    assert np.array_equal(gpu_grid(x, y, w, 1, 2), want), shape
    t = int(want.max()) - 6
    rr, cc = np.nonzero(want >= t)
    gr, gc, gh = ap.plot_threshold_arrays(x, y, cfg(w, 1, 2), t)
    assert np.array_equal(gr, rr) and np.array_equal(gc, cc) and np.array_equal(gh, want[rr, cc]), shape


@pytest.mark.parametrize("shape,w,r", [("32,32,2,0,1", 640, 1), ("16,16,4,0,1", 256, 1), ("8,32,2,0,1", 120, 2)])
def test_forced_generic_fp16_keys_long(shape, w, r, monkeypatch):
    """fp16-key generic kernel at the largest span it accepts (w = 640: W + L*K = 704, rebased
    every 192 columns), at C5's shape and in r = 2 mode, over a long y with planted homology."""
    monkeypatch.setenv("AP_SHAPE", shape)
    monkeypatch.setenv("AP_NO_R2", "1")
    rng = np.random.default_rng(w + r)
    x = rng.integers(1, 5, w + 70).astype(np.uint8)
    y = np.concatenate([rng.integers(1, 5, 1200), x[30:w + 50], rng.integers(1, 5, 2200)]).astype(np.uint8)
    rc, want = ol.plot_rows(x, y, w, 1, r)
    assert np.array_equal(gpu_grid(x, y, w, 1, r), want), shape
    t = int(want.max()) - 6
    rr, cc = np.nonzero(want >= t)
    gr, gc, gh = ap.plot_threshold_arrays(x, y, cfg(w, 1, r), t)
    assert np.array_equal(gr, rr) and np.array_equal(gc, cc) and np.array_equal(gh, want[rr, cc]), shape


def test_dense_u8_and_i32_match_u16():
    rng = np.random.default_rng(8)
    x = rng.integers(1, 5, 600).astype(np.uint8)
    y = np.concatenate([x[50:350], rng.integers(1, 5, 400)]).astype(np.uint8)
    for w, h, r in ((100, 1, 2), (127, 2, 1), (30, 3, 2)):
        c = cfg(w, h, r)
        assert np.array_equal(ap.plot_dense_u8(x, y, c).astype(np.int32), gpu_grid(x, y, w, h, r))
        assert np.array_equal(ap.plot_dense_i32(x, y, c), gpu_grid(x, y, w, h, r))
        assert np.array_equal(ap.plot_dense_i32(x, y, c, 3, 9), gpu_grid(x, y, w, h, r)[3:9])
    with pytest.raises(ap.ConfigError):
        ap.plot_dense_u8(x, y, cfg(128, 1, 1))


@pytest.mark.parametrize("ndev", [2, 3, 4])
def test_multi_device_row_shards(ndev, monkeypatch):
    """The in-library multi-device path (contiguous row shards, x halo per shard,
    count gather and in-order concatenation), with one GPU standing in for ndev
    shard devices (AP_SHARDS_PER_DEVICE), equals the single-device result."""
    monkeypatch.setenv("AP_SHARDS_PER_DEVICE", str(ndev))
    rng = np.random.default_rng(40 + ndev)
    x = rng.integers(1, 5, 900).astype(np.uint8)
    y = np.concatenate([x[100:500], rng.integers(1, 5, 300)]).astype(np.uint8)
    for w, h, r in ((48, 1, 1), (30, 3, 2)):
        one = ap.plot_dense_u16(x, y, cfg(w, h, r, n_devices=1))
        many = ap.plot_dense_u16(x, y, cfg(w, h, r, n_devices=ndev))
        assert np.array_equal(one, many)
        rc, want = ol.plot_rows(x, y, w, h, r)
        assert np.array_equal(many.astype(np.int32), want)
        t = int(np.quantile(want, 0.97))
        r1 = ap.plot_threshold_arrays(x, y, cfg(w, h, r, n_devices=1), t)
        rn = ap.plot_threshold_arrays(x, y, cfg(w, h, r, n_devices=ndev), t)
        for a, b in zip(r1, rn):
            assert np.array_equal(a, b)
        # a row range split across shards
        part = ap.plot_dense_u16(x, y, cfg(w, h, r, n_devices=ndev), 7, 7 + 2 * ndev + 5)
        assert np.array_equal(part, one[7:7 + 2 * ndev + 5])


@pytest.mark.parametrize("w,r,h,sigma", [(64, 1, 1, 4), (128, 1, 2, 4), (256, 1, 1, 4), (33, 1, 1, 4), (255, 1, 3, 2),
                                         (100, 2, 1, 4), (64, 2, 1, 20), (512, 2, 1, 4), (7, 2, 2, 4)])
def test_long_sequences_dense_and_threshold(w, r, h, sigma):
    """Long y (many interior extraction chunks, several key rebases per strip) with
    planted homology: dense grid and thresholded lists bit-exact, including
    thresholds outside the score range (the kernel clamps t to +-0x4000)."""
    rng = np.random.default_rng(w * 7 + r * 3 + sigma)
    m = w + 5 * h
    x = rng.integers(1, sigma + 1, m).astype(np.uint8)
    parts = []
    while sum(p.size for p in parts) < 70000:
        parts.append(rng.integers(1, sigma + 1, int(rng.integers(50, 3000))).astype(np.uint8))
        blk = x[int(rng.integers(0, max(1, m - w))):][:w + 20].copy()
        flip = rng.random(blk.size) < 0.08
        blk[flip] = rng.integers(1, sigma + 1, int(flip.sum()))
        parts.append(blk)
    y = np.concatenate(parts)
    rc, want = ol.plot_rows(x, y, w, h, r)
    assert rc == 0
    got = gpu_grid(x, y, w, h, r)
    assert np.array_equal(got, want)
    for t in (int(np.quantile(want, 0.999)), int(want.max()), int(want.min()) - 3, 5000, -5000):
        rr, cc = np.nonzero(want >= t)
        gr, gc, gh = ap.plot_threshold_arrays(x, y, cfg(w, h, r), t)
        assert np.array_equal(gr, rr) and np.array_equal(gc, cc), (t, gr.size, rr.size)
        assert np.array_equal(gh, want[rr, cc]), t


@pytest.mark.parametrize("shape", ["4,32,4", "8,16,4", "16,8,2", "32,8,2"])
def test_forced_generic_shapes_long_y(shape, monkeypatch):
    """Forced generic shapes on a y long enough for interior chunks and rebases, both r."""
    monkeypatch.setenv("AP_SHAPE", shape)
    monkeypatch.setenv("AP_NO_R2", "1")
    L, R, K = map(int, shape.split(","))
    rng = np.random.default_rng(L * 100 + R)
    for r in (1, 2):
        w = max(2, min((L * R) // r - 1, 200))
        x = rng.integers(1, 5, w + 9).astype(np.uint8)
        y = np.concatenate([rng.integers(1, 5, 30000), x[:w], rng.integers(1, 5, 3000)]).astype(np.uint8)
        rc, want = ol.plot_rows(x, y, w, 1, r)
        assert np.array_equal(gpu_grid(x, y, w, 1, r), want), (shape, r)
        t = int(np.quantile(want, 0.999))
        rr, cc = np.nonzero(want >= t)
        gr, gc, gh = ap.plot_threshold_arrays(x, y, cfg(w, 1, r), t)
        assert np.array_equal(gr, rr) and np.array_equal(gc, cc) and np.array_equal(gh, want[rr, cc])


def test_threshold_cells_aos_matches_soa():
    """ap_plot_threshold_cells (array of ap_cell) == ap_plot_threshold (parallel arrays),
    including the AP_CAPACITY retry and both score modes."""
    rng = np.random.default_rng(91)
    x = rng.integers(1, 5, 1500).astype(np.uint8)
    y = np.concatenate([rng.integers(1, 5, 300), x[200:900], rng.integers(1, 5, 200)]).astype(np.uint8)
    for w, h, r in ((40, 1, 1), (25, 2, 2)):
        rc, grid = ol.plot_rows(x, y, w, h, r)
        t = int(np.quantile(grid, 0.99))
        cells = ap.plot_threshold_cells(x, y, cfg(w, h, r), t)
        gr, gc, gh = ap.plot_threshold_arrays(x, y, cfg(w, h, r), t)
        assert len(cells) == gr.size > 100
        assert [c.row for c in cells] == gr.tolist() and [c.col for c in cells] == gc.tolist()
        assert [c.score_half for c in cells] == grid[gr, gc].tolist()


def test_host_api_concurrent_threads():
    """The host API is reentrant: concurrent calls from several threads (one shared
    per-device context, serialised inside the library) give the serial results."""
    import threading
    rng = np.random.default_rng(123)
    cases = []
    for k in range(6):
        w = int(rng.integers(8, 90))
        x = rng.integers(1, 5, w + 200).astype(np.uint8)
        y = rng.integers(1, 5, w + 900).astype(np.uint8)
        cases.append((x, y, w, 1 + k % 3, 1 + k % 2))
    want = [gpu_grid(*c) for c in cases]
    got = [None] * len(cases)
    errs = []

    def run(i):
        try:
            for _ in range(3):
                got[i] = gpu_grid(*cases[i])
        except Exception as e:   # surfaced below
            errs.append(e)

    ts = [threading.Thread(target=run, args=(i,)) for i in range(len(cases))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for a, b in zip(got, want):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("name,u8", [("C2", False), ("C2", True)])
def test_streamed_host_plot_equals_device_plot(name, u8):
    """The host API streams the dense plot out in row blocks (D2H-bound uint16: short-task blocks
    of growing size on one stream; compute-bound uint8: equal blocks on two streams); at C2's full
    size (16285 x 16280, ~10 blocks) it must equal the one-launch device-API plot bit for bit,
    and the rows at the block seams must equal the oracle."""
    import ctypes

    import torch

    from paper_0909_2000_b200 import _native

    c = datagen.CONFIGS[name]
    x, y = datagen.make_inputs(name)
    pc = cfg(c.w, c.h, c.r)
    host = (ap.plot_dense_u8(x, y, pc) if u8 else ap.plot_dense_u16(x, y, pc)).reshape(-1)
    L = _native.lib()
    ctx = ctypes.c_void_p()
    assert L.ap_ctx_create(0, ctypes.byref(ctx)) == 0
    try:
        dx, dy = torch.from_numpy(x.copy()).cuda(), torch.from_numpy(y.copy()).cuda()
        dout = torch.empty(host.size, dtype=torch.uint8 if u8 else torch.int16, device="cuda")
        fn = L.ap_ctx_plot_dense_u8_device if u8 else L.ap_ctx_plot_dense_device
        assert fn(ctx, dx.data_ptr(), x.size, dy.data_ptr(), y.size, ctypes.byref(ap._cfg(pc)),
                  dout.data_ptr(), None) == 0
        torch.cuda.synchronize()
        dev = dout.cpu().numpy().view(np.uint8 if u8 else np.uint16)
    finally:
        L.ap_ctx_destroy(ctx)
    assert np.array_equal(host, dev)
    rows, cols = (x.size - c.w) // c.h + 1, y.size - c.w + 1
    grid = host.reshape(rows, cols)
    # around the first block seams (one wave = 74 pair groups of 6 rows with 32 segments) and
    # the old 148-group ones
    for rb in (443, 444, 887, 888, 2663, 2664):
        rc, want = ol.plot_rows(x, y, c.w, c.h, c.r, rb, rb + 1)
        assert rc == 0 and np.array_equal(grid[rb:rb + 1].astype(np.int32), want), rb


def test_speculative_alphabet_plan_reruns_when_y_grows():
    """Repeated calls plan for the previous call's alphabet size without waiting for this y's
    (ap_capi.cu run_device): a call whose y has more codes must be detected on the device and
    re-run; one with fewer codes runs on the larger plan.  Alternate alphabets of 2, 20, 4, 60
    and 3 letters for the same (w, r, output) and check every dense and thresholded result."""
    rng = np.random.default_rng(4242)
    for r in (1, 2):
        for sigma in (2, 20, 4, 60, 3, 60):
            w = 24
            x = rng.integers(1, sigma + 1, 300).astype(np.uint8)
            y = np.concatenate([x[40:140], rng.integers(1, sigma + 1, 250)]).astype(np.uint8)
            rc, want = ol.plot_rows(x, y, w, 1, r)
            assert rc == 0
            assert np.array_equal(gpu_grid(x, y, w, 1, r), want), (r, sigma)
            assert np.array_equal(ap.plot_dense_u8(x, y, cfg(w, 1, r)).astype(np.int32), want), (r, sigma)
            t = int(np.quantile(want, 0.97))
            rr, cc = np.nonzero(want >= t)
            gr, gc, gh = ap.plot_threshold_arrays(x, y, cfg(w, 1, r), t)
            assert np.array_equal(gr, rr) and np.array_equal(gc, cc) and np.array_equal(gh, want[rr, cc]), (r, sigma)


def test_tiny_windows_and_degenerate_alphabets():
    """w = 1..8 in both modes and steps 1..3, a one-letter y, x letters absent from y, and y of
    exactly w characters (one column) -- the smallest shapes of every code path."""
    rng = np.random.default_rng(99)
    cases = []
    for w in range(1, 9):
        for r in (1, 2):
            for h in (1, 3):
                x = rng.integers(1, 5, w + 40).astype(np.uint8)
                y = rng.integers(1, 5, w + 70).astype(np.uint8)
                cases.append((x, y, w, h, r))
    one = np.full(90, 7, np.uint8)
    cases.append((rng.integers(6, 9, 60).astype(np.uint8), one, 12, 1, 1))   # one-letter y
    cases.append((rng.integers(6, 9, 60).astype(np.uint8), one, 12, 2, 2))
    cases.append((rng.integers(20, 24, 80).astype(np.uint8), rng.integers(1, 5, 120).astype(np.uint8), 16, 1, 1))
    xw = rng.integers(1, 5, 50).astype(np.uint8)
    cases.append((xw, xw[5:35].copy(), 30, 1, 1))                             # y of exactly w characters
    cases.append((xw, xw[5:35].copy(), 30, 1, 2))
    for x, y, w, h, r in cases:
        rc, want = ol.plot_rows(x, y, w, h, r)
        assert rc == 0
        assert np.array_equal(gpu_grid(x, y, w, h, r), want), (w, h, r, x.size, y.size)
        t = int(want.max())
        rr, cc = np.nonzero(want >= t)
        gr, gc, gh = ap.plot_threshold_arrays(x, y, cfg(w, h, r), t)
        assert np.array_equal(gr, rr) and np.array_equal(gc, cc) and np.array_equal(gh, want[rr, cc]), (w, h, r)


def test_threshold_staging_overflow_rerun():
    """More hits than the staging area (65536 records on a fresh context) and than the caller's
    capacity: the kernel re-runs with exact staging, the call reports AP_CAPACITY with the exact
    count, and a second call with that capacity returns the oracle's row-major list."""
    import ctypes

    import torch

    from paper_0909_2000_b200 import _native

    rng = np.random.default_rng(5)
    x = rng.integers(1, 5, 420).astype(np.uint8)
    y = rng.integers(1, 5, 400).astype(np.uint8)
    w, h, r, t = 20, 1, 1, 0            # every cell is a hit: 401 x 381 = 152781 > 65536
    rc, want = ol.plot_rows(x, y, w, h, r)
    er, ec = np.nonzero(want >= t)
    L = _native.lib()
    ctx = ctypes.c_void_p()
    assert L.ap_ctx_create(0, ctypes.byref(ctx)) == 0
    try:
        dx, dy = torch.from_numpy(x.copy()).cuda(), torch.from_numpy(y.copy()).cuda()
        c = ap._cfg(cfg(w, h, r, t))
        count = ctypes.c_uint64()
        small = 1000
        dr, dc, dh = (torch.empty(small, dtype=dt, device="cuda") for dt in (torch.int32, torch.int32, torch.int16))
        rc = L.ap_ctx_plot_threshold_device(ctx, dx.data_ptr(), x.size, dy.data_ptr(), y.size, ctypes.byref(c),
                                            ctypes.byref(count), dr.data_ptr(), dc.data_ptr(), dh.data_ptr(), small,
                                            None)
        assert rc == _native.AP_CAPACITY and count.value == er.size
        n = count.value
        dr, dc, dh = (torch.empty(n, dtype=dt, device="cuda") for dt in (torch.int32, torch.int32, torch.int16))
        rc = L.ap_ctx_plot_threshold_device(ctx, dx.data_ptr(), x.size, dy.data_ptr(), y.size, ctypes.byref(c),
                                            ctypes.byref(count), dr.data_ptr(), dc.data_ptr(), dh.data_ptr(), n, None)
        assert rc == 0 and count.value == n
        assert np.array_equal(dr.cpu().numpy(), er) and np.array_equal(dc.cpu().numpy(), ec)
        assert np.array_equal(dh.cpu().numpy().astype(np.int32), want[er, ec])
    finally:
        L.ap_ctx_destroy(ctx)


@pytest.mark.parametrize("w,r,sigma", [(128, 1, 4), (100, 2, 4), (64, 2, 20)])
def test_plot_transpose_symmetry_mid_size(w, r, sigma):
    """Size-independent property at a size the oracle cannot check whole: the window LCS and the
    alignment score are symmetric, so plot(x, y) == plot(y, x)^T (different kernels' row/column
    roles, segments and extraction chunks), here on ~6000 x 5000 grids."""
    rng = np.random.default_rng(w * 10 + r)
    x = rng.integers(1, sigma + 1, 6000).astype(np.uint8)
    y = np.concatenate([x[1000:3500], rng.integers(1, sigma + 1, 2600)]).astype(np.uint8)
    a = ap.plot_dense_u16(x, y, cfg(w, 1, r))
    b = ap.plot_dense_u16(y, x, cfg(w, 1, r))
    assert np.array_equal(a, b.T)
    rc, want = ol.plot_rows(x, y, w, 1, r, 2500, 2502)   # plus two rows against the oracle
    assert rc == 0 and np.array_equal(a[2500:2502].astype(np.int32), want)


def test_c2_full_grid_transpose_symmetry():
    """C2 at full size (16285 x 16280 alignment-score plot): plot(x, y) == plot(y, x)^T."""
    c = datagen.CONFIGS["C2"]
    x, y = datagen.make_inputs("C2")
    a = ap.plot_dense_u16(x, y, cfg(c.w, c.h, c.r))
    b = ap.plot_dense_u16(y, x, cfg(c.w, c.h, c.r))
    assert a.shape == (x.size - c.w + 1, y.size - c.w + 1) and np.array_equal(a, b.T)


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_full_size_threshold_list_transpose_symmetry(name):
    """C3 / C4 at full size: the thresholded list of (x, y) is the transposed list of (y, x)
    (C4: 2.17e6 hits of a 262081 x 262081 plot, row-major order on both sides)."""
    c = datagen.CONFIGS[name]
    x, y = datagen.make_inputs(name)
    r1, c1, h1 = ap.plot_threshold_arrays(x, y, cfg(c.w, c.h, c.r), c.t_half)
    r2, c2, h2 = ap.plot_threshold_arrays(y, x, cfg(c.w, c.h, c.r), c.t_half)
    assert r1.size == r2.size
    # transpose (y, x)'s list and put it in row-major order
    o = np.lexsort((r2, c2))
    assert np.array_equal(r1, c2[o]) and np.array_equal(c1, r2[o]) and np.array_equal(h1, h2[o])
    assert np.all(np.diff(r1.astype(np.int64) * (1 << 32) + c1) > 0)   # strictly row-major


def _mix64(v):
    """splitmix64 finaliser on uint64 arrays (order-independent list checksums)."""
    v = (v ^ (v >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    v = (v ^ (v >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return v ^ (v >> np.uint64(31))


def test_c5_full_size_threshold_checksum_symmetry():
    """C5 at full size (1048321 x 1048321 LCS plot, 1.03e8 hits at WLCS >= 180): the list of
    (x, y) and the transposed list of (y, x) have the same count and the same order-independent
    checksum of (row, col, half); each list is strictly row-major."""
    c = datagen.CONFIGS["C5"]
    x, y = datagen.make_inputs("C5")
    sums = []
    for a, b, swap in ((x, y, False), (y, x, True)):
        rr, cc, hh = ap.plot_threshold_arrays(a, b, cfg(c.w, c.h, c.r), c.t_half)
        key = rr.astype(np.uint64) * np.uint64(1 << 32) + cc.astype(np.uint64)
        assert np.all(np.diff(key.astype(np.int64)) > 0)
        if swap:
            rr, cc = cc, rr
        k = (rr.astype(np.uint64) << np.uint64(32)) | cc.astype(np.uint64)
        with np.errstate(over="ignore"):
            sums.append((rr.size, int(np.sum(_mix64(k ^ (hh.astype(np.uint64) << np.uint64(50))), dtype=np.uint64))))
        del rr, cc, hh, key, k
    assert sums[0] == sums[1]


@pytest.mark.parametrize("w,r", [(64, 1), (128, 1), (50, 2), (100, 2)])
def test_tail_split_equals_unsplit(w, r, monkeypatch):
    """Launches of >= 2 waves cut their last wave of pair groups into half-width tasks (the
    tail split, ap_capi.cu run_device).  At a size where it is active (~6000 x 5000, about
    10000 tasks), the device-API dense plot and the thresholded list must equal the same plot
    with the split disabled (AP_TAIL_SPLIT=1, the path the oracle-checked small plots take),
    and rows around the split boundary must equal the oracle."""
    import ctypes

    import torch

    from paper_0909_2000_b200 import _native

    rng = np.random.default_rng(w * 3 + r)
    x = rng.integers(1, 5, 6000).astype(np.uint8)
    y = np.concatenate([x[1000:3500], rng.integers(1, 5, 2600)]).astype(np.uint8)
    rows, cols = (x.size - w) + 1, y.size - w + 1
    L = _native.lib()
    ctx = ctypes.c_void_p()
    assert L.ap_ctx_create(0, ctypes.byref(ctx)) == 0
    try:
        dx, dy = torch.from_numpy(x.copy()).cuda(), torch.from_numpy(y.copy()).cuda()
        out = torch.empty(rows * cols, dtype=torch.int16, device="cuda")
        c = ap._cfg(cfg(w, 1, r))

        def dense():
            assert L.ap_ctx_plot_dense_device(ctx, dx.data_ptr(), x.size, dy.data_ptr(), y.size, ctypes.byref(c),
                                              out.data_ptr(), None) == 0
            torch.cuda.synchronize()
            return out.cpu().numpy().view(np.uint16).reshape(rows, cols).copy()

        split = dense()
        t = int(np.quantile(split, 0.995))
        lst = ap.plot_threshold_arrays(x, y, cfg(w, 1, r), t)
        monkeypatch.setenv("AP_TAIL_SPLIT", "1")
        unsplit = dense()
        lst1 = ap.plot_threshold_arrays(x, y, cfg(w, 1, r), t)
    finally:
        L.ap_ctx_destroy(ctx)
    assert np.array_equal(split, unsplit)
    for a, b in zip(lst, lst1):
        assert np.array_equal(a, b)
    rr, cc = np.nonzero(split >= t)
    assert np.array_equal(lst[0], rr) and np.array_equal(lst[1], cc) and np.array_equal(lst[2], split[rr, cc])
    for rb in (0, rows // 2, rows - 3):
        rc, want = ol.plot_rows(x, y, w, 1, r, rb, rb + 3)
        assert rc == 0 and np.array_equal(split[rb:rb + 3].astype(np.int32), want), rb


def test_threshold_host_api_concurrent_threads():
    """Thresholded host calls from several threads on one device context (the list
    must not be overwritten between the comb and the copy-out): each gets its own list."""
    import threading
    rng = np.random.default_rng(321)
    cases = []
    for k in range(6):
        w = int(rng.integers(10, 70))
        x = rng.integers(1, 5, w + 300).astype(np.uint8)
        y = np.concatenate([x[20:200], rng.integers(1, 5, 400 + 50 * k)]).astype(np.uint8)
        rc, g = ol.plot_rows(x, y, w, 1, 1 + k % 2)
        t = int(np.quantile(g, 0.98))
        rr, cc = np.nonzero(g >= t)
        cases.append((x, y, w, 1 + k % 2, t, (rr, cc, g[rr, cc])))
    errs, bad = [], []

    def run(i):
        x, y, w, r, t, want = cases[i]
        try:
            for _ in range(4):
                got = ap.plot_threshold_arrays(x, y, cfg(w, 1, r), t)
                if not all(np.array_equal(a, b) for a, b in zip(got, want)):
                    bad.append(i)
        except Exception as e:   # surfaced below
            errs.append(e)

    ts = [threading.Thread(target=run, args=(i,)) for i in range(len(cases))]
    for t_ in ts:
        t_.start()
    for t_ in ts:
        t_.join()
    assert not errs, errs
    assert not bad, bad


def test_threshold_into_single_pass_and_capacity_contract():
    """ap_plot_threshold_into sizes the result through its callback (called once, also for an
    empty list); ap_plot_threshold with a short cap returns the first cap cells + AP_CAPACITY
    and the exact count; ap_plot_threshold_cells fills ap_cell records."""
    import ctypes

    from paper_0909_2000_b200 import _native
    rng = np.random.default_rng(17)
    x = rng.integers(1, 5, 900).astype(np.uint8)
    y = np.concatenate([x[100:600], rng.integers(1, 5, 300)]).astype(np.uint8)
    w, r = 40, 1
    rc, g = ol.plot_rows(x, y, w, 1, r)
    t = int(np.quantile(g, 0.97))
    er, ec = np.nonzero(g >= t)
    L = _native.lib()
    c = ap._cfg(cfg(w, 1, r, t))
    calls = []
    keep = {}

    def alloc(_u, n, pr, pc, ph):
        calls.append(int(n))
        keep["a"] = [np.empty(max(n, 1), dt) for dt in (np.uint32, np.uint32, np.int32)]
        pr[0], pc[0], ph[0] = (a.ctypes.data for a in keep["a"])
        return 0

    count = ctypes.c_uint64()
    xa, ya = np.ascontiguousarray(x), np.ascontiguousarray(y)
    assert L.ap_plot_threshold_into(xa.ctypes.data, x.size, ya.ctypes.data, y.size, ctypes.byref(c),
                                    _native.ListAllocFn(alloc), None, ctypes.byref(count)) == 0
    assert calls == [er.size] and count.value == er.size
    assert np.array_equal(keep["a"][0][:er.size], er) and np.array_equal(keep["a"][1][:er.size], ec)
    # no cell passes: one callback with 0
    c_hi = ap._cfg(cfg(w, 1, r, 10 * w))
    calls.clear()
    assert L.ap_plot_threshold_into(xa.ctypes.data, x.size, ya.ctypes.data, y.size, ctypes.byref(c_hi),
                                    _native.ListAllocFn(alloc), None, ctypes.byref(count)) == 0
    assert calls == [0] and count.value == 0
    # a failing callback aborts with AP_INVALID
    assert L.ap_plot_threshold_into(xa.ctypes.data, x.size, ya.ctypes.data, y.size, ctypes.byref(c),
                                    _native.ListAllocFn(lambda *a: 1), None, ctypes.byref(count)) == _native.AP_INVALID
    # fixed capacity: the first cap cells and the exact count
    k = er.size // 3
    rr, cc, hh = (np.zeros(k, dt) for dt in (np.uint32, np.uint32, np.uint16))
    assert L.ap_plot_threshold(xa.ctypes.data, x.size, ya.ctypes.data, y.size, ctypes.byref(c), ctypes.byref(count),
                               rr.ctypes.data, cc.ctypes.data, hh.ctypes.data, k) == _native.AP_CAPACITY
    assert count.value == er.size and np.array_equal(rr, er[:k]) and np.array_equal(cc, ec[:k])
    cells = (_native.ApCell * er.size)()
    assert L.ap_plot_threshold_cells(xa.ctypes.data, x.size, ya.ctypes.data, y.size, ctypes.byref(c),
                                     ctypes.byref(count), ctypes.cast(cells, ctypes.c_void_p), er.size) == 0
    assert [cl.row for cl in cells] == er.tolist() and [cl.half for cl in cells] == g[er, ec].tolist()


@pytest.mark.parametrize("w,r,h", [(1025, 1, 1), (513, 2, 1), (4096, 1, 2), (2048, 2, 1), (20000, 1, 1),
                                   (10000, 2, 3), (65534, 1, 1), (32767, 2, 1)])
def test_large_windows_vs_reference(w, r, h):
    """Blown windows above the packed kernels' 1024 run on the large-window path (32-bit keys,
    one CTA per strip, band by band); the reference's sea16 engine plots any w*r <= 65534
    (model.cpp:57-59, lane_kernel.cpp:117-123).  Dense grids and thresholded lists against
    oracle/_ref sea16 at w*r = 1025, 1026, 4096, 20000 and the 65534 bound."""
    import os
    assert ol.ref_available()
    rng = np.random.default_rng(w * 2 + r + h)
    W = w * r
    rows = 5 if W <= 20000 else 2
    m = w + (rows - 1) * h
    x = rng.integers(1, 5, m).astype(np.uint8)
    blk = x[: w].copy()
    flip = rng.random(blk.size) < 0.15
    blk[flip] = rng.integers(1, 5, int(flip.sum()))
    y = np.concatenate([rng.integers(1, 5, 120), blk, rng.integers(1, 5, 180)]).astype(np.uint8)
    rc, want, err = ol.ref_compute_plot(x, y, w, h, r, ol.SEA16, os.cpu_count() or 8)
    assert rc == 0, err
    got = ap.plot_dense_i32(x, y, cfg(w, h, r))
    assert got.shape == want.shape and np.array_equal(got, want), (w, r, h)
    if ap.scores_fit_u16(cfg(w, h, r)):
        assert np.array_equal(gpu_grid(x, y, w, h, r), want)
    else:   # LCS scores up to 2w > 65535 half-units: the uint16 entry points refuse
        with pytest.raises(ap.ConfigError):
            gpu_grid(x, y, w, h, r)
    grid = ap.compute_plot(ap.Sequence("x", x), ap.Sequence("y", y), cfg(w, h, r))
    assert np.array_equal(grid.matrix(), want)
    t = int(np.quantile(want, 0.9))
    rr, cc = np.nonzero(want >= t)
    gr, gc, gh = ap.plot_threshold_arrays(x, y, cfg(w, h, r), t)
    assert np.array_equal(gr, rr) and np.array_equal(gc, cc) and np.array_equal(gh, want[rr, cc])


@pytest.mark.parametrize("variant", ["default", "no_pack", "no_table"])
def test_large_window_many_rows_and_bound(variant, monkeypatch):
    """Large-window path over many rows (several strips per launch, odd row counts, both modes,
    row ranges) against the oracle, in all three kernels: packed strip pairs with 16-bit keys and
    CTA-wide rebasing (the default for alphabets of <= 8 codes and W up to ~28K), 32-bit keys with
    the mask table (AP_WIDE_NO_PACK), computed masks (AP_WIDE_NO_TABLE, and a 20-letter alphabet);
    and the sea16 bound: w*r = 65535 is a ConfigError before device work."""
    if variant == "no_pack":
        monkeypatch.setenv("AP_WIDE_NO_PACK", "1")
    if variant == "no_table":
        monkeypatch.setenv("AP_WIDE_NO_TABLE", "1")
    rng = np.random.default_rng(1100)
    for w, r, sigma in ((1100, 1, 4), (600, 2, 4), (1500, 1, 20), (4200, 1, 3)):
        x = rng.integers(1, sigma + 1, w + 300).astype(np.uint8)   # 301 rows: the last pair is half
        y = np.concatenate([x[100:w + 200], rng.integers(1, sigma + 1, 400)]).astype(np.uint8)
        rc, want = ol.plot_rows(x, y, w, 1, r, 40, 140)
        assert rc == 0
        got = gpu_grid(x, y, w, 1, r, 40, 140)
        assert np.array_equal(got, want), (w, r, sigma)
        t = int(np.quantile(want, 0.95))
        rr, cc = np.nonzero(want >= t)
        gr, gc, gh = ap.plot_threshold_arrays(x, y, cfg(w, 1, r), t, row_begin=40, row_end=140)
        assert np.array_equal(gr - 40, rr) and np.array_equal(gc, cc) and np.array_equal(gh, want[rr, cc])
    with pytest.raises(ap.ConfigError):
        ap.plot_dense_u16(np.ones(70000, np.uint8), np.ones(70000, np.uint8), cfg(65535, 1, 1))
    with pytest.raises(ap.ConfigError):
        ap.plot_dense_u16(np.ones(40000, np.uint8), np.ones(40000, np.uint8), cfg(32768, 1, 2))


def test_dense_host_output_pinned_and_pageable_agree(monkeypatch):
    """Dense host output into pageable memory goes through the pinned bounce ring (parallel host
    copies); into pinned memory it is copied directly.  Both must give the oracle's grid, for
    uint16, uint8 and int32 outputs and a plot larger than several bounce slots."""
    import ctypes

    import torch

    from paper_0909_2000_b200 import _native
    rng = np.random.default_rng(606)
    x = rng.integers(1, 5, 5000).astype(np.uint8)
    y = np.concatenate([x[200:2200], rng.integers(1, 5, 6000)]).astype(np.uint8)
    w, h, r = 60, 1, 2
    rows, cols = x.size - w + 1, y.size - w + 1      # 4941 x 7941: 78 MB of uint16 (10 bounce slots)
    want = ap.plot_dense_u16(x, y, cfg(w, h, r))
    monkeypatch.setenv("AP_NO_BOUNCE", "1")
    assert np.array_equal(ap.plot_dense_u16(x, y, cfg(w, h, r)), want)
    monkeypatch.delenv("AP_NO_BOUNCE")
    pinned = torch.empty(rows * cols, dtype=torch.int16).pin_memory()
    L = _native.lib()
    c = ap._cfg(cfg(w, h, r))
    assert L.ap_plot_dense(x.ctypes.data, x.size, y.ctypes.data, y.size, ctypes.byref(c), pinned.data_ptr()) == 0
    assert np.array_equal(pinned.numpy().view(np.uint16).reshape(rows, cols), want)
    assert np.array_equal(ap.plot_dense_i32(x, y, cfg(w, h, r)), want.astype(np.int32))
    assert np.array_equal(ap.plot_dense_u8(x, y, cfg(w, h, r)), want.astype(np.uint8))
    rc, ref_rows = ol.plot_rows(x, y, w, h, r, 4000, 4003)
    assert rc == 0 and np.array_equal(want[4000:4003].astype(np.int32), ref_rows)


def test_large_window_packed_rebases_over_long_y():
    """The packed large-window kernel rebases its 16-bit keys every (0x7000 - W - 64 warps - 64)
    columns; over a y of 120K columns at W = 20000 (rebase step 8096, ~15 rebases) and W = 2000 with
    r = 2 (W = 4000), planted homology far from the start must still give the oracle's rows."""
    rng = np.random.default_rng(7070)
    for w, r, n in ((20000, 1, 120000), (2000, 2, 60000)):
        x = rng.integers(1, 5, w + 3).astype(np.uint8)
        blk = x[:w].copy()
        flip = rng.random(w) < 0.1
        blk[flip] = rng.integers(1, 5, int(flip.sum()))
        y = np.concatenate([rng.integers(1, 5, n - w - 500), blk, rng.integers(1, 5, 500)]).astype(np.uint8)
        rc, want, err = ol.ref_compute_plot(x, y, w, 1, r, ol.SEA16, 16)
        assert rc == 0, err
        assert np.array_equal(ap.plot_dense_i32(x, y, cfg(w, 1, r)), want), (w, r)


@pytest.mark.parametrize("ndev", [2, 3])
def test_multi_shard_capacity_and_cells(ndev, monkeypatch):
    """Several shard devices (one GPU standing in): a fixed capacity that ends inside the second
    shard's list gets exactly the first cap cells of the global row-major list, the ap_cell form
    and the int32 dense form agree with one device, and a row range crossing shards too."""
    import ctypes

    from paper_0909_2000_b200 import _native
    monkeypatch.setenv("AP_SHARDS_PER_DEVICE", str(ndev))
    rng = np.random.default_rng(900 + ndev)
    x = rng.integers(1, 5, 1200).astype(np.uint8)
    y = np.concatenate([x[100:900], rng.integers(1, 5, 400)]).astype(np.uint8)
    w, h, r = 40, 1, 2
    rc, want = ol.plot_rows(x, y, w, h, r)
    t = int(np.quantile(want, 0.97))
    er, ec = np.nonzero(want >= t)
    c = ap._cfg(cfg(w, h, r, t, n_devices=ndev))
    L = _native.lib()
    cap = int(er.size * 0.6)            # ends inside a later shard's part of the list
    rr, cc, hh = (np.zeros(cap, dt) for dt in (np.uint32, np.uint32, np.uint16))
    count = ctypes.c_uint64()
    assert L.ap_plot_threshold(x.ctypes.data, x.size, y.ctypes.data, y.size, ctypes.byref(c), ctypes.byref(count),
                               rr.ctypes.data, cc.ctypes.data, hh.ctypes.data, cap) == _native.AP_CAPACITY
    assert count.value == er.size
    assert np.array_equal(rr, er[:cap]) and np.array_equal(cc, ec[:cap])
    assert np.array_equal(hh.astype(np.int32), want[er[:cap], ec[:cap]])
    cells = ap.plot_threshold_cells(x, y, cfg(w, h, r, n_devices=ndev), t)
    assert [q.row for q in cells] == er.tolist() and [q.score_half for q in cells] == want[er, ec].tolist()
    dense = ap.plot_dense_i32(x, y, cfg(w, h, r, n_devices=ndev))
    assert np.array_equal(dense, want)
    part = ap.plot_threshold_arrays(x, y, cfg(w, h, r, n_devices=ndev), t, row_begin=300, row_end=900)
    sel = (er >= 300) & (er < 900)
    assert np.array_equal(part[0], er[sel]) and np.array_equal(part[1], ec[sel])


def test_empty_row_ranges():
    """row_begin == row_end (and a range past the last row): no device work, an empty dense block,
    a zero count with one allocation callback of 0, for the packed and the large-window paths."""
    rng = np.random.default_rng(12)
    x = rng.integers(1, 5, 3000).astype(np.uint8)
    y = rng.integers(1, 5, 3200).astype(np.uint8)
    for w, r in ((40, 1), (30, 2), (1500, 1)):
        rows = x.size - w + 1
        for rb, re in ((5, 5), (rows, rows + 10)):
            assert ap.plot_dense_u16(x, y, cfg(w, 1, r), rb, re).shape[0] == 0
            got = ap.plot_threshold_arrays(x, y, cfg(w, 1, r), -10, row_begin=rb, row_end=re)
            assert all(a.size == 0 for a in got), (w, r, rb, re)
