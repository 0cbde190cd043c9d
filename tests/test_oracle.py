"""Pins the CPU oracle (oracle/alignplot_oracle.c) before it is trusted as the parity checker.

Checks it against (1) the known-answer vectors written in the reference unit
tests and (2) the golden fixtures the reference library itself produced
(tests/golden/*.json, oracle/golden_gen.cpp), and (3) cross-checks it against
the compiled reference (oracle/_ref) on fresh random instances when that
library is present.  CPU only.
"""
import numpy as np
import pytest

import golden_util as gu
import oracle_lib as ol


# ---- known answers from the reference unit tests ---------------------------------------------

def test_single_cell_match_and_mismatch():
    # test_seaweed.cpp:29-43
    bs, rs = ol.comb_strip(b"a", b"a")
    assert list(bs) == [-1] and list(rs) == [0]
    bs, rs = ol.comb_strip(b"a", b"b")
    assert list(bs) == [0] and list(rs) == [-1]


def test_all_mismatch_strip_falls_straight_through():
    # test_lane_kernel.cpp:72-86
    bs, _ = ol.comb_strip([1, 2, 3], [10, 11, 12, 13, 14])
    assert list(bs) == [0, 1, 2, 3, 4]


def test_window_scan_kat():
    # test_seaweed.cpp:140-146: "aaa" vs "aaabbb", W=3 -> [3,2,1,0]
    bs, _ = ol.comb_strip(b"aaa", b"aaabbb")
    rc, ll = ol.window_llcs(bs, 3, 1)
    assert rc == 0 and list(ll) == [3, 2, 1, 0]


def test_window_scan_rejects_malformed():
    # test_seaweed.cpp:167-178
    bs, _ = ol.comb_strip(b"ab", b"ab")
    assert ol.window_llcs(bs, 0, 1)[0] == 3
    assert ol.window_llcs(bs, 3, 1)[0] == 3
    assert ol.window_llcs(bs, 2, 0)[0] == 3


def test_every_seaweed_exits_once():
    # test_seaweed.cpp:45-73 (permutation property), own seeded instances
    rng = np.random.default_rng(7)
    for it in range(60):
        w, n = 1 + it % 6, 1 + (it * 7) % 12
        sigma = 2 if it % 2 else 4
        xw = rng.integers(1, sigma + 1, w)
        y = rng.integers(1, sigma + 1, n)
        bs, rs = ol.comb_strip(xw, y)
        starts = set(bs.tolist())
        assert len(starts) == n
        starts |= set(rs.tolist())
        assert len(starts) == w + n
        assert min(starts) == -w and max(starts) == n - 1


def test_llcs_query_exhaustive_small_binary():
    # test_seaweed.cpp:111-129 (Theorem 1 identity), w <= 4, n <= 6
    L = ol.oracle()
    import ctypes
    for w in range(1, 5):
        for xb in range(1 << w):
            xw = np.array([2 if (xb >> k) & 1 else 1 for k in range(w)], dtype=np.uint8)
            for n in range(1, 7):
                for yb in range(1 << n):
                    y = np.array([2 if (yb >> k) & 1 else 1 for k in range(n)], dtype=np.uint8)
                    bs, rs = ol.comb_strip(xw, y)
                    for i in range(n + 1):
                        for j in range(i, n + 1):
                            out = ctypes.c_size_t()
                            L.or_llcs_query(ol._p(bs), n, ol._p(rs), w, i, j, ctypes.byref(out))
                            assert out.value == ol.ref_llcs(xw, y[i:j])


def test_blowup_and_score_recovery():
    # test_scoring.cpp:11-37
    import ctypes
    L = ol.oracle()
    raw = ol.u8(b"abab")
    out = np.empty(8, dtype=np.uint8)
    assert L.or_blowup(ol._p(raw), 4, ol._p(out)) == 0
    assert list(out) == [0, ord("a"), 0, ord("b"), 0, ord("a"), 0, ord("b")]
    bad = ol.u8([1, 0, 2])
    assert L.or_blowup(ol._p(bad), 3, ol._p(np.empty(6, dtype=np.uint8))) == 1
    assert L.or_recover_score(4, 2, 2) == 4
    assert L.or_recover_score(2, 2, 2) == 0
    assert L.or_recover_score(2, 1, 2) == 1


def test_blown_llcs_is_alignment_score():
    # test_scoring.cpp:39-53 / acceptance.cpp:210-229
    L = ol.oracle()
    rng = np.random.default_rng(1234)
    for sigma in (2, 4, 20):
        for _ in range(40):
            a = rng.integers(1, sigma + 1, rng.integers(0, 25)).astype(np.uint8)
            b = rng.integers(1, sigma + 1, rng.integers(0, 25)).astype(np.uint8)
            ab = np.zeros(2 * a.size, np.uint8); ab[1::2] = a
            bb = np.zeros(2 * b.size, np.uint8); bb[1::2] = b
            llcs = ol.ref_llcs(ab, bb)
            assert L.or_recover_score(llcs, a.size, b.size) == ol.ref_align_score_half(a, b)


def test_grid_dims():
    # test_model.cpp:27-35
    assert ol.grid_dims(100, 100, 100, 5) == (0, 1, 1)
    assert ol.grid_dims(2712, 628, 100, 5) == (0, 523, 529)
    assert ol.grid_dims(104, 100, 100, 5) == (0, 1, 1)
    assert ol.grid_dims(105, 100, 100, 5) == (0, 2, 1)
    assert ol.grid_dims(10, 10, 20, 1)[0] == 2
    assert ol.grid_dims(50, 10, 20, 1)[0] == 2


def test_validate():
    # test_model.cpp:49-79
    L = ol.oracle()
    assert L.or_validate(200, 200, 100, 5, 2, 1, 4) == 0
    assert L.or_validate(200, 200, 0, 5, 2, 1, 4) == 1
    assert L.or_validate(200, 200, 100, 0, 2, 1, 4) == 1
    assert L.or_validate(200, 200, 100, 5, 2, 0, 4) == 1
    assert L.or_validate(200, 200, 100, 5, 3, 1, 4) == 1
    assert L.or_validate(50, 200, 100, 5, 2, 1, 4) == 2
    assert L.or_validate(300, 300, 255, 1, 1, 1, 4) == 1
    assert L.or_validate(300, 300, 254, 1, 1, 1, 4) == 0
    assert L.or_validate(300, 300, 255, 1, 1, 1, 3) == 0


def test_threshold_order():
    # test_scoring.cpp:55-68
    import ctypes
    L = ol.oracle()
    g = np.array([[4, 1], [3, 4]], dtype=np.int32)
    r = np.empty(4, np.uint64); c = np.empty(4, np.uint64); h = np.empty(4, np.int32)
    k = L.or_apply_threshold(ol._p(g), 2, 2, 3, ol._p(r), ol._p(c), ol._p(h), 4)
    assert k == 3
    assert list(zip(r[:3], c[:3], h[:3])) == [(0, 0, 4), (1, 0, 3), (1, 1, 4)]
    assert L.or_apply_threshold(ol._p(g), 2, 2, 5, ol._p(r), ol._p(c), ol._p(h), 4) == 0
    assert L.or_apply_threshold(ol._p(g), 2, 2, -10, ol._p(r), ol._p(c), ol._p(h), 4) == 4


def test_identical_windows_score_maximum():
    # test_runner.cpp:129-145
    rc, g = ol.plot_rows(np.ones(25, np.uint8), np.ones(11, np.uint8), 10, 5, 1)
    assert rc == 0 and g.shape == (4, 2) and g[0, 0] == 20


# ---- golden fixtures from the reference library -----------------------------------------------

def _grid_of(case):
    x, y = gu.unhex(case["x"]), gu.unhex(case["y"])
    rc, g = ol.plot_rows(x, y, case["w"], case["h"], case["r"])
    assert rc == 0
    assert g.shape == (case["rows"], case["cols"])
    return g


@pytest.mark.parametrize("name", ["runner_engines.json", "runner_modes.json"])
def test_oracle_matches_reference_grids(name):
    for case in gu.load(name)["cases"]:
        g = _grid_of(case)
        assert np.array_equal(g.reshape(-1), np.array(case["grid"], dtype=np.int32))
        assert gu.grid_hash(g) == int(case["hash"])


def test_oracle_matches_reference_strips():
    for case in gu.load("strips.json")["cases"]:
        xw, y = gu.unhex(case["xw"]), gu.unhex(case["y"])
        if case["r"] == 2:
            xb = np.zeros(2 * xw.size, np.uint8); xb[1::2] = xw
            yb = np.zeros(2 * y.size, np.uint8); yb[1::2] = y
            xw, y = xb, yb
        bs, _ = ol.comb_strip(xw, y)
        if "starts" in case:
            assert list(bs) == case["starts"]
        rc, ll = ol.window_llcs(bs, case["window_cols"], case["stride"])
        assert rc == 0 and list(ll) == case["llcs"]


def test_oracle_matches_reference_acceptance1():
    cases = gu.load("acceptance1.json")["cases"]
    assert len(cases) == 540
    for case in cases:
        assert gu.grid_hash(_grid_of(case)) == int(case["hash"]), case


def test_oracle_matches_reference_acceptance7():
    (case,) = gu.load("acceptance7.json")["cases"]
    assert gu.grid_hash(_grid_of(case)) == int(case["hash"])


@pytest.mark.skipif(not ol.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
def test_oracle_matches_compiled_reference_random():
    rng = np.random.default_rng(99)
    for it in range(30):
        w = int(rng.integers(2, 40))
        m, n = int(rng.integers(w, 160)), int(rng.integers(w, 160))
        sigma = [2, 4, 20][it % 3]
        x = rng.integers(1, sigma + 1, m).astype(np.uint8)
        y = rng.integers(1, sigma + 1, n).astype(np.uint8)
        h, r = 1 + it % 3, 1 + it % 2
        rc, g = ol.plot_rows(x, y, w, h, r)
        rc2, g2, _ = ol.ref_compute_plot(x, y, w, h, r)
        assert rc == rc2 == 0 and np.array_equal(g, g2)
