"""Host-side mirror of the reference interface (paper_0909_2000_b200.alignplot) and the
synthetic input generator — CPU only, no device calls."""
import numpy as np
import pytest

from paper_0909_2000_b200 import alignplot as ap
from paper_0909_2000_b200 import datagen


def test_sequence_validation():
    # test_model.cpp:5-17
    s = ap.Sequence.from_text("s", "ACGTN#z")
    assert s.size() == 7 and s.codes()[4] == ord("N")
    with pytest.raises(ap.ConfigError):
        ap.Sequence("bad", [1, 0, 2])
    with pytest.raises(ap.ConfigError):
        ap.Sequence("bad", [1, 5, 2], 4)
    ap.Sequence("ok", [1, 3, 2], 4)


def test_mode_names_round_trip():
    for m in ap.Mode:
        assert ap.mode_from_name(ap.mode_name(m)) == m
    assert ap.mode_from_name("sea32") is None


def test_grid_dims():
    assert ap.window_grid_dims(100, 100, 100, 5) == (1, 1)
    assert ap.window_grid_dims(2712, 628, 100, 5) == (523, 529)
    assert ap.window_grid_dims(105, 100, 100, 5) == (2, 1)
    with pytest.raises(ap.EmptyPlotError):
        ap.window_grid_dims(10, 10, 20, 1)


def test_config_validation_matches_reference_order():
    # test_model.cpp:49-92
    c = ap.PlotConfig(window_w=100, step_h=5)
    c.validate(200, 200)
    for kw in ({"window_w": 0}, {"step_h": 0}, {"workers": 0}, {"blowup_r": 3}):
        with pytest.raises(ap.ConfigError):
            ap.PlotConfig(**{**dict(window_w=100, step_h=5), **kw}).validate(200, 200)
    with pytest.raises(ap.EmptyPlotError):
        c.validate(50, 200)
    s8 = ap.PlotConfig(window_w=255, step_h=1, mode=ap.Mode.sea8)
    with pytest.raises(ap.ConfigError):
        s8.validate(300, 300)
    ap.PlotConfig(window_w=254, step_h=1, blowup_r=1, mode=ap.Mode.sea8).validate(300, 300)
    ap.PlotConfig(window_w=255, step_h=1, blowup_r=1, mode=ap.Mode.sea16).validate(300, 300)
    # Mode.cuda: the sea16 bound (model.cpp:57-59), w*r <= 65534
    ap.PlotConfig(window_w=513, step_h=1, blowup_r=2, mode=ap.Mode.cuda).validate(2000, 2000)
    ap.PlotConfig(window_w=32767, step_h=1, blowup_r=2, mode=ap.Mode.cuda).validate(40000, 40000)
    with pytest.raises(ap.ConfigError):
        ap.PlotConfig(window_w=32768, step_h=1, blowup_r=2, mode=ap.Mode.cuda).validate(40000, 40000)


def test_plan_strips():
    # test_runner.cpp:12-28
    cfg = ap.PlotConfig(window_w=100, step_h=5)
    assert [(t.row_index, t.x_offset) for t in ap.plan_strips(cfg, 100)] == [(0, 0)]
    many = ap.plan_strips(cfg, 2712)
    assert len(many) == 523 and many[1].x_offset == 5 and many[522].x_offset == 2610
    with pytest.raises(ap.EmptyPlotError):
        ap.plan_strips(cfg, 99)


def test_scoring_helpers():
    # test_scoring.cpp:11-37, 55-68
    b = ap.blowup(ap.Sequence.from_text("s", "abab"))
    assert list(b.data) == [0, 97, 0, 98, 0, 97, 0, 98] and b.raw_len == 4
    assert list(ap.unblow(b)) == [97, 98, 97, 98]
    assert ap.blowup(np.zeros(0, np.uint8)).data.size == 0
    with pytest.raises(ap.ConfigError):
        ap.blowup(np.array([1, 0, 2], np.uint8))
    assert ap.recover_score(4, 2, 2) == 4 and ap.recover_score(2, 2, 2) == 0 and ap.recover_score(2, 1, 2) == 1
    g = ap.PlotGrid(2, 2, 4, 1, values=np.array([4, 1, 3, 4], np.int32))
    assert ap.apply_threshold(g, 3) == [ap.PlotCell(0, 0, 4), ap.PlotCell(1, 0, 3), ap.PlotCell(1, 1, 4)]
    assert ap.apply_threshold(g, 5) == [] and len(ap.apply_threshold(g, -10)) == 4


def test_plot_grid_geometry():
    # test_model.cpp:84-92
    g = ap.PlotGrid(3, 4, 10, 5, values=np.zeros(12, np.int32))
    assert g.x_offset(0) == 0 and g.x_offset(2) == 10 and g.y_offset(3) == 3


def test_datagen_deterministic_and_shaped():
    for name in datagen.CONFIGS:
        x1, y1 = datagen.make_inputs(name, scale=0.01)
        x2, y2 = datagen.make_inputs(name, scale=0.01)
        assert np.array_equal(x1, x2) and np.array_equal(y1, y2)
        assert x1.dtype == np.uint8 and (x1 != 0).all() and (y1 != 0).all()
    x, y = datagen.make_inputs("C2")
    assert x.size == 16384 and abs(y.size - x.size) < 200
    x, _ = datagen.make_inputs("C4", scale=0.05)
    assert set(np.unique(x).tolist()) <= set(datagen.PROTEIN.tolist())
    x, y = datagen.make_inputs("C5", scale=0.05)
    same = (x == y).mean()
    assert 0.6 < same < 0.8   # ~70% of blocks kept (fresh blocks still agree 1/4), then 5% substitutions
