"""Python mirror of the reference ``alignplot`` library interface for the hot path.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/include/alignplot/*.hpp), with the compute routed through
the B200 engine's C ABI (include/alignplot_b200.h):

=====================  =====================================================
reference              here
=====================  =====================================================
``Sequence``           ``Sequence``            (model.hpp:38-52, model.cpp:7-24)
``PlotConfig``         ``PlotConfig``          (model.hpp:70-86, model.cpp:46-61)
``Mode``               ``Mode`` (+ ``cuda``)   (model.hpp:65)
``window_grid_dims``   ``window_grid_dims``    (model.cpp:63-72)
``PlotGrid``           ``PlotGrid``            (model.hpp:95-114)
``plan_strips``        ``plan_strips``         (runner.cpp:15-27)
``compute_plot``       ``compute_plot``        (runner.cpp:78-131) -> ap_plot_dense
``blowup``/``unblow``  same                    (scoring.cpp:5-24)
``recover_score``      same                    (scoring.cpp:26-28)
``apply_threshold``    ``apply_threshold``     (scoring.cpp:30-39)
(grid + threshold)     ``compute_plot_threshold`` -> ap_plot_threshold (fused)
=====================  =====================================================

Every reference ``Mode`` is served by the CUDA engine: the reference proves
all engines produce the identical grid (acceptance.cpp:34-73), so routing
them to one engine preserves outputs, while ``PlotConfig.validate`` keeps each
mode's own limits (sea8 w <= 254, sea16 w*r <= 65534) so a config the
reference rejects is still rejected.  ``Mode.cuda`` carries the sea16 bound
(w*r <= 65534); blown windows above 1024 run on the large-window kernels.
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence as _Seq

import numpy as np

from . import _native

SENTINEL_CODE = 0  # kSentinelCode, model.hpp:34


class ConfigError(RuntimeError):
    """model.hpp:17-20."""


class EmptyPlotError(ConfigError):
    """model.hpp:22-26: no window of the requested size fits the inputs."""


class NoDeviceError(RuntimeError):
    """No CUDA device: the engine has no CPU fallback."""


class EngineError(RuntimeError):
    """A CUDA runtime failure inside the engine."""


def _raise(rc: int) -> None:
    if rc == _native.AP_OK:
        return
    msg = _native.last_error()
    if rc == _native.AP_EMPTY:
        raise EmptyPlotError(msg)
    if rc == _native.AP_CONFIG:
        raise ConfigError(msg)
    if rc == _native.AP_INVALID:
        raise ValueError(msg)
    if rc == _native.AP_NODEV:
        raise NoDeviceError(msg)
    raise EngineError(f"status {rc}: {msg}")


class Mode(enum.IntEnum):
    """model.hpp:65, plus the B200 engine."""
    dp = 0
    blcs = 1
    sea_scalar = 2
    sea16 = 3
    sea8 = 4
    cuda = 5


def mode_name(m: Mode) -> str:
    return Mode(m).name


def mode_from_name(name: str) -> Optional[Mode]:
    try:
        return Mode[name]
    except KeyError:
        return None


class Sequence:
    """A validated byte string (model.cpp:7-19): code 0 is reserved, codes must be < alphabet_size."""

    def __init__(self, name: str, data, alphabet_size: int = 256):
        self.name = name
        self.data = np.ascontiguousarray(np.frombuffer(bytes(data), dtype=np.uint8)
                                         if isinstance(data, (bytes, bytearray)) else np.asarray(data, dtype=np.uint8))
        self.alphabet_size = alphabet_size
        if self.data.size and (self.data == SENTINEL_CODE).any():
            raise ConfigError(f"sequence '{name}' contains the reserved sentinel code 0")
        if alphabet_size < 256 and self.data.size and int(self.data.max()) >= alphabet_size:
            bad = int(self.data[self.data >= alphabet_size][0])
            raise ConfigError(f"sequence '{name}' contains code {bad} outside alphabet of size {alphabet_size}")

    @staticmethod
    def from_text(name: str, text) -> "Sequence":
        return Sequence(name, text.encode("latin-1") if isinstance(text, str) else bytes(text))

    def size(self) -> int:
        return int(self.data.size)

    def __len__(self) -> int:
        return int(self.data.size)

    def codes(self) -> np.ndarray:
        return self.data


@dataclass
class PlotConfig:
    """model.hpp:70-86 (defaults w=100, h=5, r=2, sea8, 1 worker) + device sharding."""
    window_w: int = 100
    step_h: int = 5
    blowup_r: int = 2
    threshold_half: Optional[int] = None
    mode: Mode = Mode.sea8
    workers: int = 1
    n_devices: int = 1

    def validate(self, m: int, n: int) -> None:
        """model.cpp:46-61, in the same order, plus the CUDA engine limit."""
        if self.window_w == 0:
            raise ConfigError("window size must be positive")
        if self.step_h == 0:
            raise ConfigError("step size must be positive")
        if self.workers == 0:
            raise ConfigError("worker count must be positive")
        if self.blowup_r not in (1, 2):
            raise ConfigError("blowup factor must be 1 (LCS) or 2 (alignment score)")
        if self.mode == Mode.sea8 and self.window_w + 1 > 255:
            raise ConfigError(f"sea8 mode supports windows up to 254 (got {self.window_w}): "
                              "spans plus INF must fit 8-bit lanes")
        if self.mode == Mode.sea16 and self.window_w * self.blowup_r + 1 > 65535:
            raise ConfigError("sea16 mode supports blown windows up to 65534")
        window_grid_dims(m, n, self.window_w, self.step_h)
        if self.window_w * self.blowup_r > _native.AP_MAX_BLOWN_WINDOW:
            raise ConfigError(f"blown windows up to {_native.AP_MAX_BLOWN_WINDOW} are supported "
                              f"(got {self.window_w * self.blowup_r})")


def window_grid_dims(m: int, n: int, w: int, h: int):
    """model.cpp:63-72: (rows, cols) = ((m-w)//h + 1, n-w+1)."""
    if w == 0 or h == 0:
        raise ConfigError("window and step must be positive")
    if w > m or w > n:
        raise EmptyPlotError(f"no window of size {w} fits inputs of lengths {m} and {n}")
    return (m - w) // h + 1, n - w + 1


@dataclass
class PlotGrid:
    """model.hpp:95-114: row-major half-unit scores; row i = x-window at row_origin + i*step_h."""
    rows: int = 0
    cols: int = 0
    window_w: int = 0
    step_h: int = 1
    row_origin: int = 0
    col_origin: int = 0
    values: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int32))

    def at(self, r: int, c: int) -> int:
        return int(self.values[r * self.cols + c])

    def x_offset(self, r: int) -> int:
        return self.row_origin + r * self.step_h

    def y_offset(self, c: int) -> int:
        return self.col_origin + c

    def matrix(self) -> np.ndarray:
        return self.values.reshape(self.rows, self.cols)

    def __eq__(self, other) -> bool:
        return (isinstance(other, PlotGrid) and self.rows == other.rows and self.cols == other.cols
                and self.window_w == other.window_w and self.step_h == other.step_h
                and self.row_origin == other.row_origin and self.col_origin == other.col_origin
                and np.array_equal(self.values, other.values))


@dataclass(frozen=True)
class StripTask:
    """runner.hpp:11-17."""
    row_index: int
    x_offset: int
    engine: Mode


def plan_strips(cfg: PlotConfig, m: int) -> List[StripTask]:
    """runner.cpp:15-27: one task per grid row."""
    if cfg.window_w > m:
        raise EmptyPlotError(f"no window of size {cfg.window_w} fits an input of length {m}")
    rows = (m - cfg.window_w) // cfg.step_h + 1
    return [StripTask(r, r * cfg.step_h, cfg.mode) for r in range(rows)]


@dataclass
class BlownSequence:
    """scoring.hpp:13-22."""
    data: np.ndarray
    raw_len: int

    def codes(self) -> np.ndarray:
        return self.data

    def size(self) -> int:
        return int(self.data.size)


def blowup(raw) -> BlownSequence:
    """scoring.cpp:5-17: "abab" -> "$a$b$a$b" (sentinel 0 before every character)."""
    a = raw.codes() if isinstance(raw, Sequence) else np.asarray(raw, dtype=np.uint8)
    if a.size and (a == SENTINEL_CODE).any():
        raise ConfigError("cannot blow up a sequence that contains the sentinel code")
    out = np.zeros(2 * a.size, dtype=np.uint8)
    out[1::2] = a
    return BlownSequence(out, int(a.size))


def unblow(b: BlownSequence) -> np.ndarray:
    """scoring.cpp:19-24."""
    return b.data[1::2].copy()


def recover_score(llcs_blown: int, m: int, n: int) -> int:
    """scoring.cpp:26-28: half = 2*llcs_blown - (m+n)."""
    return 2 * llcs_blown - (m + n)


@dataclass(frozen=True)
class PlotCell:
    """scoring.hpp:33-39."""
    row: int
    col: int
    score_half: int


def apply_threshold(grid: PlotGrid, t_half: int) -> List[PlotCell]:
    """scoring.cpp:30-39: cells with score >= t, row-major."""
    v = grid.values.reshape(grid.rows, grid.cols)
    rr, cc = np.nonzero(v >= t_half)
    return [PlotCell(int(r), int(c), int(v[r, c])) for r, c in zip(rr, cc)]


def _ptr(a: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


def _cfg(cfg: PlotConfig, row_begin: int = 0, row_end: int = 0) -> _native.ApConfig:
    c = _native.ApConfig()
    c.window_w = cfg.window_w
    c.step_h = cfg.step_h
    c.blowup_r = cfg.blowup_r
    c.has_threshold = 1 if cfg.threshold_half is not None else 0
    c.threshold_half = int(cfg.threshold_half) if cfg.threshold_half is not None else 0
    c.n_devices = max(1, int(cfg.n_devices))
    c.row_begin = row_begin
    c.row_end = row_end
    return c


def _codes(s) -> np.ndarray:
    if isinstance(s, Sequence):
        return s.codes()
    return np.ascontiguousarray(np.asarray(s, dtype=np.uint8))


def plot_dense_u16(x, y, cfg: PlotConfig, row_begin: int = 0, row_end: int = 0) -> np.ndarray:
    """Dense uint16 half-unit grid of rows [row_begin, row_end) via ap_plot_dense."""
    xa, ya = _codes(x), _codes(y)
    rows, cols = window_grid_dims(xa.size, ya.size, cfg.window_w, cfg.step_h)
    re = rows if row_end == 0 else min(row_end, rows)
    out = np.empty((max(re - row_begin, 0), cols), dtype=np.uint16)
    _raise(_native.lib().ap_plot_dense(_ptr(xa), xa.size, _ptr(ya), ya.size,
                                       ctypes.byref(_cfg(cfg, row_begin, row_end)), _ptr(out)))
    return out


def plot_dense_u8(x, y, cfg: PlotConfig, row_begin: int = 0, row_end: int = 0) -> np.ndarray:
    """Dense half-unit grid as bytes (w <= 127) via ap_plot_dense_u8: half the D2H of uint16."""
    xa, ya = _codes(x), _codes(y)
    rows, cols = window_grid_dims(xa.size, ya.size, cfg.window_w, cfg.step_h)
    re = rows if row_end == 0 else min(row_end, rows)
    out = np.empty((max(re - row_begin, 0), cols), dtype=np.uint8)
    _raise(_native.lib().ap_plot_dense_u8(_ptr(xa), xa.size, _ptr(ya), ya.size,
                                          ctypes.byref(_cfg(cfg, row_begin, row_end)), _ptr(out)))
    return out


def plot_dense_i32(x, y, cfg: PlotConfig, row_begin: int = 0, row_end: int = 0) -> np.ndarray:
    """Dense int32 half-unit grid (PlotGrid's own type) via ap_plot_dense_i32: every window size,
    including LCS plots with w > 32767 whose scores exceed 16 bits."""
    xa, ya = _codes(x), _codes(y)
    rows, cols = window_grid_dims(xa.size, ya.size, cfg.window_w, cfg.step_h)
    re = rows if row_end == 0 else min(row_end, rows)
    out = np.empty((max(re - row_begin, 0), cols), dtype=np.int32)
    _raise(_native.lib().ap_plot_dense_i32(_ptr(xa), xa.size, _ptr(ya), ya.size,
                                           ctypes.byref(_cfg(cfg, row_begin, row_end)), _ptr(out)))
    return out


def scores_fit_u16(cfg: PlotConfig) -> bool:
    """Half-unit scores lie in [0, 2w]; only LCS plots with w > 32767 leave uint16."""
    return not (cfg.blowup_r == 1 and 2 * cfg.window_w > 65535)


def compute_plot(x: Sequence, y: Sequence, cfg: PlotConfig) -> PlotGrid:
    """runner.cpp:78-131 on the CUDA engine: validate first, then the dense grid (int32 half-units;
    transferred as uint16 whenever the scores fit, half the device-to-host bytes)."""
    cfg.validate(x.size(), y.size())
    rows, cols = window_grid_dims(x.size(), y.size(), cfg.window_w, cfg.step_h)
    if not scores_fit_u16(cfg):
        return PlotGrid(rows, cols, cfg.window_w, cfg.step_h, 0, 0, plot_dense_i32(x, y, cfg).reshape(-1))
    u16 = plot_dense_u16(x, y, cfg)
    return PlotGrid(rows, cols, cfg.window_w, cfg.step_h, 0, 0, u16.reshape(-1).astype(np.int32))


def plot_threshold_arrays(x, y, cfg: PlotConfig, t_half: int, cap: Optional[int] = None,
                          row_begin: int = 0, row_end: int = 0):
    """Fused threshold + row-major compaction: (rows, cols, halves) arrays.

    One comb of the plot: through ap_plot_threshold_into, whose callback allocates the arrays
    once the count is known (apply_threshold's exact-size result, scoring.cpp:30-39).  With an
    explicit ``cap`` the fixed-capacity entry ap_plot_threshold is used instead; a longer list
    raises ``EngineError`` (AP_CAPACITY)."""
    xa, ya = _codes(x), _codes(y)
    c = _cfg(cfg, row_begin, row_end)
    c.has_threshold = 1
    c.threshold_half = int(t_half)
    L = _native.lib()
    count = ctypes.c_uint64(0)
    if cap is not None:
        r = np.empty(cap, dtype=np.uint32)
        k = np.empty(cap, dtype=np.uint32)
        hv = np.empty(cap, dtype=np.uint16)
        _raise(L.ap_plot_threshold(_ptr(xa), xa.size, _ptr(ya), ya.size, ctypes.byref(c), ctypes.byref(count),
                                   _ptr(r), _ptr(k), _ptr(hv), cap))
        n = int(count.value)
        return r[:n], k[:n], hv[:n]
    held = {}

    def alloc(_user, n, pr, pc, ph):
        try:
            held["r"] = np.empty(max(int(n), 1), dtype=np.uint32)
            held["c"] = np.empty(max(int(n), 1), dtype=np.uint32)
            held["h"] = np.empty(max(int(n), 1), dtype=np.int32)
        except MemoryError:
            return 1
        pr[0] = held["r"].ctypes.data
        pc[0] = held["c"].ctypes.data
        ph[0] = held["h"].ctypes.data
        return 0

    cb = _native.ListAllocFn(alloc)
    _raise(L.ap_plot_threshold_into(_ptr(xa), xa.size, _ptr(ya), ya.size, ctypes.byref(c), cb, None,
                                    ctypes.byref(count)))
    n = int(count.value)
    return held["r"][:n], held["c"][:n], held["h"][:n]


def plot_threshold_cells(x, y, cfg: PlotConfig, t_half: int, row_begin: int = 0, row_end: int = 0) -> List[PlotCell]:
    """The same list through the array-of-structs entry point ap_plot_threshold_cells."""
    xa, ya = _codes(x), _codes(y)
    c = _cfg(cfg, row_begin, row_end)
    c.has_threshold = 1
    c.threshold_half = int(t_half)
    L = _native.lib()
    count = ctypes.c_uint64(0)
    cap = 1 << 12
    while True:
        buf = (_native.ApCell * max(cap, 1))()
        rc = L.ap_plot_threshold_cells(_ptr(xa), xa.size, _ptr(ya), ya.size, ctypes.byref(c), ctypes.byref(count),
                                       ctypes.cast(buf, ctypes.c_void_p), cap)
        if rc == _native.AP_CAPACITY:
            cap = int(count.value)
            continue
        _raise(rc)
        return [PlotCell(int(buf[i].row), int(buf[i].col), int(buf[i].half)) for i in range(int(count.value))]


def compute_plot_threshold(x: Sequence, y: Sequence, cfg: PlotConfig, t_half: Optional[int] = None) -> List[PlotCell]:
    """apply_threshold(compute_plot(x, y, cfg), t) fused on the GPU (no dense grid is materialised)."""
    t = cfg.threshold_half if t_half is None else t_half
    if t is None:
        raise ValueError("no threshold given")
    cfg.validate(x.size(), y.size())
    r, c, h = plot_threshold_arrays(x, y, cfg, t)
    return [PlotCell(int(a), int(b), int(v)) for a, b, v in zip(r, c, h)]


def device_count() -> int:
    return int(_native.lib().ap_device_count())
