"""Output writers on the engine's results — byte-identical to the reference io.cpp.

* ``half_to_decimal``  io.cpp:102-109
* ``write_tsv``        io.cpp:111-123 (dense grid) and ``write_tsv_cells`` (from a
  thresholded row-major list straight off the GPU, no dense grid)
* ``write_dots``       io.cpp:125-134 and ``write_dots_cells``
* ``write_pgm``        io.cpp:136-153; ``plot_pgm`` gets the raster already
  quantised inside the comb kernel (ap_plot_pgm) and only adds the header.
"""
from __future__ import annotations

import ctypes
from typing import BinaryIO, Optional, TextIO

import numpy as np

from . import _native
from .alignplot import PlotConfig, PlotGrid, _cfg, _codes, _ptr, _raise, window_grid_dims


def half_to_decimal(half: int) -> str:
    a = -half if half < 0 else half
    return ("-" if half < 0 else "") + str(a // 2) + (".5" if a % 2 else ".0")


def _dec_array(v: np.ndarray) -> np.ndarray:
    v = v.astype(np.int64)
    a = np.abs(v)
    s = np.char.add(np.where(v < 0, "-", ""), (a // 2).astype(str))
    return np.char.add(s, np.where(a % 2 == 1, ".5", ".0"))


def write_tsv(out: TextIO, grid: PlotGrid, threshold_half: Optional[int] = None, dense: bool = False) -> None:
    out.write("# x_offset y_offset score\n")
    v = grid.values.reshape(grid.rows, grid.cols)
    keep = np.ones_like(v, dtype=bool) if (dense or threshold_half is None) else v >= threshold_half
    rr, cc = np.nonzero(keep)
    write_tsv_cells(out, rr, cc, v[rr, cc], grid.step_h, grid.row_origin, grid.col_origin, header=False)


def write_tsv_cells(out: TextIO, rows, cols, halves, step_h: int, row_origin: int = 0, col_origin: int = 0,
                    header: bool = True) -> None:
    """TSV lines for a row-major cell list (e.g. ap_plot_threshold's output)."""
    if header:
        out.write("# x_offset y_offset score\n")
    rows = np.asarray(rows, dtype=np.int64)
    if rows.size == 0:
        return
    xs = (row_origin + rows * step_h).astype(str)
    ys = (col_origin + np.asarray(cols, dtype=np.int64)).astype(str)
    lines = np.char.add(np.char.add(np.char.add(np.char.add(xs, "\t"), ys), "\t"), _dec_array(np.asarray(halves)))
    out.write("\n".join(lines.tolist()) + "\n")


def write_dots(out: TextIO, grid: PlotGrid, threshold_half: Optional[int] = None) -> None:
    v = grid.values.reshape(grid.rows, grid.cols)
    keep = np.ones_like(v, dtype=bool) if threshold_half is None else v >= threshold_half
    rr, cc = np.nonzero(keep)
    write_dots_cells(out, rr, cc, grid.step_h, grid.row_origin, grid.col_origin)


def write_dots_cells(out: TextIO, rows, cols, step_h: int, row_origin: int = 0, col_origin: int = 0) -> None:
    rows = np.asarray(rows, dtype=np.int64)
    if rows.size == 0:
        return
    xs = (row_origin + rows * step_h).astype(str)
    ys = (col_origin + np.asarray(cols, dtype=np.int64)).astype(str)
    out.write("\n".join(np.char.add(np.char.add(xs, " "), ys).tolist()) + "\n")


def pgm_pixels(grid: PlotGrid, threshold_half: Optional[int] = None) -> np.ndarray:
    """Host quantisation (io.cpp:136-153), for grids already on the host."""
    full = 2 * grid.window_w
    v = grid.values.reshape(grid.rows, grid.cols).astype(np.int64)
    if threshold_half is not None:
        v = np.where(v < threshold_half, 0, v)
    h = np.clip(v, 0, full)
    return ((255 * h + full // 2) // full).astype(np.uint8)


def pgm_header(rows: int, cols: int) -> bytes:
    return f"P5\n{cols} {rows}\n255\n".encode()


def write_pgm(out: BinaryIO, grid: PlotGrid, threshold_half: Optional[int] = None) -> None:
    out.write(pgm_header(grid.rows, grid.cols))
    out.write(pgm_pixels(grid, threshold_half).tobytes())


def plot_pgm(x, y, cfg: PlotConfig) -> bytes:
    """The whole PGM file, pixels quantised on the GPU (ap_plot_pgm); cfg.threshold_half cuts cells to 0."""
    xa, ya = _codes(x), _codes(y)
    cfg.validate(xa.size, ya.size)
    rows, cols = window_grid_dims(xa.size, ya.size, cfg.window_w, cfg.step_h)
    pix = np.empty((rows, cols), dtype=np.uint8)
    _raise(_native.lib().ap_plot_pgm(_ptr(xa), xa.size, _ptr(ya), ya.size, ctypes.byref(_cfg(cfg)), _ptr(pix)))
    return pgm_header(rows, cols) + pix.tobytes()
