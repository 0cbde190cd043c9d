"""Command-line front end — the reference CLI (tools/alignplot.cpp:45-147) on the CUDA engine.

  python -m paper_0909_2000_b200 --x x.fa --y y.fa [--window 100] [--step 5] [--lcs-only]
         [--threshold T] [--format tsv|pgm|dots] [--dense] [--output PATH] [--record NAME ...]
         [--bench --modes dp,sea8]

Same flags, defaults and output bytes as the reference.  Every --mode runs on the
GPU (the reference's engine names are aliases of the CUDA engine: its engines agree bit
for bit, acceptance.cpp:34-73; --bench reports the aliasing); thresholded TSV/dots come from
the fused threshold+compact kernel and PGM pixels from the fused quantiser, so no
dense grid is materialised for them.
"""
from __future__ import annotations

import argparse
import io
import json
import math
import os
import sys
import time
from typing import List

import numpy as np

from . import alignplot as ap
from . import writers
from .fasta import ParseError, read_fasta, select_record, to_sequence


def _llround(v: float) -> int:
    return int(math.floor(abs(v) + 0.5)) * (1 if v >= 0 else -1)


def benchmark(x: ap.Sequence, y: ap.Sequence, cfg: ap.PlotConfig, modes: List[ap.Mode]) -> dict:
    """The shape of io.cpp:192-233 (time each requested mode; Mcups normalised to the DP cost
    rows*cols*(w*r)^2), on this engine.

    The reference races different engines and insists their grids agree.  Here every mode is
    served by the one CUDA engine -- dp / blcs / sea_scalar / sea16 / sea8 are aliases of
    ``cuda`` (each entry says so in ``engine``) -- so that check cannot compare engines; what
    it checks instead is run-to-run determinism of the engine (bitwise-identical grids), and
    the report says which it was.  Cross-engine agreement with the reference is the job of the
    parity tests (tests/test_gpu_parity.py against oracle/_ref)."""
    if not modes:
        raise ap.ConfigError("benchmark needs at least one mode")
    rep = {"rows": 0, "cols": 0, "window": cfg.window_w, "step": cfg.step_h, "blowup": cfg.blowup_r,
           "workers": cfg.workers, "results": [],
           "agreement_check": "run-to-run determinism of the CUDA engine (every mode is an alias of cuda)"}
    reference = None
    for m in modes:
        c = ap.PlotConfig(**{**cfg.__dict__, "mode": m})
        t0 = time.perf_counter()
        grid = ap.compute_plot(x, y, c)
        secs = max(time.perf_counter() - t0, 1e-9)
        if reference is None:
            reference = grid
            rep["rows"], rep["cols"] = grid.rows, grid.cols
        elif grid != reference:
            raise RuntimeError(f"benchmark: run for mode {m.name} is not bitwise identical to the first run")
        wr = float(cfg.window_w * cfg.blowup_r)
        cells = float(rep["rows"]) * float(rep["cols"]) * wr * wr
        first = rep["results"][0]["seconds"] if rep["results"] else secs
        rep["results"].append({"mode": m.name, "engine": "cuda", "seconds": secs, "cell_updates_per_sec": cells / secs,
                               "speedup_vs_first": first / secs})
    return rep


def bench_text(rep: dict) -> str:
    """BenchReport::to_text layout (io.cpp:155-174), plus the engine each mode ran on."""
    out = [f"plot {rep['rows']} x {rep['cols']} windows, w={rep['window']}, h={rep['step']}, "
           f"r={rep['blowup']}, workers={rep['workers']}",
           f"{'mode':<12} {'seconds':>10} {'Mcups':>12} {'speedup':>9}  engine"]
    for e in rep["results"]:
        out.append(f"{e['mode']:<12} {e['seconds']:10.3f} {e['cell_updates_per_sec'] / 1e6:12.1f} "
                   f"{e['speedup_vs_first']:8.2f}x  {e['engine']}")
    out.append("every mode runs on the CUDA engine (the reference's engine names are aliases); "
               "agreement = run-to-run determinism")
    return "\n".join(out) + "\n"


def run(argv=None) -> int:
    p = argparse.ArgumentParser(prog="alignplot",
                                description="Alignment plots: window-vs-window LCS/alignment scores of two sequences")
    p.add_argument("--x", required=True, help="FASTA file for the vertical sequence")
    p.add_argument("--y", required=True, help="FASTA file for the horizontal sequence")
    p.add_argument("--window", type=int, default=100)
    p.add_argument("--step", type=int, default=5)
    p.add_argument("--mode", default="sea8")
    p.add_argument("--threshold", type=float, default=None)
    p.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    p.add_argument("--devices", type=int, default=1, help="GPUs to shard rows over (engine extra)")
    p.add_argument("--output", default="-")
    p.add_argument("--format", default="tsv", choices=["tsv", "pgm", "dots"])
    p.add_argument("--lcs-only", action="store_true")
    p.add_argument("--record", action="append", default=[])
    p.add_argument("--bench", action="store_true")
    p.add_argument("--modes", default="dp,sea8")
    p.add_argument("--dense", action="store_true")
    a = p.parse_args(argv)

    mode = ap.mode_from_name(a.mode)
    if mode is None:
        raise ap.ConfigError(f"unknown mode '{a.mode}'")
    if len(a.record) > 2:
        raise ap.ConfigError("--record given more than twice")
    xr = yr = a.record[0] if len(a.record) == 1 else ""
    if len(a.record) == 2:
        xr, yr = a.record
    x = to_sequence(select_record(read_fasta(a.x), xr, a.x))
    y = to_sequence(select_record(read_fasta(a.y), yr, a.y))
    cfg = ap.PlotConfig(window_w=a.window, step_h=a.step, blowup_r=1 if a.lcs_only else 2, mode=mode,
                        workers=a.workers, n_devices=a.devices,
                        threshold_half=None if a.threshold is None else _llround(a.threshold * 2))

    sink = sys.stdout.buffer if a.output == "-" else open(a.output, "wb")
    try:
        if a.bench:
            modes = []
            for item in a.modes.split(","):
                if not item:
                    continue
                m = ap.mode_from_name(item)
                if m is None:
                    raise ap.ConfigError(f"unknown mode '{item}'")
                modes.append(m)
            if not modes:
                raise ap.ConfigError("no benchmark modes given")
            rep = benchmark(x, y, cfg, modes)
            sys.stdout.write(bench_text(rep))
            if a.output != "-":
                sink.write((json.dumps(rep, indent=2) + "\n").encode())
            return 0
        cfg.validate(x.size(), y.size())
        if a.format == "pgm":
            sink.write(writers.plot_pgm(x, y, cfg))
        elif cfg.threshold_half is not None and not (a.format == "tsv" and a.dense):
            rr, cc, hh = ap.plot_threshold_arrays(x, y, cfg, cfg.threshold_half)
            txt = io.StringIO()
            if a.format == "tsv":
                writers.write_tsv_cells(txt, rr, cc, hh, cfg.step_h)
            else:
                writers.write_dots_cells(txt, rr, cc, cfg.step_h)
            sink.write(txt.getvalue().encode())
        else:
            grid = ap.compute_plot(x, y, cfg)
            txt = io.StringIO()
            if a.format == "tsv":
                writers.write_tsv(txt, grid, cfg.threshold_half, a.dense)
            else:
                writers.write_dots(txt, grid, cfg.threshold_half)
            sink.write(txt.getvalue().encode())
        sink.flush()
    finally:
        if sink is not sys.stdout.buffer:
            sink.close()
    return 0


def main() -> None:
    try:
        sys.exit(run())
    except (ap.ConfigError, ParseError, ValueError, RuntimeError, OSError) as e:
        sys.stderr.write(f"alignplot: {e}\n")
        sys.exit(1)


if __name__ == "__main__":
    main()
