#!/usr/bin/env python3
"""Benchmark of the alignment-plot hot path (BASELINE.json metric: window-pair cell updates/s).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--scaling strong|weak]
                  [--impl engine|reference]

A *step* is one pass of the hot path over one full plot of the workload: the
code-stream kernels plus the fused comb+extract kernel writing the dense
uint16 grid (C1/C2) or the thresholded row-major list (C3-C5; scan + placement
of every hit).  The default workload is BASELINE.json configs[3] = C4 (the
config its "1/2/4/8 B200" metric is quoted on: alignment-score plot, sigma=20,
m=n=262144, w=64, score >= 16), which fits one B200.

* ``value``  -- WPCU/s = rows*cols*w / t of the whole plot, inputs resident in HBM
  (ap_ctx_*_device), timed with CUDA events on the launching stream (max over
  ranks), L2 flushed (256 MiB write) between steps outside the timed events.
* ``e2e``    -- the same metric through the public host API (ap_plot_dense /
  ap_plot_threshold) with pinned host buffers: H2D of x, y and D2H of the plot
  or list inside the timed region.
* ``roofline`` -- the comb kernel's ALU instructions (its minimal count per comb
  cell, kernel_alu_ops_per_cell) per second against the measured ALU-pipe issue
  peak (profiles/int_peak_r01.json x the SM clock sampled during the run), so
  ``frac`` <= 1; ``vs_generic_recurrence`` keeps SURVEY.md §8d's basis (3 int32
  lane-ops per comb cell).  Comb cells = rows * (w*r) * (n*r).
* ``cpu_baseline`` -- the unmodified reference library (oracle/_ref, sea8 /
  sea16, all host cores) on a bounded, evenly spaced row sample; ``parity``
  compares the timed output with the reference on exactly those rows.

Multi-GPU (torchrun): grid rows shard over ranks in contiguous blocks with a w-1
x halo.  ``--scaling strong`` (C4, C5) splits the config's fixed plot;
``--scaling weak`` (C1-C3) grows x with the rank count.  No data-path collective:
thresholded configs all_gather one hit count per rank (NCCL).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_0909_2000_b200 import datagen  # noqa: E402
from paper_0909_2000_b200.sharding import plan_row_shards, shard_x  # noqa: E402

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
INT_PEAK = os.path.join(ROOT, "profiles", "int_peak_r01.json")
NCU_TRAFFIC = os.path.join(ROOT, "profiles", "ncu_traffic_r02.json")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---- clocks -------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # wait until the sampler is live so short timed regions are covered too
            t0 = time.perf_counter()
            while not self.lines and time.perf_counter() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.005)
        except Exception:
            self.proc = None
        self.start = len(self.lines)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            # a region shorter than the 50 ms period: take the first sample after it
            # (still at the load clocks, before the GPU idles down)
            t0 = time.perf_counter()
            while len(self.lines) <= self.start and time.perf_counter() - t0 < 0.2:
                time.sleep(0.002)
        self.lines = self.lines[self.start:]
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [v.strip() for v in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                mx = max(mx, float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---- workload -------------------------------------------------------------------------------
def default_scaling(name: str) -> str:
    """C4 / C5 are the fixed plots BASELINE.json shards over 1/2/4/8 GPUs (strong); the smaller
    configs grow x with the rank count (weak)."""
    return "strong" if name in ("C4", "C5") else "weak"


def workload(name: str, world: int, scaling: str):
    c = datagen.CONFIGS[name]
    x, y = datagen.make_inputs(name)
    if world > 1 and scaling == "weak":
        # weak scaling: x grows by world; each rank gets the base workload's row count
        extra = datagen.uniform(1000 + world, 7, (world - 1) * x.size, datagen.DNA if name != "C4" else datagen.PROTEIN)
        x = np.concatenate([x, extra])
    return c, x, y


# ALU-pipe instructions per comb cell of each kernel family (both strips of a packed u32 counted
# as two cells); the kernel's useful ALU work, the numerator of roofline.frac.
def kernel_alu_ops_per_cell(kernel: str):
    """Generic kernel per u32 (one cell of each of two strips): VIADDMNMX + LOP3 = 2 ALU ops; fp16
    keys move one row in four's LOP3 to two HADD2s on the FMA pipe (1.75); computed masks add
    LOP3 + IADD + LOP3 (5).  r = 2 kernel per u32 block of 2 x 2 blown cells x two strips:
    3 VIMNMX + VIADDMNMX + LOP3 = 5 ALU ops for 8 cells (the ($,$) swap is free; the other
    mismatch min runs on the FMA pipe).  Large-window kernel: 32-bit keys, one strip per
    register: VIADDMNMX + LOP3 per cell."""
    if kernel.startswith("comb2"):
        return 5.0 / 8.0, "r=2 kernel: 5 ALU ops per 8 blown cells"
    if kernel.startswith("combw"):
        if kernel.endswith(",packed>"):
            return 1.0, f"large-window kernel {kernel}: VIADDMNMX + LOP3 per two packed cells"
        if ",table" in kernel:
            return 2.0, f"large-window kernel {kernel}: VIADDMNMX + LOP3 per cell (32-bit keys)"
        return 3.0, f"large-window kernel {kernel}: 3 ALU ops per cell (32-bit keys, computed masks)"
    ops = 5.0 if ",computed," in kernel else (1.75 if kernel.endswith("fp16>") else 2.0)
    return ops / 2.0, f"generic kernel {kernel}: {ops:g} ALU ops per 2 cells"


def comb_cells(rows, c, n):
    return rows * (c.w * c.r) * (n * c.r)


def load_json(path):
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f)
    return None


# ---- reference CPU arm ------------------------------------------------------------------------
def reference_rows(c, x, y, budget_s: float, max_rows: int, on_block=None):
    """Time the unmodified reference (oracle/_ref compute_plot) on a bounded, evenly spaced row sample.

    on_block(row_begin, row_end, grid) is called after each block, outside the timed calls
    (bench.py's parity check).  Returns (rows_done, seconds, cores, sample_desc) or None."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as ol

    if not ol.ref_available():
        return None
    cores = os.cpu_count() or 1
    mode = ol.SEA8 if c.w <= 254 else ol.SEA16
    rows_total = (x.size - c.w) // c.h + 1
    blk = max(cores, 8)
    t0 = time.perf_counter()
    rc, g, err = ol.ref_plot_rows(x, y, c.w, c.h, c.r, 0, min(blk, rows_total), mode, cores)
    t_cal = time.perf_counter() - t0
    if rc:
        raise RuntimeError(f"reference failed: {err}")
    per_row = t_cal / min(blk, rows_total)
    nrows = int(min(max_rows, rows_total, max(blk, budget_s / max(per_row, 1e-9))))
    nblocks = max(1, nrows // blk)
    starts = np.linspace(0, rows_total - blk, nblocks).astype(int) if rows_total > blk else [0]
    done, dt = 0, 0.0
    for s_ in starts:
        s_ = int(s_)
        e = min(rows_total, s_ + blk)
        t0 = time.perf_counter()
        rc, g, err = ol.ref_plot_rows(x, y, c.w, c.h, c.r, s_, e, mode, cores)
        dt += time.perf_counter() - t0
        if rc:
            raise RuntimeError(f"reference failed: {err}")
        done += e - s_
        if on_block is not None:
            on_block(s_, e, g)
    desc = (f"{done} of {rows_total} grid rows ({len(starts)} evenly spaced blocks of {blk}), "
            f"reference compute_plot mode={'sea8' if mode == ol.SEA8 else 'sea16'}, workers={cores}")
    return done, dt, cores, desc


def run_reference(args, rank, world):
    # the same workload as the engine arm at this world size (weak scaling grows x), sampled by rows
    c, x, y = workload(args.config, world, args.scaling)
    rows_total, cols = (x.size - c.w) // c.h + 1, y.size - c.w + 1
    metric_unit = "window-pair cell updates/s"
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as ol
    if not ol.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libalignplot_ref.so not built"}))
        return
    t_all = 0.0
    rows_all = 0
    for _ in range(args.steps):
        done, dt, cores, desc = reference_rows(c, x, y, budget_s=args.ref_seconds / max(1, args.steps),
                                               max_rows=rows_total)
        t_all += dt
        rows_all += done
    value = rows_all * cols * c.w / t_all
    line = {
        "metric": "window-pair cell updates/s (m*n*w/s)", "value": value, "unit": metric_unit,
        "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * t_all / args.steps, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "u8", "data": "synthetic (paper_0909_2000_b200.datagen)",
        "config": dict(config_desc(c, x, y, world, args.config, args.scaling),
                       parallelism=f"reference CPU on rank 0 ({cores} host threads)"),
        "cpu_baseline": {"value": value, "unit": metric_unit, "cores": cores, "kind": "reference",
                         "sample": desc},
        "e2e": {"value": value, "unit": metric_unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_desc(c, x, y, world, name, scaling):
    rows, cols = (x.size - c.w) // c.h + 1, y.size - c.w + 1
    par = "1 GPU" if world == 1 else (f"row shards x{world} of the fixed plot (w-1 halo)" if scaling == "strong"
                                      else f"row shards x{world}, x grown x{world} (weak)")
    return {"workload": f"{name}: {c.description}", "m": int(x.size), "n": int(y.size), "w": c.w, "h": c.h,
            "r": c.r, "rows": rows, "cols": cols,
            "output": "dense uint16 half-units" if c.t_half is None else f"threshold half >= {c.t_half}, row-major list",
            "parallelism": par,
            "l2": "flushed between steps (256 MiB write, outside the timed events)"}


# ---- engine arm -------------------------------------------------------------------------------
def run_engine(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_0909_2000_b200 import _native
    from paper_0909_2000_b200 import alignplot as ap

    local_rank = local_rank % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    c, x, y = workload(args.config, world, args.scaling)
    shard = plan_row_shards(x.size, c.w, c.h, world)[rank]
    xs = shard_x(x, shard)
    n = y.size
    rows_local, cols = shard.rows, n - c.w + 1
    rows_global = (x.size - c.w) // c.h + 1
    L = _native.lib()
    ctx = ctypes.c_void_p()
    rc = L.ap_ctx_create(local_rank, ctypes.byref(ctx))
    if rc:
        raise RuntimeError(_native.last_error())
    cfgc = _native.ApConfig(window_w=c.w, step_h=c.h, blowup_r=c.r, has_threshold=0 if c.t_half is None else 1,
                            threshold_half=c.t_half or 0, n_devices=1, row_begin=0, row_end=0)
    d_x = torch.from_numpy(xs.copy()).to(dev)
    d_y = torch.from_numpy(y.copy()).to(dev)
    dense = c.t_half is None
    # a dedicated stream: handle 0 would mean "the context's own stream" to the C ABI
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    count = ctypes.c_uint64(0)
    lists = {}

    def alloc_list(cap):
        lists["cap"] = cap
        lists["r"] = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
        lists["c"] = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
        lists["h"] = torch.empty(max(cap, 1), dtype=torch.int16, device=dev)

    if dense:
        d_out = torch.empty(rows_local * cols, dtype=torch.int16, device=dev)
    else:
        alloc_list(1 << 16)

    def step(strict=True):
        if dense:
            rc = L.ap_ctx_plot_dense_device(ctx, d_x.data_ptr(), xs.size, d_y.data_ptr(), n, ctypes.byref(cfgc),
                                            d_out.data_ptr(), stream.cuda_stream)
        else:
            rc = L.ap_ctx_plot_threshold_device(ctx, d_x.data_ptr(), xs.size, d_y.data_ptr(), n,
                                                ctypes.byref(cfgc), ctypes.byref(count), lists["r"].data_ptr(),
                                                lists["c"].data_ptr(), lists["h"].data_ptr(), lists["cap"],
                                                stream.cuda_stream)
            if rc == _native.AP_CAPACITY and not strict:
                return
        if rc:
            raise RuntimeError(f"engine status {rc}: {_native.last_error()}")

    # the first call sizes the device list; every timed step then places the whole list
    step(strict=False)
    if not dense and count.value > lists["cap"]:
        alloc_list(int(count.value))
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kern_ms, launches, kernel = [], 0, ""
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        for i in range(args.steps):
            flush.zero_()
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
            evs[i][1].synchronize()   # so the comb-kernel events of this step can be read
            kern_ms.append(L.ap_ctx_last_kernel_ms(ctx))
            kernel = (L.ap_ctx_last_kernel(ctx) or b"").decode()
            launches += L.ap_ctx_last_launches(ctx)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    t_local = sum(step_ms) / 1000.0
    kern_local = sum(kern_ms) / len(kern_ms) / 1000.0
    red_dev = dev if (world == 1 or dist.get_backend() == "nccl") else torch.device("cpu")
    t = torch.tensor([t_local, kern_local], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max, kern_max = float(t[0]), float(t[1])
    hits_local = int(count.value) if not dense else 0
    # thresholded output: the one collective of the path, a gather of per-rank hit counts (the
    # exclusive prefix of it places each rank's row-major list in the global one)
    hits_all = [hits_local]
    if world > 1 and not dense:
        cnt_t = torch.tensor([hits_local], dtype=torch.int64, device=red_dev)
        gathered = [torch.zeros_like(cnt_t) for _ in range(world)]
        dist.all_gather(gathered, cnt_t)
        hits_all = [int(g_.item()) for g_ in gathered]
    # what the last timed step produced (parity below)
    if dense:
        last_out = d_out.cpu().numpy().view(np.uint16).reshape(rows_local, cols)
    else:
        k = hits_local
        last_list = (lists["r"][:k].cpu().numpy().view(np.uint32), lists["c"][:k].cpu().numpy().view(np.uint32),
                     lists["h"][:k].cpu().numpy().view(np.int16).astype(np.int32))

    # ---- end to end through the public host API (pinned host buffers) ----
    hx = torch.from_numpy(x.copy()).pin_memory()
    hy = torch.from_numpy(y.copy()).pin_memory()
    cfg_py = ap.PlotConfig(window_w=c.w, step_h=c.h, blowup_r=c.r, threshold_half=c.t_half, mode=ap.Mode.cuda)
    if dense:
        hout = torch.empty(rows_local * cols, dtype=torch.int16).pin_memory()
    else:
        cap_h = max(1, hits_local)
        hr = torch.empty(cap_h, dtype=torch.int32).pin_memory()
        hc = torch.empty(cap_h, dtype=torch.int32).pin_memory()
        hh = torch.empty(cap_h, dtype=torch.int16).pin_memory()
    # this rank's rows of the plot of (x, y): the host API uploads only their x bytes (+ halo)
    apc = ap._cfg(cfg_py, shard.row_begin, shard.row_end)

    def e2e_step():
        if dense:
            rc = L.ap_plot_dense(hx.data_ptr(), x.size, hy.data_ptr(), n, ctypes.byref(apc), hout.data_ptr())
        else:
            rc = L.ap_plot_threshold(hx.data_ptr(), x.size, hy.data_ptr(), n, ctypes.byref(apc), ctypes.byref(count),
                                     hr.data_ptr(), hc.data_ptr(), hh.data_ptr(), cap_h)
        if rc:
            raise RuntimeError(f"engine status {rc}: {_native.last_error()}")

    torch.cuda.set_device(local_rank)
    e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    t_e2e_local = time.perf_counter() - t0
    te = torch.tensor([t_e2e_local], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    t_e2e = float(te[0])
    d2h = rows_local * cols * 2 if dense else hits_local * 10 + 8
    h2d = (shard.x_end - shard.x_begin) + n
    # the same through ap_plot_dense_u8 (lossless bytes for w <= 127): half the D2H
    e2e_u8 = None
    if dense and c.w <= 127:
        hout8 = torch.empty(rows_local * cols, dtype=torch.uint8).pin_memory()

        def e2e_u8_step():
            rc = L.ap_plot_dense_u8(hx.data_ptr(), x.size, hy.data_ptr(), n, ctypes.byref(apc), hout8.data_ptr())
            if rc:
                raise RuntimeError(f"engine status {rc}: {_native.last_error()}")

        e2e_u8_step()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_u8_step()
        te8 = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(te8, op=dist.ReduceOp.MAX)
        e2e_u8 = {"value": rows_global * cols * c.w * args.steps / float(te8[0]), "unit": "window-pair cell updates/s",
                  "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(rows_local * cols),
                  "api": "ap_plot_dense_u8 (half-unit scores as bytes, lossless for w <= 127)"}

    if rank != 0:
        L.ap_ctx_destroy(ctx)
        return
    wpcu = rows_global * cols * c.w
    value = wpcu * args.steps / t_max
    clocks = clk.summary()
    cells_local = comb_cells(rows_local, c, n)
    int_peak = load_json(INT_PEAK) or {}
    peak_ops_clk = int_peak.get("lane_ops_per_clk_per_sm")
    sm_mhz = clocks["sm_mhz"] or 1965.0
    props = torch.cuda.get_device_properties(dev)
    roof = None
    if peak_ops_clk:
        peak = props.multi_processor_count * peak_ops_clk * sm_mhz * 1e6 / 1e12   # T lane-ops/s
        ops_cell, ops_what = kernel_alu_ops_per_cell(kernel)
        achieved = cells_local * ops_cell / kern_max / 1e12
        traffic = ((load_json(NCU_TRAFFIC) or {}).get(args.config) or {}).get("dram_bytes_per_launch")
        roof = {"bound": "int_alu", "achieved": achieved, "peak": peak, "unit": "T ALU lane-ops/s",
                "frac": achieved / peak, "traffic": traffic,
                "what": f"the comb kernel's own ALU instructions ({ops_what}) x comb cells / kernel time, against "
                        f"the measured ALU-pipe issue peak: {props.multi_processor_count} SMs x "
                        f"{peak_ops_clk:.1f} lane-ops/clk/SM (profiles/int_peak_r01.json) x {sm_mhz:.0f} MHz "
                        "(median SM clock during the timed region)",
                "kernel": kernel, "kernel_ms": kern_max * 1000.0, "comb_cells_per_s": cells_local / kern_max,
                # SURVEY §8d's fixed basis: the reference recurrence at 3 int32 lane-ops per comb cell.
                # Above 1 = the kernel does less ALU work per cell than that recurrence, not faster
                # than the hardware.
                "vs_generic_recurrence": cells_local * 3.0 / kern_max / 1e12 / peak}
    hbm_peak = (load_json(MEASURED_PEAKS) or {}).get("hbm_gbs")
    out_bytes = rows_local * cols * 2 if dense else hits_local * 10 + 8
    hbm = {"bound": "hbm", "achieved": out_bytes / kern_max / 1e9, "peak": hbm_peak, "unit": "GB/s",
           "frac": out_bytes / kern_max / 1e9 / hbm_peak if hbm_peak else None,
           "what": "plot output stream written by the comb kernel"}

    # ---- CPU baseline (the unmodified reference) and parity of the timed output on its rows ----
    cpu, parity = None, None
    if world == 1 and not args.no_cpu_baseline:
        par = {"rows": 0, "dense_mismatches": 0, "list_cells": 0, "list_mismatches": 0}
        dense_buf = None

        def check_block(rb, re, g):
            nonlocal dense_buf
            par["rows"] += re - rb
            if dense:
                par["dense_mismatches"] += int(np.count_nonzero(last_out[rb:re].astype(np.int32) != g))
                return
            # the timed list restricted to these rows vs apply_threshold of the reference rows
            lr, lc, lh = last_list
            i0, i1 = np.searchsorted(lr, rb), np.searchsorted(lr, re)
            er, ec = np.nonzero(g >= c.t_half)
            got = (lr[i0:i1].astype(np.int64) - rb, lc[i0:i1].astype(np.int64), lh[i0:i1])
            same = (got[0].size == er.size and np.array_equal(got[0], er) and np.array_equal(got[1], ec)
                    and np.array_equal(got[2], g[er, ec]))
            par["list_cells"] += int(er.size)
            par["list_mismatches"] += 0 if same else max(1, abs(int(got[0].size) - int(er.size)))
            # and the dense scores of the same rows (device API, row range)
            cb = _native.ApConfig(window_w=c.w, step_h=c.h, blowup_r=c.r, has_threshold=0, threshold_half=0,
                                  n_devices=1, row_begin=rb, row_end=re)
            if dense_buf is None or dense_buf.numel() < (re - rb) * cols:
                dense_buf = torch.empty((re - rb) * cols, dtype=torch.int16, device=dev)
            rc = L.ap_ctx_plot_dense_device(ctx, d_x.data_ptr(), xs.size, d_y.data_ptr(), n, ctypes.byref(cb),
                                            dense_buf.data_ptr(), stream.cuda_stream)
            if rc:
                raise RuntimeError(f"engine status {rc}: {_native.last_error()}")
            gd = dense_buf[:(re - rb) * cols].cpu().numpy().view(np.uint16).reshape(re - rb, cols)
            par["dense_mismatches"] += int(np.count_nonzero(gd.astype(np.int32) != g))

        res = reference_rows(c, x, y, budget_s=args.ref_seconds, max_rows=rows_global, on_block=check_block)
        if res:
            done, dt, cores, desc = res
            cpu = {"value": done * cols * c.w / dt, "unit": "window-pair cell updates/s", "cores": cores,
                   "kind": "reference", "sample": desc}
            parity = dict(par, against="oracle/_ref (unmodified reference compute_plot) on the cpu_baseline rows",
                          what="dense: the timed plot's rows; threshold: the timed list restricted to those rows "
                               "(+ the device API's dense scores of the same rows)")
    line = {
        "metric": "window-pair cell updates/s (m*n*w/s)", "value": value, "unit": "window-pair cell updates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * t_max / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "u16",
        "data": "synthetic (seeded, paper_0909_2000_b200.datagen)",
        "config": config_desc(c, x, y, world, args.config, args.scaling),
        "entries_per_s": rows_global * cols * args.steps / t_max,
        "comb_cells_per_s": comb_cells(rows_global, c, n) * args.steps / t_max,
        "roofline": roof, "roofline_hbm_output": hbm, "clocks": clocks,
        "e2e": {"value": wpcu * args.steps / t_e2e, "unit": "window-pair cell updates/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "api": "ap_plot_dense" if dense else "ap_plot_threshold (pinned host arrays sized by the count)"},
        "e2e_compact": e2e_u8,
        "gpu_launches": launches, "kernel": kernel, "cpu_baseline": cpu, "parity": parity,
    }
    if not dense:
        line["hits_rank0"] = hits_local
        line["hits_total"] = sum(hits_all)
        line["hits_per_rank"] = hits_all
    print(json.dumps(line), flush=True)
    L.ap_ctx_destroy(ctx)


def main():
    ap_ = argparse.ArgumentParser()
    ap_.add_argument("--gpus", type=int, default=1)
    ap_.add_argument("--steps", type=int, default=10)
    ap_.add_argument("--warmup", type=int, default=3)
    ap_.add_argument("--config", default="C4", choices=sorted(datagen.CONFIGS))
    ap_.add_argument("--scaling", default=None, choices=["strong", "weak"],
                     help="strong: shard the config's fixed plot over the ranks (default for C4, C5); "
                          "weak: grow x with the rank count (default for C1-C3)")
    ap_.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap_.add_argument("--ref-seconds", type=float, default=8.0, help="wall-clock budget of the CPU reference sample")
    ap_.add_argument("--no-cpu-baseline", action="store_true")
    ap_.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                     help="gloo: exercise the N>1 code path with several ranks on one GPU (timing not meaningful)")
    args = ap_.parse_args()
    if args.scaling is None:
        args.scaling = default_scaling(args.config)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.impl == "engine" and args.dist_backend == "nccl":
            # communicator set-up lines (rank, nRanks) on stderr, so a scaling run shows its ranks
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group("gloo")
    if world > 1:
        import torch.distributed as dist
        log(f"[bench] rank {rank} of {world}: process group backend {dist.get_backend()}, "
            f"world size {dist.get_world_size()}, local rank {local_rank}")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_engine(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
