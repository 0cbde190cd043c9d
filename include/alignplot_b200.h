/*
 * alignplot_b200.h — C ABI of the B200-native alignment-plot engine.
 *
 * This is the drop-in boundary for the reference path
 *   alignplot::compute_plot(const Sequence&, const Sequence&, const PlotConfig&)
 *       (/root/reference/proj/include/alignplot/runner.hpp:24, runner.cpp:78-131)
 *   alignplot::apply_threshold(const PlotGrid&, half_score_t)
 *       (scoring.hpp:42, scoring.cpp:30-39)
 *   alignplot::window_grid_dims(m, n, w, h)   (model.hpp:90-91, model.cpp:63-72)
 *   PlotConfig::validate(m, n)                (model.hpp:85, model.cpp:46-61)
 * Plain pointers and sizes only; no C++ or torch types cross it.  A C++ shim
 * with the reference's exact types and exceptions sits on top of it
 * (paper_0909_2000_b200/csrc/alignplot_shim.hpp); INTEGRATION.md shows the
 * bindings.
 *
 * Scores are half-units (score x 2, reference model.hpp:13-15).  In both modes
 * a window-pair score lies in [0, 2w]: the uint16 entry points hold every score
 * except LCS plots with w > 32767 (up to the sea16 bound w*r <= 65534), which
 * take the int32 entry points (ap_plot_dense_i32, ap_plot_threshold_into,
 * ap_plot_threshold_cells).
 * Output layout: row-major, out[row * cols + col] for grid row `row` (x-window
 * starting at row*h) and column `col` (y-window starting at col), exactly the
 * PlotGrid::values layout (model.hpp:95-114).
 *
 * Every entry point is reentrant (calls on one device serialise on its
 * context; a thresholded call's list lives in memory owned by the call until it
 * is copied out); errors are status codes, and the message of the calling
 * thread's last failure is returned by ap_last_error().  There is no CPU
 * fallback: without a usable CUDA device every compute call returns AP_NODEV.
 * Host output buffers may be pageable (large dense outputs then go through a
 * pinned bounce ring) or pinned (copied directly). 
 */
#ifndef ALIGNPLOT_B200_H
#define ALIGNPLOT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  AP_CONFIG / AP_EMPTY map to the reference's ConfigError /
 * EmptyPlotError (model.hpp:17-26); AP_INVALID to std::invalid_argument. */
enum {
  AP_OK = 0,
  AP_CONFIG = 1,    /* bad w/h/r, sentinel byte in input, window too large */
  AP_EMPTY = 2,     /* no window fits (w > min(m, n)) */
  AP_INVALID = 3,   /* bad pointer / row range / capacity arguments */
  AP_CUDA = 4,      /* a CUDA runtime call failed */
  AP_NODEV = 5,     /* no CUDA device (the engine never falls back to the CPU) */
  AP_CAPACITY = 6,  /* thresholded list longer than the caller's cap (count is still set) */
  AP_NOMEM = 7      /* device allocation failed */
};

/* Mirrors PlotConfig (model.hpp:70-86) plus the engine's sharding fields. */
typedef struct ap_config {
  uint64_t window_w;      /* PlotConfig::window_w */
  uint64_t step_h;        /* PlotConfig::step_h */
  uint32_t blowup_r;      /* PlotConfig::blowup_r: 1 = LCS, 2 = alignment score */
  int32_t has_threshold;  /* PlotConfig::threshold_half.has_value() */
  int32_t threshold_half; /* keep cells with half >= threshold_half (scoring.cpp:36) */
  int32_t n_devices;      /* GPUs to shard grid rows over (0 or 1 = current device only) */
  uint64_t row_begin;     /* first grid row to compute (resumable / sharded runs) */
  uint64_t row_end;       /* one past the last grid row; 0 = all rows */
} ap_config;

/* window_grid_dims (model.cpp:63-72): rows = (m-w)/h + 1, cols = n-w+1. */
int ap_grid_dims(size_t m, size_t n, size_t w, size_t h, size_t* rows, size_t* cols);

/* PlotConfig::validate (model.cpp:46-61) with the sea16 lane bound: blown windows
 * w*r <= AP_MAX_BLOWN_WINDOW (model.cpp:57-59).  Windows up to AP_PACKED_WINDOW run on
 * the packed 16-bit-key kernels; larger ones on the large-window path (32-bit keys,
 * one CTA per strip). */
#define AP_MAX_BLOWN_WINDOW 65534
#define AP_PACKED_WINDOW 1024
int ap_validate(size_t m, size_t n, const ap_config* cfg);

/* Dense plot of grid rows [row_begin, row_end): out_half receives
 * (row_end-row_begin) * cols uint16 half-unit scores, row-major (AP_CONFIG for
 * LCS plots with w > 32767).  Replaces compute_plot (runner.cpp:78-131). */
int ap_plot_dense(const uint8_t* x, size_t m, const uint8_t* y, size_t n, const ap_config* cfg,
                  uint16_t* out_half);

/* Thresholded plot: the cells with half >= cfg->threshold_half, in row-major
 * order (apply_threshold, scoring.cpp:30-39), as three parallel arrays.
 * *count receives the total number of such cells (64-bit exact); if it exceeds
 * cap only the first cap are written and AP_CAPACITY is returned (cap = 0 is a
 * count-only query).  Rows are grid rows (global, i.e. counted from 0 even when
 * row_begin > 0).  uint16 scores: AP_CONFIG for LCS plots with w > 32767. */
int ap_plot_threshold(const uint8_t* x, size_t m, const uint8_t* y, size_t n, const ap_config* cfg,
                      uint64_t* count, uint32_t* rows, uint32_t* cols, uint16_t* halves,
                      size_t cap);

/* Single-pass form of ap_plot_threshold for callers that cannot size the list in
 * advance (apply_threshold returns a vector of exactly the passing cells,
 * scoring.cpp:30-39): the plot is combed once; when the total is known the
 * engine calls alloc(user, count, &rows, &cols, &halves) exactly once (also for
 * count 0) to get host arrays of at least `count` entries, then writes the
 * row-major list into them (int32 scores: every window size).  A nonzero return
 * from alloc aborts with AP_INVALID. */
typedef int (*ap_list_alloc_fn)(void* user, uint64_t count, uint32_t** rows, uint32_t** cols,
                                int32_t** halves);
int ap_plot_threshold_into(const uint8_t* x, size_t m, const uint8_t* y, size_t n, const ap_config* cfg,
                           ap_list_alloc_fn alloc, void* user, uint64_t* count);

/* One thresholded cell (PlotCell, scoring.hpp:33-42) for the array-of-structs
 * form below. */
typedef struct ap_cell {
  uint32_t row;   /* grid row (global) */
  uint32_t col;   /* grid column */
  int32_t half;   /* half-unit score */
} ap_cell;

/* As ap_plot_threshold, filling ap_cell records -- the PlotCell list
 * apply_threshold returns (scoring.cpp:30-39) -- instead of parallel arrays;
 * same count / cap / AP_CAPACITY contract. */
int ap_plot_threshold_cells(const uint8_t* x, size_t m, const uint8_t* y, size_t n, const ap_config* cfg,
                            uint64_t* count, ap_cell* cells, size_t cap);

/* As ap_plot_dense with the half-unit scores stored as bytes (lossless for
 * w <= 127, where scores lie in [0, 2w]; AP_CONFIG otherwise): half the
 * device-to-host bytes of the uint16 layout. */
int ap_plot_dense_u8(const uint8_t* x, size_t m, const uint8_t* y, size_t n, const ap_config* cfg,
                     uint8_t* out_half);

/* As ap_plot_dense with int32 half-units -- PlotGrid::values' own type (model.hpp:95-114).
 * Every config: the uint16 entry points return AP_CONFIG for LCS plots with w > 32767,
 * whose scores (up to 2w half-units) exceed 16 bits. */
int ap_plot_dense_i32(const uint8_t* x, size_t m, const uint8_t* y, size_t n, const ap_config* cfg,
                      int32_t* out_half);

/* Dense 8-bit PGM raster of rows [row_begin, row_end), the pixels of
 * write_pgm (io.cpp:136-153) quantised inside the comb kernel:
 * pixel = (255 * clamp(half, 0, 2w) + w) / (2w), and, when has_threshold,
 * 0 for cells below threshold_half.  Header formatting stays on the host. */
int ap_plot_pgm(const uint8_t* x, size_t m, const uint8_t* y, size_t n, const ap_config* cfg,
                uint8_t* pixels);

/* Message for the calling thread's last non-OK status. */
const char* ap_last_error(void);

/* Number of CUDA devices the engine can use (0 when none). */
int ap_device_count(void);

/* ---- device-resident API (inputs/outputs already in HBM) --------------- */
typedef struct ap_ctx ap_ctx;

/* One context per device; holds the stream, scratch buffers and events. */
int ap_ctx_create(int device, ap_ctx** out);
int ap_ctx_destroy(ap_ctx* ctx);

/* As ap_plot_dense, but x/y/out are device pointers on ctx's device and the
 * work runs on the given stream (0 = the context's own); the output is
 * complete when the call returns.  The launch plan depends on y's alphabet
 * size: the first call with a given (w, r, output) learns it with a stream
 * synchronisation before the comb kernel; later calls plan for the previous
 * size without waiting and have the kernel verify it on the device (the plot
 * re-runs if y has more codes).  Sentinel bytes are not checked (the host API
 * checks them). */
int ap_ctx_plot_dense_device(ap_ctx* ctx, const uint8_t* d_x, size_t m, const uint8_t* d_y,
                             size_t n, const ap_config* cfg, uint16_t* d_out, void* stream);

/* As ap_plot_dense_u8 on device pointers (stream semantics of ap_ctx_plot_dense_device). */
int ap_ctx_plot_dense_u8_device(ap_ctx* ctx, const uint8_t* d_x, size_t m, const uint8_t* d_y, size_t n,
                                const ap_config* cfg, uint8_t* d_out, void* stream);

/* As ap_plot_dense_i32 on device pointers (stream semantics of ap_ctx_plot_dense_device). */
int ap_ctx_plot_dense_i32_device(ap_ctx* ctx, const uint8_t* d_x, size_t m, const uint8_t* d_y, size_t n,
                                 const ap_config* cfg, int32_t* d_out, void* stream);

/* As ap_plot_pgm on device pointers (stream semantics of ap_ctx_plot_dense_device). */
int ap_ctx_plot_pgm_device(ap_ctx* ctx, const uint8_t* d_x, size_t m, const uint8_t* d_y, size_t n,
                           const ap_config* cfg, uint8_t* d_pixels, void* stream);

/* Thresholded plot into device arrays of capacity cap; *count (host) gets the
 * total.  Synchronises ctx's stream. */
int ap_ctx_plot_threshold_device(ap_ctx* ctx, const uint8_t* d_x, size_t m, const uint8_t* d_y,
                                 size_t n, const ap_config* cfg, uint64_t* count,
                                 uint32_t* d_rows, uint32_t* d_cols, uint16_t* d_halves,
                                 size_t cap, void* stream);

/* Duration in ms of the comb kernel(s) of the last call on ctx, measured with
 * CUDA events on the launching stream (roofline accounting in bench.py). */
float ap_ctx_last_kernel_ms(ap_ctx* ctx);

/* Number of kernel launches the last call on ctx enqueued. */
int ap_ctx_last_launches(ap_ctx* ctx);

/* The comb kernel the last call on ctx chose, e.g. "comb2<10,10,2,fp16>" or
 * "comb<4,32,2,table,fp16>" (lanes per strip pair, rows per lane, bands; mask
 * source; key encoding); "" before the first call.  Valid until the next call. */
const char* ap_ctx_last_kernel(ap_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* ALIGNPLOT_B200_H */
