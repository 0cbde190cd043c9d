/*
 * alignplot_oracle.c — CPU restatement of the reference alignment-plot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * engine in paper_0909_2000_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it; the product path never does
 * (the C-ABI library has no CPU fallback).
 *
 * Every function restates, in plain C, the reference algorithm it cites
 * (paths relative to /root/reference/proj).  The restatement is pinned by
 * tests/test_oracle.py against (a) the known-answer vectors of the reference
 * unit tests and (b) golden fixtures produced by the reference library itself
 * (oracle/_ref, built by oracle/Makefile; fixtures in tests/golden/ made by
 * oracle/golden_gen.cpp).
 *
 * Conventions (reference model.hpp:13-15): scores are half-units (score x 2)
 * in int32.  Return codes: 0 ok, 1 ConfigError, 2 EmptyPlotError,
 * 3 invalid_argument.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define OR_OK 0
#define OR_CONFIG 1
#define OR_EMPTY 2
#define OR_INVALID 3

/* window_grid_dims — model.cpp:63-72.  rows = (m-w)/h + 1, cols = n-w+1. */
int or_window_grid_dims(size_t m, size_t n, size_t w, size_t h, size_t* rows, size_t* cols) {
  if (w == 0 || h == 0) return OR_CONFIG;
  if (w > m || w > n) return OR_EMPTY;
  *rows = (m - w) / h + 1;
  *cols = n - w + 1;
  return OR_OK;
}

/* PlotConfig::validate — model.cpp:46-61.  mode: 3 = sea16, 4 = sea8 (the
 * reference Mode enum order, model.hpp:65); other modes carry no width limit. */
int or_validate(size_t m, size_t n, size_t w, size_t h, unsigned r, unsigned workers, int mode) {
  if (w == 0) return OR_CONFIG;
  if (h == 0) return OR_CONFIG;
  if (workers == 0) return OR_CONFIG;
  if (r != 1 && r != 2) return OR_CONFIG;
  if (mode == 4 && w + 1 > 255) return OR_CONFIG;
  if (mode == 3 && w * r + 1 > 65535) return OR_CONFIG;
  size_t rows, cols;
  return or_window_grid_dims(m, n, w, h, &rows, &cols);
}

/* blowup — scoring.cpp:5-17: out[2k] = 0 (sentinel), out[2k+1] = raw[k];
 * a raw 0 byte is a ConfigError. */
int or_blowup(const uint8_t* raw, size_t n, uint8_t* out) {
  for (size_t k = 0; k < n; ++k) {
    if (raw[k] == 0) return OR_CONFIG;
    out[2 * k] = 0;
    out[2 * k + 1] = raw[k];
  }
  return OR_OK;
}

/* recover_score — scoring.cpp:26-28: half = 2*llcs_blown - (m+n). */
int32_t or_recover_score(size_t llcs_blown, size_t m, size_t n) {
  return (int32_t)(2 * llcs_blown) - (int32_t)(m + n);
}

/* llcs_to_half — runner.cpp:31-35. */
static int32_t llcs_to_half(size_t llcs, size_t w, unsigned r) {
  return r == 1 ? (int32_t)(2 * llcs) : or_recover_score(llcs, w, w);
}

/* comb_strip — seaweed_scalar.cpp:11-49.  Row-major seaweed combing of the
 * strip xw (w rows) against y (n columns).  front[j] starts as j (top
 * seaweeds carry their start column); row i's left seaweed has id -(i+1).
 * At each cell the seaweeds exchange iff the characters match or the
 * left-entrant started right of the top-entrant (seaweed_scalar.cpp:26-32).
 * bottom_start[j] = start of the seaweed leaving the bottom at column j;
 * right_start[i] (optional) = start of the seaweed leaving row i on the right. */
void or_comb_strip(const uint8_t* xw, size_t w, const uint8_t* y, size_t n,
                   int32_t* bottom_start, int32_t* right_start) {
  for (size_t j = 0; j < n; ++j) bottom_start[j] = (int32_t)j;
  for (size_t i = 0; i < w; ++i) {
    int32_t runner = -(int32_t)i - 1;
    const uint8_t xc = xw[i];
    for (size_t j = 0; j < n; ++j) {
      const int32_t top = bottom_start[j];
      if (xc == y[j] || runner > top) {
        bottom_start[j] = runner;
        runner = top;
      }
    }
    if (right_start) right_start[i] = runner;
  }
}

/* llcs_query — seaweed_scalar.cpp:51-63, on the critical points of one strip:
 * bottom exits (start, end=j) and right exits (start, end=n+i).
 * A(i,j) = (j-i) - |{(s,e): s >= i, e < j}|. */
int or_llcs_query(const int32_t* bottom_start, size_t n, const int32_t* right_start, size_t w,
                  size_t i, size_t j, size_t* out) {
  if (i > j || j > n) return OR_INVALID;
  size_t dominated = 0;
  for (size_t e = 0; e < n; ++e)
    if (bottom_start[e] >= (int32_t)i && (int32_t)e < (int32_t)j) ++dominated;
  for (size_t r = 0; r < w; ++r)
    if (right_start[r] >= (int32_t)i && (int32_t)(n + r) < (int32_t)j) ++dominated;
  *out = (j - i) - dominated;
  return OR_OK;
}

/* Min-heap of int32 (the std::priority_queue<..., std::greater<>> of
 * seaweed_scalar.cpp:80). */
typedef struct { int32_t* a; size_t n; } heap_t;
static void heap_push(heap_t* h, int32_t v) {
  size_t i = h->n++;
  h->a[i] = v;
  while (i > 0) {
    size_t p = (i - 1) / 2;
    if (h->a[p] <= h->a[i]) break;
    int32_t t = h->a[p]; h->a[p] = h->a[i]; h->a[i] = t;
    i = p;
  }
}
static void heap_pop(heap_t* h) {
  h->a[0] = h->a[--h->n];
  size_t i = 0;
  for (;;) {
    size_t l = 2 * i + 1, r = l + 1, s = i;
    if (l < h->n && h->a[l] < h->a[s]) s = l;
    if (r < h->n && h->a[r] < h->a[s]) s = r;
    if (s == i) break;
    int32_t t = h->a[s]; h->a[s] = h->a[i]; h->a[i] = t;
    i = s;
  }
}

/* window_llcs_from_events — seaweed_scalar.cpp:65-99.  starts[j] is the
 * start column of the bottom event at end column j (the stream has exactly
 * one event per column, checked at :73-78 by construction here).  Entry k is
 * the LLCS of the window of window_cols columns starting at k*stride: push
 * each start, and at report column pop starts left of the window; the LLCS is
 * window_cols minus the heap size (:86-97).  out must hold
 * (n - window_cols)/stride + 1 entries. */
int or_window_llcs_from_events(const int32_t* starts, size_t n, size_t window_cols, size_t stride,
                               size_t* out) {
  if (stride == 0) return OR_INVALID;
  if (window_cols == 0 || window_cols > n) return OR_INVALID;
  heap_t h;
  h.a = (int32_t*)malloc(sizeof(int32_t) * (n + 1));
  h.n = 0;
  size_t window_start = 0, report_at = window_cols - 1, k = 0;
  for (size_t j = 0; j < n; ++j) {
    heap_push(&h, starts[j]);
    if (j == report_at) {
      while (h.n > 0 && h.a[0] < (int32_t)window_start) heap_pop(&h);
      out[k++] = window_cols - h.n;
      window_start += stride;
      report_at += stride;
    }
  }
  free(h.a);
  return OR_OK;
}

/* compute_row sea_scalar branch — runner.cpp:43-48: comb the (blown) strip,
 * extract window LLCS at stride r, convert to half-units. */
static void compute_row(const uint8_t* xw, size_t W, const uint8_t* y_eff, size_t N, size_t w,
                        unsigned r, int32_t* out, int32_t* scratch_start, size_t* scratch_llcs) {
  or_comb_strip(xw, W, y_eff, N, scratch_start, NULL);
  or_window_llcs_from_events(scratch_start, N, W, r, scratch_llcs);
  const size_t cols = (N - W) / r + 1;
  for (size_t k = 0; k < cols; ++k) out[k] = llcs_to_half(scratch_llcs[k], w, r);
}

typedef struct {
  const uint8_t* x; const uint8_t* y_eff; size_t N, w, h, cols; unsigned r;
  size_t row_begin, row_end, worker, stride; int32_t* out;
} job_t;

static void* run_rows(void* arg) {
  job_t* j = (job_t*)arg;
  const size_t W = j->w * j->r;
  uint8_t* xw = (uint8_t*)malloc(W);
  int32_t* st = (int32_t*)malloc(sizeof(int32_t) * j->N);
  size_t* ll = (size_t*)malloc(sizeof(size_t) * (j->cols + 1));
  for (size_t row = j->row_begin + j->worker; row < j->row_end; row += j->stride) {
    const uint8_t* raw = j->x + row * j->h;
    if (j->r == 2) or_blowup(raw, j->w, xw); else memcpy(xw, raw, j->w);
    compute_row(xw, W, j->y_eff, j->N, j->w, j->r,
                j->out + (row - j->row_begin) * j->cols, st, ll);
  }
  free(xw); free(st); free(ll);
  return NULL;
}

/* compute_plot (sea_scalar engine) — runner.cpp:78-131, restricted to grid
 * rows [row_begin, row_end) so large configs can be sampled.  Validation
 * order follows runner.cpp:81 (validate before any work); the y blowup is done
 * once (runner.cpp:90-93) and each x-window is blown per row (:104-107).
 * out holds (row_end-row_begin)*cols int32 half-units, row-major. */
int or_plot_rows(const uint8_t* x, size_t m, const uint8_t* y, size_t n, size_t w, size_t h,
                 unsigned r, size_t row_begin, size_t row_end, unsigned workers, int32_t* out) {
  int rc = or_validate(m, n, w, h, r, workers ? workers : 1, 0);
  if (rc) return rc;
  for (size_t k = 0; k < m; ++k) if (x[k] == 0) return OR_CONFIG;  /* Sequence ctor, model.cpp:11-13 */
  for (size_t k = 0; k < n; ++k) if (y[k] == 0) return OR_CONFIG;
  size_t rows, cols;
  or_window_grid_dims(m, n, w, h, &rows, &cols);
  if (row_end > rows) row_end = rows;
  if (row_begin >= row_end) return OR_OK;
  const size_t N = n * r;
  uint8_t* y_eff = (uint8_t*)malloc(N);
  if (r == 2) or_blowup(y, n, y_eff); else memcpy(y_eff, y, n);
  if (workers == 0) workers = 1;
  if (workers > row_end - row_begin) workers = (unsigned)(row_end - row_begin);
  job_t* jobs = (job_t*)calloc(workers, sizeof(job_t));
  pthread_t* th = (pthread_t*)calloc(workers, sizeof(pthread_t));
  for (unsigned t = 0; t < workers; ++t) {
    job_t jb = {x, y_eff, N, w, h, cols, r, row_begin, row_end, t, workers, out};
    jobs[t] = jb;
    if (workers > 1) pthread_create(&th[t], NULL, run_rows, &jobs[t]);
    else run_rows(&jobs[t]);
  }
  if (workers > 1) for (unsigned t = 0; t < workers; ++t) pthread_join(th[t], NULL);
  free(jobs); free(th); free(y_eff);
  return OR_OK;
}

/* apply_threshold — scoring.cpp:30-39: cells with half >= t in row-major
 * order.  Writes up to cap (row, col, half) triples; returns the total. */
size_t or_apply_threshold(const int32_t* grid, size_t rows, size_t cols, int32_t t,
                          uint64_t* out_row, uint64_t* out_col, int32_t* out_half, size_t cap) {
  size_t k = 0;
  for (size_t r = 0; r < rows; ++r)
    for (size_t c = 0; c < cols; ++c) {
      const int32_t v = grid[r * cols + c];
      if (v >= t) {
        if (k < cap) { out_row[k] = r; out_col[k] = c; out_half[k] = v; }
        ++k;
      }
    }
  return k;
}

/* Independent full-table DP LLCS — tests/test_util.hpp:28-39 (the reference
 * test suite's own ground truth, written independently of the library). */
size_t or_ref_llcs(const uint8_t* a, size_t m, const uint8_t* b, size_t n) {
  size_t* prev = (size_t*)calloc(n + 1, sizeof(size_t));
  size_t* cur = (size_t*)calloc(n + 1, sizeof(size_t));
  for (size_t i = 1; i <= m; ++i) {
    for (size_t j = 1; j <= n; ++j) {
      size_t up = prev[j], left = cur[j - 1];
      cur[j] = a[i - 1] == b[j - 1] ? prev[j - 1] + 1 : (up > left ? up : left);
    }
    size_t* t = prev; prev = cur; cur = t;
  }
  size_t res = prev[n];
  free(prev); free(cur);
  return res;
}

/* Global alignment score, match +1 / mismatch 0 / gap -0.5, in half-units —
 * tests/test_util.hpp:42-57. */
int32_t or_ref_align_score_half(const uint8_t* a, size_t m, const uint8_t* b, size_t n) {
  int32_t* prev = (int32_t*)malloc(sizeof(int32_t) * (n + 1));
  int32_t* cur = (int32_t*)malloc(sizeof(int32_t) * (n + 1));
  for (size_t j = 0; j <= n; ++j) prev[j] = -(int32_t)j;
  for (size_t i = 1; i <= m; ++i) {
    cur[0] = -(int32_t)i;
    for (size_t j = 1; j <= n; ++j) {
      int32_t diag = prev[j - 1] + (a[i - 1] == b[j - 1] ? 2 : 0);
      int32_t up = prev[j] - 1, left = cur[j - 1] - 1;
      int32_t best = diag > up ? diag : up;
      cur[j] = best > left ? best : left;
    }
    int32_t* t = prev; prev = cur; cur = t;
  }
  int32_t res = prev[n];
  free(prev); free(cur);
  return res;
}
