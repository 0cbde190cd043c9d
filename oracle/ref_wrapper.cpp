// ref_wrapper.cpp — extern "C" shim over the UNMODIFIED reference library.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file
// together with the reference's own sources, where they lie under
// /root/reference/proj/src, into oracle/_ref/libalignplot_ref.so (git-ignored,
// travels to the GPU box).  No reference source is copied into this repo.
// Used by tests/ (parity cross-check), tests/golden/make_golden.py (fixture
// generation) and bench.py --impl reference / cpu_baseline (the reference CPU
// arm).
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "alignplot/lane_kernel.hpp"
#include "alignplot/model.hpp"
#include "alignplot/runner.hpp"
#include "alignplot/scoring.hpp"
#include "alignplot/seaweed_scalar.hpp"

using namespace alignplot;

namespace {
void set_err(char* err, size_t len, const char* what) {
  if (err && len) { std::strncpy(err, what, len - 1); err[len - 1] = 0; }
}
}  // namespace

extern "C" {

// compute_plot (runner.hpp:24) on Sequences built from the raw bytes.
// mode follows the reference Mode enum (model.hpp:65): 0 dp, 1 blcs,
// 2 sea_scalar, 3 sea16, 4 sea8.  Returns 0 ok, 1 ConfigError, 2
// EmptyPlotError, 3 std::invalid_argument, 4 other; out gets rows*cols int32.
int ref_compute_plot(const uint8_t* x, size_t m, const uint8_t* y, size_t n, size_t w, size_t h,
                     unsigned r, int mode, unsigned workers, int32_t* out, size_t out_cap,
                     size_t* rows, size_t* cols, char* err, size_t errlen) {
  try {
    Sequence sx("x", std::vector<uint8_t>(x, x + m));
    Sequence sy("y", std::vector<uint8_t>(y, y + n));
    PlotConfig cfg;
    cfg.window_w = w;
    cfg.step_h = h;
    cfg.blowup_r = r;
    cfg.mode = static_cast<Mode>(mode);
    cfg.workers = workers;
    PlotGrid g = compute_plot(sx, sy, cfg);
    *rows = g.rows;
    *cols = g.cols;
    if (g.values.size() > out_cap) { set_err(err, errlen, "output capacity"); return 4; }
    std::memcpy(out, g.values.data(), g.values.size() * sizeof(int32_t));
    return 0;
  } catch (const EmptyPlotError& e) { set_err(err, errlen, e.what()); return 2; }
  catch (const ConfigError& e) { set_err(err, errlen, e.what()); return 1; }
  catch (const std::invalid_argument& e) { set_err(err, errlen, e.what()); return 3; }
  catch (const std::exception& e) { set_err(err, errlen, e.what()); return 4; }
}

// comb_strip_lanes (lane_kernel.hpp:132-134) → to_bottom_events →
// window_llcs_from_events, i.e. the sea8/sea16 row pipeline of runner.cpp:49-56
// on one already-blown strip.  out gets (N - w*r)/r + 1 LLCS values.
int ref_lane_window_llcs(const uint8_t* xw, size_t W, const uint8_t* y, size_t N, size_t w,
                         unsigned r, unsigned v, uint64_t* out, char* err, size_t errlen) {
  try {
    RestrictedHSMEvents ev = comb_strip_lanes({xw, W}, {y, N}, w, r, v);
    auto ll = window_llcs_from_events(to_bottom_events(ev), ev.window_cols, ev.stride);
    for (size_t k = 0; k < ll.size(); ++k) out[k] = ll[k];
    return 0;
  } catch (const ConfigError& e) { set_err(err, errlen, e.what()); return 1; }
  catch (const std::invalid_argument& e) { set_err(err, errlen, e.what()); return 3; }
  catch (const std::exception& e) { set_err(err, errlen, e.what()); return 4; }
}

// comb_strip (seaweed_scalar.hpp:46) bottom-event starts, one per column.
int ref_comb_strip(const uint8_t* xw, size_t W, const uint8_t* y, size_t N, int32_t* starts) {
  try {
    CombResult res = comb_strip({xw, W}, {y, N});
    for (size_t j = 0; j < N; ++j) starts[j] = res.events[j].start_col;
    return 0;
  } catch (...) { return 4; }
}

}  // extern "C"
