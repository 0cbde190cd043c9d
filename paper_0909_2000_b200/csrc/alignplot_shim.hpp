// alignplot_shim.hpp — C++ drop-in for the reference library's hot-path API.
//
// Same namespace, names, types, argument meaning and exceptions as the
// reference headers under /root/reference/proj/include/alignplot/:
//   model.hpp    half_score_t, ConfigError, EmptyPlotError, kSentinelCode,
//                Sequence, ScoringScheme, Mode, mode_name/mode_from_name,
//                PlotConfig (+validate), window_grid_dims, PlotGrid
//   runner.hpp   StripTask, plan_strips, compute_plot
//   scoring.hpp  BlownSequence, blowup, unblow, recover_score, PlotCell,
//                apply_threshold
// so hot-path code written against the reference compiles unchanged and links
// libalignplot_b200.so instead.  The reference's io layer (FASTA, writers,
// benchmark; io.hpp) is not mirrored: plot output comes from the device as
// write_{tsv,dots,pgm}_gpu below (same bytes as io.cpp:102-153).  compute_plot runs on the CUDA engine through
// the C ABI (include/alignplot_b200.h) for every Mode: the reference proves all
// its engines produce the identical grid (tests/acceptance.cpp:34-73), while
// PlotConfig::validate keeps each mode's limits.  Extras: Mode::cuda,
// PlotConfig::n_devices, compute_plot_threshold (fused threshold + row-major
// compaction without a dense grid) and the GPU-fed writers.
#pragma once

#include <algorithm>
#include <charconv>
#include <cstdint>
#include <optional>
#include <ostream>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "../../include/alignplot_b200.h"

namespace alignplot {

using half_score_t = std::int32_t;

class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& what) : std::runtime_error(what) {}
};

class EmptyPlotError : public ConfigError {
 public:
  explicit EmptyPlotError(const std::string& what) : ConfigError(what) {}
};

// No CUDA device or a CUDA runtime failure: the engine has no CPU fallback.
class EngineError : public std::runtime_error {
 public:
  explicit EngineError(const std::string& what) : std::runtime_error(what) {}
};

inline constexpr std::uint8_t kSentinelCode = 0;

namespace detail {
inline void check(int rc) {
  if (rc == AP_OK) return;
  const std::string msg = ap_last_error();
  switch (rc) {
    case AP_EMPTY: throw EmptyPlotError(msg);
    case AP_CONFIG: throw ConfigError(msg);
    case AP_INVALID: throw std::invalid_argument(msg);
    default: throw EngineError("alignplot_b200 status " + std::to_string(rc) + ": " + msg);
  }
}
}  // namespace detail

struct Sequence {
  std::string name;
  std::vector<std::uint8_t> data;
  unsigned alphabet_size = 256;

  Sequence() = default;
  Sequence(std::string name_, std::vector<std::uint8_t> data_, unsigned alphabet_size_ = 256)
      : name(std::move(name_)), data(std::move(data_)), alphabet_size(alphabet_size_) {
    for (std::uint8_t c : data) {
      if (c == kSentinelCode)
        throw ConfigError("sequence '" + name + "' contains the reserved sentinel code 0");
      if (c >= alphabet_size)
        throw ConfigError("sequence '" + name + "' contains code " + std::to_string(c) +
                          " outside alphabet of size " + std::to_string(alphabet_size));
    }
  }
  static Sequence from_text(std::string name, std::string_view text) {
    return Sequence(std::move(name), std::vector<std::uint8_t>(text.begin(), text.end()));
  }
  std::size_t size() const { return data.size(); }
  std::span<const std::uint8_t> codes() const { return data; }
};

struct ScoringScheme {
  half_score_t match_half = 2;
  half_score_t mismatch_half = 0;
  half_score_t gap_half = -1;
  static ScoringScheme alignment() { return {2, 0, -1}; }
  static ScoringScheme lcs_only() { return {2, 0, 0}; }
};

enum class Mode { dp, blcs, sea_scalar, sea16, sea8, cuda };

inline const char* mode_name(Mode m) {
  switch (m) {
    case Mode::dp: return "dp";
    case Mode::blcs: return "blcs";
    case Mode::sea_scalar: return "sea_scalar";
    case Mode::sea16: return "sea16";
    case Mode::sea8: return "sea8";
    case Mode::cuda: return "cuda";
  }
  return "?";
}

inline std::optional<Mode> mode_from_name(std::string_view name) {
  for (Mode m : {Mode::dp, Mode::blcs, Mode::sea_scalar, Mode::sea16, Mode::sea8, Mode::cuda})
    if (name == mode_name(m)) return m;
  return std::nullopt;
}

inline std::pair<std::size_t, std::size_t> window_grid_dims(std::size_t m, std::size_t n, std::size_t w,
                                                            std::size_t h) {
  std::size_t rows = 0, cols = 0;
  detail::check(ap_grid_dims(m, n, w, h, &rows, &cols));
  return {rows, cols};
}

struct PlotConfig {
  std::size_t window_w = 100;
  std::size_t step_h = 5;
  unsigned blowup_r = 2;
  std::optional<half_score_t> threshold_half;
  Mode mode = Mode::sea8;
  unsigned workers = 1;
  int n_devices = 1;   // engine extra: GPUs to shard rows over

  ScoringScheme scoring() const {
    return blowup_r == 1 ? ScoringScheme::lcs_only() : ScoringScheme::alignment();
  }

  // model.cpp:46-61, same order and exception types, then the engine limit.
  void validate(std::size_t m, std::size_t n) const {
    if (window_w == 0) throw ConfigError("window size must be positive");
    if (step_h == 0) throw ConfigError("step size must be positive");
    if (workers == 0) throw ConfigError("worker count must be positive");
    if (blowup_r != 1 && blowup_r != 2)
      throw ConfigError("blowup factor must be 1 (LCS) or 2 (alignment score)");
    if (mode == Mode::sea8 && window_w + 1 > 255)
      throw ConfigError("sea8 mode supports windows up to 254 (got " + std::to_string(window_w) +
                        "): spans plus INF must fit 8-bit lanes");
    if (mode == Mode::sea16 && window_w * blowup_r + 1 > 65535)
      throw ConfigError("sea16 mode supports blown windows up to 65534");
    window_grid_dims(m, n, window_w, step_h);
    const ap_config c = to_c();
    detail::check(ap_validate(m, n, &c));
  }

  ap_config to_c(std::size_t row_begin = 0, std::size_t row_end = 0) const {
    ap_config c{};
    c.window_w = window_w;
    c.step_h = step_h;
    c.blowup_r = blowup_r;
    c.has_threshold = threshold_half.has_value();
    c.threshold_half = threshold_half.value_or(0);
    c.n_devices = n_devices;
    c.row_begin = row_begin;
    c.row_end = row_end;
    return c;
  }
};

struct PlotGrid {
  std::size_t rows = 0;
  std::size_t cols = 0;
  std::size_t window_w = 0;
  std::size_t step_h = 1;
  std::size_t row_origin = 0;
  std::size_t col_origin = 0;
  std::vector<half_score_t> values;

  PlotGrid() = default;
  PlotGrid(std::size_t rows_, std::size_t cols_, std::size_t w, std::size_t h)
      : rows(rows_), cols(cols_), window_w(w), step_h(h), values(rows_ * cols_, 0) {}

  half_score_t& at(std::size_t r, std::size_t c) { return values[r * cols + c]; }
  half_score_t at(std::size_t r, std::size_t c) const { return values[r * cols + c]; }
  std::size_t x_offset(std::size_t r) const { return row_origin + r * step_h; }
  std::size_t y_offset(std::size_t c) const { return col_origin + c; }
  bool operator==(const PlotGrid& other) const = default;
};

struct StripTask {
  std::size_t row_index;
  std::size_t x_offset;
  Mode engine;
  bool operator==(const StripTask&) const = default;
};

// runner.cpp:15-27
inline std::vector<StripTask> plan_strips(const PlotConfig& cfg, std::size_t m) {
  if (cfg.window_w > m)
    throw EmptyPlotError("no window of size " + std::to_string(cfg.window_w) +
                         " fits an input of length " + std::to_string(m));
  const std::size_t rows = (m - cfg.window_w) / cfg.step_h + 1;
  std::vector<StripTask> tasks;
  tasks.reserve(rows);
  for (std::size_t r = 0; r < rows; ++r) tasks.push_back({r, r * cfg.step_h, cfg.mode});
  return tasks;
}

// runner.cpp:78-131 on the CUDA engine: validate, then the dense plot (uint16
// half-units from the device, widened to the reference's int32 layout).
inline PlotGrid compute_plot(const Sequence& x, const Sequence& y, const PlotConfig& cfg) {
  cfg.validate(x.size(), y.size());
  const auto [rows, cols] = window_grid_dims(x.size(), y.size(), cfg.window_w, cfg.step_h);
  PlotGrid grid(rows, cols, cfg.window_w, cfg.step_h);
  PlotConfig dense = cfg;
  dense.threshold_half.reset();
  const ap_config c = dense.to_c();
  if (cfg.blowup_r == 1 && 2 * cfg.window_w > 65535) {   // scores beyond 16 bits: straight into the grid
    detail::check(ap_plot_dense_i32(x.data.data(), x.size(), y.data.data(), y.size(), &c, grid.values.data()));
    return grid;
  }
  std::vector<std::uint16_t> half(rows * cols);   // half the device-to-host bytes, widened here
  detail::check(ap_plot_dense(x.data.data(), x.size(), y.data.data(), y.size(), &c, half.data()));
  std::copy(half.begin(), half.end(), grid.values.begin());
  return grid;
}

struct BlownSequence {
  std::vector<std::uint8_t> data;
  std::size_t raw_len = 0;
  std::span<const std::uint8_t> codes() const { return data; }
  std::size_t size() const { return data.size(); }
};

// scoring.cpp:5-17
inline BlownSequence blowup(std::span<const std::uint8_t> raw) {
  BlownSequence out;
  out.raw_len = raw.size();
  out.data.reserve(2 * raw.size());
  for (std::uint8_t c : raw) {
    if (c == kSentinelCode) throw ConfigError("cannot blow up a sequence that contains the sentinel code");
    out.data.push_back(kSentinelCode);
    out.data.push_back(c);
  }
  return out;
}
inline BlownSequence blowup(const Sequence& s) { return blowup(s.codes()); }

inline std::vector<std::uint8_t> unblow(const BlownSequence& b) {
  std::vector<std::uint8_t> raw;
  raw.reserve(b.raw_len);
  for (std::size_t i = 1; i < b.data.size(); i += 2) raw.push_back(b.data[i]);
  return raw;
}

// scoring.cpp:26-28
inline half_score_t recover_score(std::size_t llcs_blown, std::size_t m, std::size_t n) {
  return static_cast<half_score_t>(2 * llcs_blown) - static_cast<half_score_t>(m + n);
}

struct PlotCell {
  std::size_t row;
  std::size_t col;
  half_score_t score_half;
  bool operator==(const PlotCell&) const = default;
};

// scoring.cpp:30-39 (host-side filter of an existing grid)
inline std::vector<PlotCell> apply_threshold(const PlotGrid& grid, half_score_t t_half) {
  std::vector<PlotCell> out;
  for (std::size_t r = 0; r < grid.rows; ++r)
    for (std::size_t c = 0; c < grid.cols; ++c)
      if (grid.at(r, c) >= t_half) out.push_back({r, c, grid.at(r, c)});
  return out;
}

// apply_threshold(compute_plot(x, y, cfg), t) fused on the GPU: no dense grid
// is materialised; cells come back in the same row-major order.  One comb: the
// engine sizes the result through ap_plot_threshold_into's callback.
inline std::vector<PlotCell> compute_plot_threshold(const Sequence& x, const Sequence& y, const PlotConfig& cfg,
                                                    half_score_t t_half) {
  cfg.validate(x.size(), y.size());
  PlotConfig tc = cfg;
  tc.threshold_half = t_half;
  const ap_config c = tc.to_c();
  struct Lists {
    std::vector<std::uint32_t> r, c;
    std::vector<std::int32_t> h;
  } lists;
  auto alloc = [](void* user, std::uint64_t count, std::uint32_t** rows, std::uint32_t** cols,
                  std::int32_t** halves) -> int {
    auto* l = static_cast<Lists*>(user);
    l->r.resize(count);
    l->c.resize(count);
    l->h.resize(count);
    *rows = l->r.data();
    *cols = l->c.data();
    *halves = l->h.data();
    return 0;
  };
  std::uint64_t count = 0;
  detail::check(ap_plot_threshold_into(x.data.data(), x.size(), y.data.data(), y.size(), &c, alloc, &lists, &count));
  std::vector<PlotCell> out(count);
  for (std::size_t k = 0; k < count; ++k)
    out[k] = {lists.r[k], lists.c[k], lists.h[k]};
  return out;
}

// ---- GPU-fed plot output ------------------------------------------------------
// The reference writes its three formats from a materialised PlotGrid (io.cpp:102-153).
// Here the device produces what each format needs -- the thresholded row-major list for
// sparse TSV / dot output, quantised pixels for PGM (ap_plot_pgm), dense row blocks
// otherwise -- and the host only formats bytes.  The bytes equal the reference writers'
// (tests/golden/cli, tests/cpp/test_shim.cpp).
namespace detail {
// "<a> <sep> <b> <sep> <half as decimal>" with the half-unit score printed as k.0 / k.5
inline char* put_half(char* p, half_score_t half) {
  if (half < 0) *p++ = '-';
  const std::uint64_t mag = half < 0 ? std::uint64_t(-std::int64_t(half)) : std::uint64_t(half);
  p = std::to_chars(p, p + 24, mag >> 1).ptr;
  *p++ = '.';
  *p++ = (mag & 1) ? '5' : '0';
  return p;
}

// A buffered sink: format into a local block, hand full blocks to the stream.
struct LineSink {
  std::ostream& out;
  std::vector<char> buf = std::vector<char>(size_t(1) << 20);
  std::size_t used = 0;
  explicit LineSink(std::ostream& o) : out(o) {}
  char* reserve(std::size_t n) {
    if (used + n > buf.size()) flush();
    return buf.data() + used;
  }
  void commit(char* end) { used = std::size_t(end - buf.data()); }
  void flush() {
    out.write(buf.data(), static_cast<std::streamsize>(used));
    used = 0;
  }
};

// (row offset, col offset[, score]) lines of the cells passing the threshold, from the list
template <typename Emit>
inline void for_list(const Sequence& x, const Sequence& y, const PlotConfig& cfg, half_score_t t, Emit emit) {
  for (const PlotCell& cell : compute_plot_threshold(x, y, cfg, t)) emit(cell.row, cell.col, cell.score_half);
}

// every cell, from dense row blocks of about 64 MiB (bounded host memory for any plot size)
template <typename Emit>
inline void for_dense(const Sequence& x, const Sequence& y, const PlotConfig& cfg, Emit emit) {
  const auto [rows, cols] = window_grid_dims(x.size(), y.size(), cfg.window_w, cfg.step_h);
  PlotConfig dc = cfg;
  dc.threshold_half.reset();
  const std::size_t block = std::max<std::size_t>(1, (std::size_t(32) << 20) / std::max<std::size_t>(cols, 1));
  std::vector<std::int32_t> half;
  for (std::size_t r0 = 0; r0 < rows; r0 += block) {
    const std::size_t r1 = std::min(rows, r0 + block);
    half.resize((r1 - r0) * cols);
    const ap_config c = dc.to_c(r0, r1);
    check(ap_plot_dense_i32(x.data.data(), x.size(), y.data.data(), y.size(), &c, half.data()));
    for (std::size_t r = r0; r < r1; ++r)
      for (std::size_t k = 0; k < cols; ++k) emit(r, k, half[(r - r0) * cols + k]);
  }
}
}  // namespace detail

// TSV of compute_plot(x, y, cfg): header line, then "x_offset\ty_offset\tscore" per cell;
// without `dense`, only cells passing cfg.threshold_half (io.cpp:102-119 semantics).
inline void write_tsv_gpu(std::ostream& out, const Sequence& x, const Sequence& y, const PlotConfig& cfg,
                          bool dense) {
  cfg.validate(x.size(), y.size());
  detail::LineSink sink(out);
  const std::string head = "# x_offset y_offset score\n";
  char* p = sink.reserve(head.size());
  sink.commit(std::copy(head.begin(), head.end(), p));
  auto emit = [&](std::size_t r, std::size_t c, half_score_t v) {
    char* q = sink.reserve(64);
    q = std::to_chars(q, q + 24, r * cfg.step_h).ptr;
    *q++ = '\t';
    q = std::to_chars(q, q + 24, c).ptr;
    *q++ = '\t';
    q = detail::put_half(q, v);
    *q++ = '\n';
    sink.commit(q);
  };
  if (!dense && cfg.threshold_half) detail::for_list(x, y, cfg, *cfg.threshold_half, emit);
  else detail::for_dense(x, y, cfg, emit);
  sink.flush();
  if (!out) throw std::runtime_error("write failure on TSV sink");
}

// "x_offset y_offset" per cell passing cfg.threshold_half (every cell without one; io.cpp:121-133).
inline void write_dots_gpu(std::ostream& out, const Sequence& x, const Sequence& y, const PlotConfig& cfg) {
  cfg.validate(x.size(), y.size());
  detail::LineSink sink(out);
  auto emit = [&](std::size_t r, std::size_t c, half_score_t) {
    char* q = sink.reserve(64);
    q = std::to_chars(q, q + 24, r * cfg.step_h).ptr;
    *q++ = ' ';
    q = std::to_chars(q, q + 24, c).ptr;
    *q++ = '\n';
    sink.commit(q);
  };
  if (cfg.threshold_half) detail::for_list(x, y, cfg, *cfg.threshold_half, emit);
  else detail::for_dense(x, y, cfg, emit);
  sink.flush();
  if (!out) throw std::runtime_error("write failure on dot sink");
}

// The PGM of compute_plot(x, y, cfg) without a dense grid on the host: pixels
// are quantised inside the comb kernel (ap_plot_pgm), cfg.threshold_half cuts.
inline void write_pgm_gpu(std::ostream& out, const Sequence& x, const Sequence& y, const PlotConfig& cfg) {
  cfg.validate(x.size(), y.size());
  const auto [rows, cols] = window_grid_dims(x.size(), y.size(), cfg.window_w, cfg.step_h);
  std::vector<unsigned char> pix(rows * cols);
  const ap_config c = cfg.to_c();
  detail::check(ap_plot_pgm(x.data.data(), x.size(), y.data.data(), y.size(), &c, pix.data()));
  out << "P5\n" << cols << ' ' << rows << "\n255\n";
  out.write(reinterpret_cast<const char*>(pix.data()), static_cast<std::streamsize>(pix.size()));
  if (!out) throw std::runtime_error("write failure on PGM sink");
}

}  // namespace alignplot
