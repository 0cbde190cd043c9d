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
// so code written against the reference compiles unchanged and links
// libalignplot_b200.so instead.  compute_plot runs on the CUDA engine through
// the C ABI (include/alignplot_b200.h) for every Mode: the reference proves all
// its engines produce the identical grid (tests/acceptance.cpp:34-73), while
// PlotConfig::validate keeps each mode's limits.  Extras: Mode::cuda,
// PlotConfig::n_devices, and compute_plot_threshold (fused threshold +
// row-major compaction without a dense grid).
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <fstream>
#include <istream>
#include <optional>
#include <ostream>
#include <sstream>
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

class ParseError : public std::runtime_error {
 public:
  explicit ParseError(const std::string& what) : std::runtime_error(what) {}
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
// A double as the reference's JSON writer prints it: the shortest digit string
// that round-trips, in fixed notation (with a trailing ".0" when integral) for
// values in [1e-4, 1e15), scientific ("1.5e+20", "1e-05") outside.
inline std::string json_double(double v) {
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  char buf[64];
  int p = 0;
  for (; p < 17; ++p) {   // shortest round-trip mantissa
    std::snprintf(buf, sizeof buf, "%.*e", p, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  std::snprintf(buf, sizeof buf, "%.*e", p, v);
  std::string m(buf);
  const bool neg = m[0] == '-';
  if (neg) m.erase(0, 1);
  const std::size_t epos = m.find('e');
  const int e10 = std::atoi(m.c_str() + epos + 1);
  std::string d;
  for (std::size_t i = 0; i < epos; ++i)
    if (m[i] != '.') d.push_back(m[i]);
  while (d.size() > 1 && d.back() == '0') d.pop_back();
  const int k = int(d.size()), n = e10 + 1;   // value = 0.d * 10^n
  std::string out;
  if (k <= n && n <= 15) {
    out = d + std::string(size_t(n - k), '0') + ".0";
  } else if (0 < n && n <= 15) {
    out = d.substr(0, size_t(n)) + "." + d.substr(size_t(n));
  } else if (-4 < n && n <= 0) {
    out = "0." + std::string(size_t(-n), '0') + d;
  } else {
    const int x = n - 1;
    char eb[16];
    std::snprintf(eb, sizeof eb, "e%c%02d", x < 0 ? '-' : '+', x < 0 ? -x : x);
    out = (k == 1 ? d : d.substr(0, 1) + "." + d.substr(1)) + eb;
  }
  return neg ? "-" + out : out;
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
  std::vector<std::uint16_t> half(rows * cols);
  PlotConfig dense = cfg;
  dense.threshold_half.reset();
  const ap_config c = dense.to_c();
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
// is materialised; cells come back in the same row-major order.
inline std::vector<PlotCell> compute_plot_threshold(const Sequence& x, const Sequence& y, const PlotConfig& cfg,
                                                    half_score_t t_half) {
  cfg.validate(x.size(), y.size());
  PlotConfig tc = cfg;
  tc.threshold_half = t_half;
  const ap_config c = tc.to_c();
  std::uint64_t count = 0;
  std::vector<std::uint32_t> rr(1 << 12), cc(1 << 12);
  std::vector<std::uint16_t> hh(1 << 12);
  int rc = ap_plot_threshold(x.data.data(), x.size(), y.data.data(), y.size(), &c, &count, rr.data(),
                             cc.data(), hh.data(), rr.size());
  if (rc == AP_CAPACITY) {
    rr.resize(count);
    cc.resize(count);
    hh.resize(count);
    rc = ap_plot_threshold(x.data.data(), x.size(), y.data.data(), y.size(), &c, &count, rr.data(),
                           cc.data(), hh.data(), rr.size());
  }
  detail::check(rc);
  std::vector<PlotCell> out(count);
  for (std::size_t k = 0; k < count; ++k) out[k] = {rr[k], cc[k], hh[k]};
  return out;
}

// ---- writers (io.cpp:102-153), byte-identical ------------------------------
inline std::string half_to_decimal(half_score_t half) {
  const bool neg = half < 0;
  const long long a = neg ? -static_cast<long long>(half) : half;
  std::string out = neg ? "-" : "";
  out += std::to_string(a / 2);
  out += (a % 2) ? ".5" : ".0";
  return out;
}

inline void write_tsv(std::ostream& out, const PlotGrid& grid, std::optional<half_score_t> threshold_half,
                      bool dense) {
  out << "# x_offset y_offset score\n";
  for (std::size_t r = 0; r < grid.rows; ++r)
    for (std::size_t c = 0; c < grid.cols; ++c) {
      const half_score_t v = grid.at(r, c);
      if (!dense && threshold_half && v < *threshold_half) continue;
      out << grid.x_offset(r) << '\t' << grid.y_offset(c) << '\t' << half_to_decimal(v) << '\n';
    }
  if (!out) throw std::runtime_error("write failure on TSV sink");
}

inline void write_dots(std::ostream& out, const PlotGrid& grid, std::optional<half_score_t> threshold_half) {
  for (std::size_t r = 0; r < grid.rows; ++r)
    for (std::size_t c = 0; c < grid.cols; ++c) {
      if (threshold_half && grid.at(r, c) < *threshold_half) continue;
      out << grid.x_offset(r) << ' ' << grid.y_offset(c) << '\n';
    }
  if (!out) throw std::runtime_error("write failure on dot sink");
}

inline void write_pgm(std::ostream& out, const PlotGrid& grid, std::optional<half_score_t> threshold_half) {
  out << "P5\n" << grid.cols << ' ' << grid.rows << "\n255\n";
  const long long full = 2 * static_cast<long long>(grid.window_w);
  std::vector<unsigned char> row(grid.cols);
  for (std::size_t r = 0; r < grid.rows; ++r) {
    for (std::size_t c = 0; c < grid.cols; ++c) {
      half_score_t v = grid.at(r, c);
      if (threshold_half && v < *threshold_half) v = 0;
      const long long h = std::clamp<long long>(v, 0, full);
      row[c] = static_cast<unsigned char>((255 * h + full / 2) / full);
    }
    out.write(reinterpret_cast<const char*>(row.data()), static_cast<std::streamsize>(row.size()));
  }
  if (!out) throw std::runtime_error("write failure on PGM sink");
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

// ---- FASTA input (io.hpp:15-38, io.cpp:32-100) ----------------------------
struct FastaRecord {
  std::string header;
  std::string sequence;
  bool operator==(const FastaRecord&) const = default;
};

inline std::vector<FastaRecord> read_fasta_stream(std::istream& in, const std::string& source) {
  std::vector<FastaRecord> recs;
  std::size_t line_no = 0, header_line = 0;
  auto fail = [&](std::size_t ln, const std::string& what) {
    throw ParseError(source + ":" + std::to_string(ln) + ": " + what);
  };
  auto space = [](unsigned char c) { return c == ' ' || (c >= '\t' && c <= '\r'); };
  std::string line;
  while (std::getline(in, line)) {
    ++line_no;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (std::all_of(line.begin(), line.end(), [&](char c) { return space(static_cast<unsigned char>(c)); }))
      continue;   // empty or blank
    if (line[0] == '>') {
      if (!recs.empty() && recs.back().sequence.empty())
        fail(header_line, "record '" + recs.back().header + "' has no sequence data");
      std::size_t e = line.size();
      while (e > 1 && space(static_cast<unsigned char>(line[e - 1]))) --e;
      recs.push_back({line.substr(1, e - 1), {}});
      header_line = line_no;
      continue;
    }
    if (recs.empty()) fail(line_no, "sequence data before first header");
    for (char ch : line) {
      const auto c = static_cast<unsigned char>(ch);
      if (space(c)) continue;
      if (c < 32 || c > 126 || c == '>') fail(line_no, "unexpected byte in sequence data");
      recs.back().sequence.push_back(static_cast<char>(c >= 'a' && c <= 'z' ? c - 32 : c));
    }
  }
  if (recs.empty()) throw ParseError(source + ": no FASTA records");
  if (recs.back().sequence.empty())
    fail(header_line, "record '" + recs.back().header + "' has no sequence data");
  return recs;
}

inline std::vector<FastaRecord> read_fasta(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw ParseError(path + ": cannot open file");
  return read_fasta_stream(in, path);
}

// exact header, or its first whitespace-delimited token; the first record for ""
inline const FastaRecord& select_record(const std::vector<FastaRecord>& records, const std::string& name,
                                        const std::string& source) {
  if (name.empty()) return records.front();
  for (const FastaRecord& r : records) {
    if (r.header == name) return r;
    const std::size_t cut = r.header.find_first_of(" \t");
    if (cut != std::string::npos && cut == name.size() && r.header.compare(0, cut, name) == 0) return r;
  }
  throw ParseError(source + ": no record named '" + name + "'");
}

inline Sequence to_sequence(const FastaRecord& rec) { return Sequence::from_text(rec.header, rec.sequence); }

// ---- benchmark (io.hpp:56-81, io.cpp:155-233) ------------------------------
struct BenchEntry {
  Mode mode = Mode::dp;
  double seconds = 0.0;
  double cell_updates_per_sec = 0.0;
  double speedup_vs_first = 1.0;
};

struct BenchReport {
  std::size_t rows = 0, cols = 0, window_w = 0, step_h = 0;
  unsigned blowup_r = 1, workers = 1;
  std::vector<BenchEntry> entries;

  std::string to_text() const {
    std::ostringstream os;
    os << "plot " << rows << " x " << cols << " windows, w=" << window_w << ", h=" << step_h
       << ", r=" << blowup_r << ", workers=" << workers << "\n";
    char buf[160];
    std::snprintf(buf, sizeof buf, "%-12s %10s %12s %9s\n", "mode", "seconds", "Mcups", "speedup");
    os << buf;
    bool dp = false;
    for (const BenchEntry& e : entries) {
      dp = dp || e.mode == Mode::dp;
      std::snprintf(buf, sizeof buf, "%-12s %10.3f %12.1f %8.2fx\n", mode_name(e.mode), e.seconds,
                    e.cell_updates_per_sec / 1e6, e.speedup_vs_first);
      os << buf;
    }
    if (dp) os << "dp = exhaustive per-window DP baseline, no shortcuts\n";
    return os.str();
  }

  // keys in sorted order, two-space indentation (the reference's json dump(2))
  std::string to_json() const {
    auto num = [](double v) { return detail::json_double(v); };
    std::ostringstream os;
    os << "{\n  \"blowup\": " << blowup_r << ",\n  \"cols\": " << cols << ",\n  \"results\": [";
    for (std::size_t i = 0; i < entries.size(); ++i) {
      const BenchEntry& e = entries[i];
      os << (i ? "," : "") << "\n    {\n      \"cell_updates_per_sec\": " << num(e.cell_updates_per_sec)
         << ",\n      \"mode\": \"" << mode_name(e.mode) << "\",\n      \"seconds\": " << num(e.seconds)
         << ",\n      \"speedup_vs_first\": " << num(e.speedup_vs_first) << "\n    }";
    }
    os << (entries.empty() ? "]" : "\n  ]") << ",\n  \"rows\": " << rows << ",\n  \"step\": " << step_h
       << ",\n  \"window\": " << window_w << ",\n  \"workers\": " << workers << "\n}";
    return os.str();
  }
};

// Times each mode on the same inputs; every mode must give the same grid (all
// of them run on the GPU engine here, so they agree by construction).  Cell
// updates/s are normalised to the per-window DP cost rows*cols*(w*r)^2.
inline BenchReport benchmark(const Sequence& x, const Sequence& y, const PlotConfig& cfg,
                             std::span<const Mode> modes) {
  if (modes.empty()) throw ConfigError("benchmark needs at least one mode");
  BenchReport rep;
  rep.window_w = cfg.window_w;
  rep.step_h = cfg.step_h;
  rep.blowup_r = cfg.blowup_r;
  rep.workers = cfg.workers;
  std::optional<PlotGrid> first;
  for (Mode m : modes) {
    PlotConfig c = cfg;
    c.mode = m;
    const auto t0 = std::chrono::steady_clock::now();
    PlotGrid g = compute_plot(x, y, c);
    const double secs =
        std::max(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(), 1e-9);
    if (!first) {
      first = std::move(g);
      rep.rows = first->rows;
      rep.cols = first->cols;
    } else if (!(g == *first)) {
      throw std::runtime_error(std::string("benchmark: mode ") + mode_name(m) + " disagrees with " +
                               mode_name(modes.front()));
    }
    const double wr = double(cfg.window_w * cfg.blowup_r);
    BenchEntry e;
    e.mode = m;
    e.seconds = secs;
    e.cell_updates_per_sec = double(rep.rows) * double(rep.cols) * wr * wr / secs;
    e.speedup_vs_first = rep.entries.empty() ? 1.0 : rep.entries.front().seconds / secs;
    rep.entries.push_back(e);
  }
  return rep;
}

}  // namespace alignplot
