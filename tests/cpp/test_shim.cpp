// C++ drop-in test: the reference's own test cases (test_runner.cpp,
// test_scoring.cpp, test_model.cpp) written against alignplot_shim.hpp, i.e.
// the reference API served by the CUDA engine.  Instances come from the same
// seeded std::mt19937 generators as the reference tests; the ground truth is an
// independent per-window DP (as tests/test_util.hpp's ref_llcs /
// ref_align_score_half).  Exit status = number of failed checks.  Needs a GPU.
#include <cmath>
#include <cstdio>
#include <sstream>
#include <random>
#include <string>
#include <vector>

#include "../../paper_0909_2000_b200/csrc/alignplot_shim.hpp"

using namespace alignplot;

static int failures = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
      ++failures;                                                     \
    }                                                                 \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                      \
  do {                                                                \
    bool thrown_ = false;                                             \
    try { (void)(expr); } catch (const T&) { thrown_ = true; } catch (...) {} \
    CHECK(thrown_ && #T);                                             \
  } while (0)

static std::vector<std::uint8_t> random_codes(std::mt19937& rng, std::size_t len, unsigned sigma) {
  std::uniform_int_distribution<unsigned> dist(1, sigma);
  std::vector<std::uint8_t> out(len);
  for (auto& c : out) c = static_cast<std::uint8_t>(dist(rng));
  return out;
}

static std::size_t ref_llcs(std::span<const std::uint8_t> a, std::span<const std::uint8_t> b) {
  std::vector<std::size_t> prev(b.size() + 1, 0), cur(b.size() + 1, 0);
  for (std::size_t i = 1; i <= a.size(); ++i) {
    for (std::size_t j = 1; j <= b.size(); ++j)
      cur[j] = a[i - 1] == b[j - 1] ? prev[j - 1] + 1 : std::max(prev[j], cur[j - 1]);
    std::swap(prev, cur);
  }
  return prev[b.size()];
}

static half_score_t ref_align_score_half(std::span<const std::uint8_t> a, std::span<const std::uint8_t> b) {
  std::vector<half_score_t> prev(b.size() + 1), cur(b.size() + 1);
  for (std::size_t j = 0; j <= b.size(); ++j) prev[j] = -static_cast<half_score_t>(j);
  for (std::size_t i = 1; i <= a.size(); ++i) {
    cur[0] = -static_cast<half_score_t>(i);
    for (std::size_t j = 1; j <= b.size(); ++j) {
      const half_score_t diag = prev[j - 1] + (a[i - 1] == b[j - 1] ? 2 : 0);
      cur[j] = std::max({diag, prev[j] - 1, cur[j - 1] - 1});
    }
    std::swap(prev, cur);
  }
  return prev[b.size()];
}

static PlotGrid truth(const Sequence& x, const Sequence& y, const PlotConfig& cfg) {
  const auto [rows, cols] = window_grid_dims(x.size(), y.size(), cfg.window_w, cfg.step_h);
  PlotGrid g(rows, cols, cfg.window_w, cfg.step_h);
  for (std::size_t r = 0; r < rows; ++r)
    for (std::size_t c = 0; c < cols; ++c) {
      const auto xw = x.codes().subspan(g.x_offset(r), cfg.window_w);
      const auto yw = y.codes().subspan(g.y_offset(c), cfg.window_w);
      g.at(r, c) = cfg.blowup_r == 1 ? static_cast<half_score_t>(2 * ref_llcs(xw, yw)) : ref_align_score_half(xw, yw);
    }
  return g;
}

int main() {
  {  // test_runner.cpp:30-50 "every engine produces the ground-truth plot"
    std::mt19937 rng(555);
    for (int it = 0; it < 12; ++it) {
      const std::size_t w = 3 + (it * 7) % 20;
      std::uniform_int_distribution<std::size_t> len(w, 90);
      const Sequence x("x", random_codes(rng, len(rng), 4));
      const Sequence y("y", random_codes(rng, len(rng), 4));
      PlotConfig cfg;
      cfg.window_w = w;
      cfg.step_h = 1 + it % 3;
      cfg.blowup_r = it % 2 ? 1 : 2;
      const PlotGrid want = truth(x, y, cfg);
      for (Mode m : {Mode::blcs, Mode::sea_scalar, Mode::sea16, Mode::sea8, Mode::cuda}) {
        PlotConfig c = cfg;
        c.mode = m;
        CHECK(compute_plot(x, y, c) == want);
      }
    }
  }
  {  // test_runner.cpp:52-70 (seed 556) and :72-89 (seed 557)
    std::mt19937 rng(556);
    const Sequence x("x", random_codes(rng, 40, 3)), y("y", random_codes(rng, 60, 3));
    PlotConfig cfg;
    cfg.window_w = 8; cfg.step_h = 2; cfg.blowup_r = 1; cfg.mode = Mode::sea_scalar;
    CHECK(compute_plot(x, y, cfg) == truth(x, y, cfg));
    std::mt19937 rng2(557);
    const Sequence x2("x", random_codes(rng2, 30, 4)), y2("y", random_codes(rng2, 45, 4));
    PlotConfig c2;
    c2.window_w = 10; c2.step_h = 3; c2.blowup_r = 2; c2.mode = Mode::sea8;
    CHECK(compute_plot(x2, y2, c2) == truth(x2, y2, c2));
  }
  {  // test_runner.cpp:91-105 "worker count never changes the plot" (+ device count)
    std::mt19937 rng(558);
    const Sequence x("x", random_codes(rng, 240, 4)), y("y", random_codes(rng, 200, 4));
    PlotConfig cfg;
    cfg.window_w = 32; cfg.step_h = 3; cfg.mode = Mode::sea8; cfg.workers = 1;
    const PlotGrid reference = compute_plot(x, y, cfg);
    CHECK(reference == truth(x, y, cfg));
    for (unsigned workers : {2u, 3u, 4u, 8u, 64u}) {
      cfg.workers = workers;
      CHECK(compute_plot(x, y, cfg) == reference);
    }
    for (int dev : {2, 4, 8}) {
      cfg.n_devices = dev;
      CHECK(compute_plot(x, y, cfg) == reference);
    }
  }
  {  // test_runner.cpp:118-127 "compute_plot validates before running"
    const Sequence x("x", {1, 2, 1}), y("y", {2, 1, 2});
    PlotConfig cfg;
    cfg.window_w = 10;
    CHECK_THROWS_AS(compute_plot(x, y, cfg), EmptyPlotError);
    cfg.window_w = 2;
    cfg.blowup_r = 7;
    CHECK_THROWS_AS(compute_plot(x, y, cfg), ConfigError);
  }
  {  // test_runner.cpp:129-145 "grid geometry carries window, step, and origins"
    const Sequence x("x", std::vector<std::uint8_t>(25, 1)), y("y", std::vector<std::uint8_t>(11, 1));
    PlotConfig cfg;
    cfg.window_w = 10; cfg.step_h = 5; cfg.mode = Mode::dp;
    const PlotGrid g = compute_plot(x, y, cfg);
    CHECK(g.rows == 4 && g.cols == 2 && g.window_w == 10 && g.step_h == 5);
    CHECK(g.x_offset(3) == 15 && g.y_offset(1) == 1);
    CHECK(g.at(0, 0) == 2 * 10);
  }
  {  // test_scoring.cpp:55-68 threshold order, and the fused GPU threshold path
    PlotGrid g(2, 2, 4, 1);
    g.at(0, 0) = 4; g.at(0, 1) = 1; g.at(1, 0) = 3; g.at(1, 1) = 4;
    const auto cells = apply_threshold(g, 3);
    CHECK(cells.size() == 3 && cells[0] == (PlotCell{0, 0, 4}) && cells[1] == (PlotCell{1, 0, 3}) &&
          cells[2] == (PlotCell{1, 1, 4}));
    std::mt19937 rng(559);
    const Sequence x("x", random_codes(rng, 300, 4));
    std::vector<std::uint8_t> yv(x.data.begin() + 50, x.data.begin() + 250);
    const Sequence y("y", yv);
    for (unsigned r : {1u, 2u}) {
      PlotConfig cfg;
      cfg.window_w = 24; cfg.step_h = 2; cfg.blowup_r = r;
      const PlotGrid grid = compute_plot(x, y, cfg);
      const half_score_t t = 30;
      CHECK(compute_plot_threshold(x, y, cfg, t) == apply_threshold(grid, t));
    }
  }
  {  // test_model.cpp:63-82 lane capacity bound and validation
    PlotConfig cfg;
    cfg.mode = Mode::sea8; cfg.step_h = 1; cfg.window_w = 100; cfg.blowup_r = 2;
    cfg.validate(300, 300);
    cfg.window_w = 254; cfg.blowup_r = 1;
    cfg.validate(300, 300);
    cfg.window_w = 255;
    CHECK_THROWS_AS(cfg.validate(300, 300), ConfigError);
    CHECK_THROWS_AS(Sequence("bad", {1, 0, 2}), ConfigError);
    CHECK_THROWS_AS(window_grid_dims(10, 10, 20, 1), EmptyPlotError);
    CHECK(window_grid_dims(2712, 628, 100, 5) == (std::pair<std::size_t, std::size_t>{523, 529}));
  }
  {  // test_scoring.cpp:11-37
    const BlownSequence b = blowup(Sequence::from_text("s", "abab"));
    CHECK(b.data == (std::vector<std::uint8_t>{0, 'a', 0, 'b', 0, 'a', 0, 'b'}));
    CHECK(unblow(b) == Sequence::from_text("s", "abab").data);
    CHECK(recover_score(4, 2, 2) == 4 && recover_score(2, 2, 2) == 0 && recover_score(2, 1, 2) == 1);
  }
  {  // writers (io.cpp:102-153 byte format) fed from the device, against formatting of compute_plot's grid
    std::mt19937 rng(560);
    const Sequence x("x", random_codes(rng, 200, 4)), y("y", random_codes(rng, 260, 4));
    auto dec = [](half_score_t v) {   // half-units as "k.0" / "k.5"
      const long long a = v < 0 ? -static_cast<long long>(v) : v;
      return std::string(v < 0 ? "-" : "") + std::to_string(a / 2) + (a % 2 ? ".5" : ".0");
    };
    for (unsigned r : {1u, 2u}) {
      PlotConfig cfg;
      cfg.window_w = 20; cfg.step_h = 3; cfg.blowup_r = r; cfg.threshold_half = 18;
      const PlotGrid g = compute_plot(x, y, cfg);
      std::string tsv_all = "# x_offset y_offset score\n", tsv_thr = tsv_all, dots;
      std::string pgm = "P5\n" + std::to_string(g.cols) + " " + std::to_string(g.rows) + "\n255\n";
      const long long full = 2 * static_cast<long long>(g.window_w);
      for (std::size_t i = 0; i < g.rows; ++i)
        for (std::size_t k = 0; k < g.cols; ++k) {
          const half_score_t v = g.at(i, k);
          const std::string pos = std::to_string(g.x_offset(i)) + "\t" + std::to_string(g.y_offset(k));
          tsv_all += pos + "\t" + dec(v) + "\n";
          if (v >= 18) {
            tsv_thr += pos + "\t" + dec(v) + "\n";
            dots += std::to_string(g.x_offset(i)) + " " + std::to_string(g.y_offset(k)) + "\n";
          }
          const long long h = std::clamp<long long>(v < 18 ? 0 : v, 0, full);
          pgm.push_back(static_cast<char>((255 * h + full / 2) / full));
        }
      std::ostringstream a, b, c, d;
      write_tsv_gpu(a, x, y, cfg, true);
      write_tsv_gpu(b, x, y, cfg, false);
      write_dots_gpu(c, x, y, cfg);
      write_pgm_gpu(d, x, y, cfg);
      CHECK(a.str() == tsv_all);
      CHECK(b.str() == tsv_thr);
      CHECK(c.str() == dots);
      CHECK(d.str() == pgm);
    }
  }
  {  // large windows: sea16 mode up to w*r = 65534 (model.cpp:57-59); LCS scores past 16 bits
    std::mt19937 rng(9090);
    const std::vector<std::uint8_t> xs = random_codes(rng, 32800, 4);
    const Sequence x("x", xs), y("y", xs);
    PlotConfig cfg;
    cfg.mode = Mode::sea16; cfg.window_w = 32800; cfg.step_h = 1; cfg.blowup_r = 1;
    const PlotGrid g = compute_plot(x, y, cfg);            // one cell: the LCS of a string with itself
    CHECK(g.rows == 1 && g.cols == 1 && g.at(0, 0) == 2 * 32800);
    const auto cells = compute_plot_threshold(x, y, cfg, 65000);
    CHECK(cells.size() == 1 && cells[0].score_half == 65600);
    cfg.window_w = 32767; cfg.blowup_r = 2;                // the alignment-score bound w*r = 65534
    CHECK(compute_plot(x, y, cfg).at(0, 0) == 2 * 32767);
    cfg.window_w = 32768;
    CHECK_THROWS_AS(compute_plot(x, y, cfg), ConfigError);
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "ok", failures);
  return failures;
}
