// golden_gen.cpp — writes the reference-generated golden fixtures under
// tests/golden/.  TEST INFRASTRUCTURE ONLY (built by oracle/Makefile against
// the reference sources in place; run in the build container, never on the
// GPU box).
//
// Each fixture replays the seeded instance generator of one reference test
// (std::mt19937 + testutil::random_codes, included in place from
// /root/reference/proj/tests/test_util.hpp, same libstdc++ as the reference
// build) and records the reference library's own output:
//   runner_engines   test_runner.cpp:30-50      seed 555, dp_plot grids
//   runner_lcs       test_runner.cpp:52-70      seed 556, sea_scalar grid
//   runner_align     test_runner.cpp:72-89      seed 557, sea8 grid
//   runner_workers   test_runner.cpp:91-105     seed 558, sea8 grid
//   lane_w100        test_lane_kernel.cpp:177-186 seed 31337, window LLCS
//   seaweed_scan     test_seaweed.cpp:148-165   seed 2025, window LLCS stride 1/2
//   acceptance1      acceptance.cpp:34-73       seed 101, 540 instances, grid hash
//   acceptance7      acceptance.cpp:248-274     seed 107, 2000x2000 w100 h5 r2, grid hash
// Grid hash (also in tests/golden_util.py): sum_i (uint32(v_i) + 0x9E37) *
// splitmix64(i) mod 2^64, row-major.
#include <cstdint>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "alignplot/baselines.hpp"
#include "alignplot/runner.hpp"
#include "alignplot/lane_kernel.hpp"
#include "alignplot/scoring.hpp"
#include "alignplot/seaweed_scalar.hpp"
#include "test_util.hpp"

using namespace alignplot;

static uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static uint64_t grid_hash(const std::vector<int32_t>& v) {
  uint64_t h = 0;
  for (size_t i = 0; i < v.size(); ++i) h += (uint64_t(uint32_t(v[i])) + 0x9E37ull) * splitmix64(i);
  return h;
}
static std::string hex(const std::vector<uint8_t>& b) {
  static const char* d = "0123456789abcdef";
  std::string s;
  for (uint8_t c : b) { s += d[c >> 4]; s += d[c & 15]; }
  return s;
}
template <typename T>
static std::string list(const std::vector<T>& v) {
  std::string s = "[";
  for (size_t i = 0; i < v.size(); ++i) { if (i) s += ","; s += std::to_string(v[i]); }
  return s + "]";
}
static FILE* open_out(const std::string& dir, const char* name) {
  std::string p = dir + "/" + name;
  FILE* f = std::fopen(p.c_str(), "w");
  if (!f) { std::perror(p.c_str()); std::exit(1); }
  return f;
}
static void grid_case(FILE* f, bool& first, const Sequence& x, const Sequence& y, const PlotConfig& c,
                      const PlotGrid& g, bool full) {
  std::fprintf(f, "%s\n {\"x\":\"%s\",\"y\":\"%s\",\"w\":%zu,\"h\":%zu,\"r\":%u,\"rows\":%zu,\"cols\":%zu,\"hash\":\"%llu\"",
               first ? "" : ",", hex(x.data).c_str(), hex(y.data).c_str(), c.window_w, c.step_h, c.blowup_r,
               g.rows, g.cols, (unsigned long long)grid_hash(g.values));
  if (full) std::fprintf(f, ",\"grid\":%s", list(g.values).c_str());
  std::fprintf(f, "}");
  first = false;
}

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "tests/golden";
  {  // test_runner.cpp:30-50
    FILE* f = open_out(dir, "runner_engines.json");
    std::fprintf(f, "{\"source\":\"test_runner.cpp:30-50 seed 555 (dp_plot ground truth)\",\"cases\":[");
    bool first = true;
    std::mt19937 rng(555);
    for (int it = 0; it < 12; ++it) {
      const std::size_t w = 3 + (it * 7) % 20;
      std::uniform_int_distribution<std::size_t> len(w, 90);
      const Sequence x = testutil::make_seq("x", testutil::random_codes(rng, len(rng), 4));
      const Sequence y = testutil::make_seq("y", testutil::random_codes(rng, len(rng), 4));
      PlotConfig cfg;
      cfg.window_w = w;
      cfg.step_h = 1 + it % 3;
      cfg.blowup_r = it % 2 ? 1 : 2;
      grid_case(f, first, x, y, cfg, dp_plot(x, y, cfg), true);
    }
    std::fprintf(f, "]}\n");
    std::fclose(f);
  }
  {  // test_runner.cpp:52-89 and :91-105
    FILE* f = open_out(dir, "runner_modes.json");
    std::fprintf(f, "{\"source\":\"test_runner.cpp:52-70 seed 556, :72-89 seed 557, :91-105 seed 558\",\"cases\":[");
    bool first = true;
    {
      std::mt19937 rng(556);
      const Sequence x = testutil::make_seq("x", testutil::random_codes(rng, 40, 3));
      const Sequence y = testutil::make_seq("y", testutil::random_codes(rng, 60, 3));
      PlotConfig cfg; cfg.window_w = 8; cfg.step_h = 2; cfg.blowup_r = 1; cfg.mode = Mode::sea_scalar;
      grid_case(f, first, x, y, cfg, compute_plot(x, y, cfg), true);
    }
    {
      std::mt19937 rng(557);
      const Sequence x = testutil::make_seq("x", testutil::random_codes(rng, 30, 4));
      const Sequence y = testutil::make_seq("y", testutil::random_codes(rng, 45, 4));
      PlotConfig cfg; cfg.window_w = 10; cfg.step_h = 3; cfg.blowup_r = 2; cfg.mode = Mode::sea8;
      grid_case(f, first, x, y, cfg, compute_plot(x, y, cfg), true);
    }
    {
      std::mt19937 rng(558);
      const Sequence x = testutil::make_seq("x", testutil::random_codes(rng, 240, 4));
      const Sequence y = testutil::make_seq("y", testutil::random_codes(rng, 200, 4));
      PlotConfig cfg; cfg.window_w = 32; cfg.step_h = 3; cfg.mode = Mode::sea8; cfg.workers = 1;
      grid_case(f, first, x, y, cfg, compute_plot(x, y, cfg), true);
    }
    std::fprintf(f, "]}\n");
    std::fclose(f);
  }
  {  // test_lane_kernel.cpp:177-186 and test_seaweed.cpp:148-165
    FILE* f = open_out(dir, "strips.json");
    std::fprintf(f, "{\"source\":\"test_lane_kernel.cpp:177-186 seed 31337; test_seaweed.cpp:148-165 seed 2025\",\"cases\":[");
    {
      std::mt19937 rng(31337);
      const auto x = testutil::random_codes(rng, 100, 4);
      const auto y = testutil::random_codes(rng, 140, 4);
      const auto xb = blowup(std::span<const std::uint8_t>(x));
      const auto yb = blowup(std::span<const std::uint8_t>(y));
      const CombResult res = comb_strip(xb.codes(), yb.codes());
      const auto ll = window_llcs_from_events(res.events, 200, 2);
      std::fprintf(f, "\n {\"xw\":\"%s\",\"y\":\"%s\",\"w\":100,\"r\":2,\"stride\":2,\"window_cols\":200,\"llcs\":%s}",
                   hex(x).c_str(), hex(y).c_str(), list(ll).c_str());
    }
    {
      std::mt19937 rng(2025);
      for (int it = 0; it < 40; ++it) {
        const std::size_t w = 2 + it % 5;
        const std::size_t n = w + (it * 3) % 20;
        const auto xw = testutil::random_codes(rng, w, 4);
        const auto y = testutil::random_codes(rng, n, 4);
        const CombResult res = comb_strip(xw, y);
        for (std::size_t stride : {std::size_t{1}, std::size_t{2}}) {
          const auto ll = window_llcs_from_events(res.events, w, stride);
          std::vector<int32_t> starts;
          for (auto& e : res.events) starts.push_back(e.start_col);
          std::fprintf(f, ",\n {\"xw\":\"%s\",\"y\":\"%s\",\"w\":%zu,\"r\":1,\"stride\":%zu,\"window_cols\":%zu,\"llcs\":%s,\"starts\":%s}",
                       hex(xw).c_str(), hex(y).c_str(), w, stride, w, list(ll).c_str(), list(starts).c_str());
        }
      }
    }
    std::fprintf(f, "]}\n");
    std::fclose(f);
  }
  {  // acceptance.cpp:34-73
    FILE* f = open_out(dir, "acceptance1.json");
    std::fprintf(f, "{\"source\":\"acceptance.cpp:34-73 seed 101, reference sea8 grid (== dp)\",\"cases\":[");
    bool first = true;
    std::mt19937 rng(101);
    for (unsigned sigma : {2u, 4u, 20u})
      for (std::size_t w : {4u, 8u, 16u, 32u, 64u})
        for (std::size_t h : {1u, 3u, 5u})
          for (unsigned r : {1u, 2u})
            for (int rep = 0; rep < 6; ++rep) {
              std::uniform_int_distribution<std::size_t> len(w, 300);
              const Sequence x = testutil::make_seq("x", testutil::random_codes(rng, len(rng), sigma));
              const Sequence y = testutil::make_seq("y", testutil::random_codes(rng, len(rng), sigma));
              PlotConfig cfg;
              cfg.window_w = w;
              cfg.step_h = h;
              cfg.blowup_r = r;
              cfg.mode = Mode::sea8;
              grid_case(f, first, x, y, cfg, compute_plot(x, y, cfg), false);
            }
    std::fprintf(f, "]}\n");
    std::fclose(f);
  }
  {  // acceptance.cpp:248-274
    FILE* f = open_out(dir, "acceptance7.json");
    std::fprintf(f, "{\"source\":\"acceptance.cpp:248-274 seed 107, reference sea8 grid\",\"cases\":[");
    bool first = true;
    std::mt19937 rng(107);
    const Sequence x = testutil::make_seq("x", testutil::random_codes(rng, 2000, 4));
    const Sequence y = testutil::make_seq("y", testutil::random_codes(rng, 2000, 4));
    PlotConfig cfg;
    cfg.window_w = 100; cfg.step_h = 5; cfg.blowup_r = 2; cfg.mode = Mode::sea8; cfg.workers = 8;
    grid_case(f, first, x, y, cfg, compute_plot(x, y, cfg), false);
    std::fprintf(f, "]}\n");
    std::fclose(f);
  }
  return 0;
}
