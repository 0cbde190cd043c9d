// ref_cli.cpp — the reference CLI's plot path (tools/alignplot.cpp:96-147)
// driven by positional arguments instead of CLI11 (absent from the image), on
// the UNMODIFIED reference library (io.cpp writers + compute_plot).
// TEST INFRASTRUCTURE ONLY: makes the byte-exact CLI fixtures in
// tests/golden/cli/ (see tests/golden/make_cli_golden.sh).
//   ref_cli X.fa Y.fa WINDOW STEP LCS_ONLY(0|1) FORMAT(tsv|pgm|dots) DENSE(0|1) [THRESHOLD]
#include <cmath>
#include <cstdio>
#include <iostream>
#include <string>

#include "alignplot/io.hpp"
#include "alignplot/model.hpp"
#include "alignplot/runner.hpp"

int main(int argc, char** argv) {
  using namespace alignplot;
  if (argc < 8) {
    std::fprintf(stderr, "usage: ref_cli X.fa Y.fa W H LCS_ONLY FORMAT DENSE [THRESHOLD]\n");
    return 2;
  }
  try {
    const auto xr = read_fasta(argv[1]);
    const auto yr = read_fasta(argv[2]);
    const Sequence x = to_sequence(select_record(xr, "", argv[1]));
    const Sequence y = to_sequence(select_record(yr, "", argv[2]));
    PlotConfig cfg;
    cfg.window_w = std::stoul(argv[3]);
    cfg.step_h = std::stoul(argv[4]);
    cfg.blowup_r = std::stoi(argv[5]) ? 1 : 2;
    cfg.mode = Mode::sea8;
    cfg.workers = 4;
    const std::string format = argv[6];
    const bool dense = std::stoi(argv[7]) != 0;
    if (argc > 8) cfg.threshold_half = static_cast<half_score_t>(std::llround(std::stod(argv[8]) * 2));
    const PlotGrid grid = compute_plot(x, y, cfg);
    if (format == "tsv") write_tsv(std::cout, grid, cfg.threshold_half, dense);
    else if (format == "pgm") write_pgm(std::cout, grid, cfg.threshold_half);
    else write_dots(std::cout, grid, cfg.threshold_half);
    std::cout.flush();
    return 0;
  } catch (const std::exception& e) {
    std::cerr << "alignplot: " << e.what() << '\n';
    return 1;
  }
}
