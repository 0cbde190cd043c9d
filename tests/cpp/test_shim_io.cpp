// CPU-only checks of the C++ drop-in's io part (alignplot_shim.hpp): the FASTA
// reader / record selection behaviour of io.cpp:32-100 (error kinds and line
// numbers), BenchReport formatting (io.cpp:155-190).  Exit status = failures.
#include <cstdio>
#include <sstream>
#include <string>

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

static std::string parse_error(const std::string& text) {
  std::istringstream in(text);
  try {
    read_fasta_stream(in, "t.fa");
  } catch (const ParseError& e) {
    return e.what();
  }
  return "";
}

int main() {
  {
    std::istringstream in(">chr1 desc  \r\nacgt\n\n  AC GT\r\n>chr2\nnn\n");
    const auto recs = read_fasta_stream(in, "t.fa");
    CHECK(recs.size() == 2);
    CHECK(recs[0].header == "chr1 desc");
    CHECK(recs[0].sequence == "ACGTACGT");
    CHECK(recs[1].sequence == "NN");
    CHECK(&select_record(recs, "", "t.fa") == &recs[0]);
    CHECK(&select_record(recs, "chr1", "t.fa") == &recs[0]);
    CHECK(&select_record(recs, "chr1 desc", "t.fa") == &recs[0]);
    CHECK(&select_record(recs, "chr2", "t.fa") == &recs[1]);
    bool threw = false;
    try { select_record(recs, "chr", "t.fa"); } catch (const ParseError& e) {
      threw = std::string(e.what()) == "t.fa: no record named 'chr'";
    }
    CHECK(threw);
    const Sequence s = to_sequence(recs[0]);
    CHECK(s.size() == 8 && s.name == "chr1 desc");
  }
  CHECK(parse_error("ACGT\n>x\nA\n") == "t.fa:1: sequence data before first header");
  CHECK(parse_error(">x\n>y\nAC\n") == "t.fa:1: record 'x' has no sequence data");
  CHECK(parse_error(">x\nAC\n>y\n\n") == "t.fa:3: record 'y' has no sequence data");
  CHECK(parse_error(">x\nA\x01C\n") == "t.fa:2: unexpected byte in sequence data");
  CHECK(parse_error(">x\nA>C\n") == "t.fa:2: unexpected byte in sequence data");
  CHECK(parse_error("\n  \n") == "t.fa: no FASTA records");
  {
    bool threw = false;
    try { read_fasta("/nonexistent/x.fa"); } catch (const ParseError& e) {
      threw = std::string(e.what()) == "/nonexistent/x.fa: cannot open file";
    }
    CHECK(threw);
  }
  {
    BenchReport r;
    r.rows = 3; r.cols = 4; r.window_w = 5; r.step_h = 1; r.blowup_r = 2; r.workers = 8;
    r.entries.push_back({Mode::dp, 2.0, 1.5e6, 1.0});
    r.entries.push_back({Mode::cuda, 0.5, 6.0e6, 4.0});
    const std::string t = r.to_text();
    CHECK(t == "plot 3 x 4 windows, w=5, h=1, r=2, workers=8\n"
               "mode            seconds        Mcups   speedup\n"
               "dp                2.000          1.5     1.00x\n"
               "cuda              0.500          6.0     4.00x\n"
               "dp = exhaustive per-window DP baseline, no shortcuts\n");
    const std::string j = r.to_json();
    CHECK(j.find("\"blowup\": 2") != std::string::npos);
    CHECK(j.find("\"mode\": \"cuda\"") != std::string::npos);
    CHECK(j.find("\"workers\": 8\n}") != std::string::npos);
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "ok", failures);
  return failures;
}
