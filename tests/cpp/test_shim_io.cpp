// CPU-only checks of the C++ drop-in's output formatting (alignplot_shim.hpp,
// no device work): half-unit scores print as io.cpp:102-119 prints them
// ("k.0" / "k.5", sign first), through the buffered line sink the GPU-fed
// writers use.  Exit status = failures.
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

static std::string half(half_score_t v) {
  char buf[32];
  return std::string(buf, detail::put_half(buf, v));
}

int main() {
  CHECK(half(0) == "0.0");
  CHECK(half(4) == "2.0");
  CHECK(half(1) == "0.5");
  CHECK(half(-3) == "-1.5");
  CHECK(half(-2) == "-1.0");
  CHECK(half(513) == "256.5");
  CHECK(half(-2147483647 - 1) == "-1073741824.0");
  {
    std::ostringstream os;
    detail::LineSink sink(os);
    std::string want;
    for (int i = 0; i < 200000; ++i) {   // several 1 MiB blocks
      char* p = sink.reserve(32);
      p = detail::put_half(p, i - 7);
      *p++ = '\n';
      sink.commit(p);
      want += half(i - 7) + "\n";
    }
    sink.flush();
    CHECK(os.str() == want);
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "ok", failures);
  return failures;
}
