// leuven_compute — the reference CLI's `compute` subcommand
// (proj/src/cli.cpp:53-119, 240-330) in C++ over include/leuven_b200.hpp:
// flag parsing only; compute_report, report_json, the human report and the
// exit-code mapping are the header's leuven::b200::cli functions, i.e. what
// a C++ maintainer gets when cli::compute_report's SimBackend is replaced by
// GpuBackend.
//
//   leuven_compute --a monday --b friday [--mode exact|skip|approx] [--ell K]
//                  [--encoding ascii7|lower26|dna4] [--budget B]
//                  [--key-encoding negated|original] [--preprocess] [--json]
//
// Report fields, field order and exit codes as the reference (report_json
// cli.cpp:93-107, print_human_report :110-119, classify_error_exit :121-129:
// 3 band too narrow, 2 input / parameter errors, 1 anything else).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "leuven_b200.hpp"

using namespace leuven;
using namespace leuven::b200;

namespace {

struct Options {
  cli::ComputeConfig c;
  bool json = false, have_a = false, have_b = false;
};

}  // namespace

int main(int argc, char** argv) {
  Options o;
  if (const char* env = std::getenv("LEUVEN_BUDGET")) o.c.budget = std::atof(env);  // cli.cpp:131-147
  for (int i = 1; i < argc; ++i) {
    const std::string k = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) {
        std::fprintf(stderr, "missing value for %s\n", k.c_str());
        std::exit(2);
      }
      return argv[++i];
    };
    if (k == "--a") o.c.a = val(), o.have_a = true;
    else if (k == "--b") o.c.b = val(), o.have_b = true;
    else if (k == "--mode") o.c.mode = val();
    else if (k == "--ell") o.c.ell = std::strtoull(val().c_str(), nullptr, 10), o.c.has_ell = true;
    else if (k == "--encoding") o.c.encoding = val();
    else if (k == "--budget") o.c.budget = std::atof(val().c_str());
    else if (k == "--key-encoding") o.c.key_encoding = val();
    else if (k == "--preprocess") o.c.preprocess = true;
    else if (k == "--json") o.json = true;
    else {
      std::fprintf(stderr, "unknown option %s\n", k.c_str());
      return 2;
    }
  }
  if (!o.have_a || !o.have_b) {
    std::fprintf(stderr, "--a and --b are required\n");
    return 2;
  }
  try {
    // cli::compute_report (cli.cpp:53-91) on the GPU backend, keys made on the device
    const cli::RunReport r = cli::compute_report(o.c);
    std::fputs(o.json ? (cli::report_json(r, true) + "\n").c_str() : cli::human_report(r).c_str(), stdout);
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return cli::classify_error_exit(e);
  }
}
