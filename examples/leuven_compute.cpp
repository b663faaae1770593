// leuven_compute — the reference CLI's `compute` subcommand
// (proj/src/cli.cpp:53-119, 240-330) written in C++ against the B200
// backend through include/leuven_b200.hpp: what a C++ maintainer gets when
// cli::compute_report's SimBackend is replaced by GpuBackend.
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

struct Alphabet {  // encoding.cpp:78-96 builtins: code and little-endian symbol widths
  std::string name;
  std::vector<int> widths;
  int code(char c) const {
    const unsigned char u = static_cast<unsigned char>(c);
    if (name == "ascii7" && u < 128) return u;
    if (name == "lower26" && c >= 'a' && c <= 'z') return c - 'a';
    if (name == "dna4") {
      const char* s = "ACGT";
      for (int i = 0; i < 4; ++i)
        if (c == s[i]) return i;
    }
    throw CharNotInAlphabet(std::string("character not in alphabet '") + name + "'");
  }
  std::vector<int32_t> symbols(char c) const {  // encode_char, encoding.cpp:169-178
    int v = code(c);
    std::vector<int32_t> out;
    for (int w : widths) {
      out.push_back(v & ((1 << w) - 1));
      v >>= w;
    }
    return out;
  }
  std::vector<char> charset() const {
    std::vector<char> cs;
    for (int u = 0; u < 128; ++u) {
      try {
        code(static_cast<char>(u));
        cs.push_back(static_cast<char>(u));
      } catch (const CharNotInAlphabet&) {
      }
    }
    return cs;
  }
};

Alphabet alphabet(const std::string& name) {
  if (name == "ascii7") return {name, {4, 3}};
  if (name == "lower26") return {name, {4, 1}};
  if (name == "dna4") return {name, {2}};
  throw InvalidParams("unknown encoding '" + name + "'");
}

EncryptedString encrypt_string(GpuBackend& be, const std::string& s, const Alphabet& al) {
  std::vector<int32_t> v;  // one batched encryption (encoding.cpp:205-217)
  for (char c : s)
    for (int32_t x : al.symbols(c)) v.push_back(x);
  EncryptedString e;
  e.symbols = static_cast<uint32_t>(al.widths.size());
  if (!v.empty()) e.syms = be.encrypt(v);
  return e;
}

struct Options {
  std::string a, b, mode = "exact", encoding = "ascii7", key = "negated";
  long long ell = -1;
  double budget = 4000.0;
  bool preprocess = false, json = false, have_a = false, have_b = false;
};

int run(const Options& o) {
  const Alphabet al = alphabet(o.encoding);
  BandSpec band = o.mode == "exact"  ? BandSpec::exact(o.a.size(), o.b.size())
                  : o.mode == "skip" ? BandSpec::skip(o.a.size(), o.b.size())
                  : o.mode == "approx"
                      ? (o.ell < 0 ? throw InvalidParams("--mode approx requires --ell")
                                   : BandSpec::approx(static_cast<uint64_t>(o.ell)))
                      : throw InvalidParams("unknown mode '" + o.mode + "'");
  const KeyEncoding ke = o.key == "original" ? KeyEncoding::original : KeyEncoding::negated;
  GpuBackend be(o.budget);  // keys generated on the device
  const auto t0 = std::chrono::steady_clock::now();
  const uint64_t pbs0 = be.stats().pbs_count;
  const EncryptedString xs = encrypt_string(be, o.a, al);
  uint64_t pre = 0;
  DistanceRun run{};
  if (o.preprocess) {  // cli.cpp:64-69
    std::vector<std::pair<char, std::vector<int32_t>>> rows;
    for (char c : al.charset()) rows.push_back({c, al.symbols(c)});
    EqTable* t = build_eq_table(be, xs, rows, &pre);
    try {
      run = distance_preprocessed(be, *t, o.b, band, ke);
    } catch (...) {
      delete t;
      throw;
    }
    delete t;
  } else {
    const EncryptedString ys = encrypt_string(be, o.b, al);
    run = distance_encrypted(be, xs, ys, band, ke);
  }
  const int distance = be.decrypt(run.score);
  const double ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  const uint64_t pbs_total = be.stats().pbs_count - pbs0;
  const lv_run& c = run.counters;
  if (o.json) {
    std::printf(
        "{\"distance\":%d,\"mode\":\"%s\",\"half_width\":%llu,\"visited_cells\":%llu,"
        "\"pbs_total\":%llu,\"pbs_equality\":%llu,\"pbs_kernel\":%llu,\"refresh_count\":%llu,"
        "\"preprocessing_pbs\":%llu,\"max_key_variance\":%lld,\"wall_time_ms\":%.3f}\n",
        distance, o.mode.c_str(), (unsigned long long)band.b.half_width,
        (unsigned long long)c.visited_cells, (unsigned long long)pbs_total,
        (unsigned long long)c.equality_pbs, (unsigned long long)c.kernel_pbs,
        (unsigned long long)c.refreshes, (unsigned long long)pre, (long long)c.max_key_variance, ms);
  } else {
    std::printf("distance: %d\nmode: %s (half-width %llu)\nvisited cells: %llu\n", distance,
                o.mode.c_str(), (unsigned long long)band.b.half_width,
                (unsigned long long)c.visited_cells);
    std::printf("bootstraps: total %llu (equality %llu, kernel %llu, refresh %llu, preprocessing %llu)\n",
                (unsigned long long)pbs_total, (unsigned long long)c.equality_pbs,
                (unsigned long long)c.kernel_pbs, (unsigned long long)c.refreshes,
                (unsigned long long)pre);
    std::printf("max key variance: %lld eps^2\nwall time: %.3f ms\n", (long long)c.max_key_variance,
                ms);
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  Options o;
  if (const char* env = std::getenv("LEUVEN_BUDGET")) o.budget = std::atof(env);  // cli.cpp:131-147
  for (int i = 1; i < argc; ++i) {
    const std::string k = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) {
        std::fprintf(stderr, "missing value for %s\n", k.c_str());
        std::exit(2);
      }
      return argv[++i];
    };
    if (k == "--a") o.a = val(), o.have_a = true;
    else if (k == "--b") o.b = val(), o.have_b = true;
    else if (k == "--mode") o.mode = val();
    else if (k == "--ell") o.ell = std::atoll(val().c_str());
    else if (k == "--encoding") o.encoding = val();
    else if (k == "--budget") o.budget = std::atof(val().c_str());
    else if (k == "--key-encoding") o.key = val();
    else if (k == "--preprocess") o.preprocess = true;
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
    return run(o);
  } catch (const BandTooNarrow& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 3;
  } catch (const CharNotInAlphabet& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 2;
  } catch (const CharNotInSubset& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 2;
  } catch (const InvalidParams& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 2;
  } catch (const OutOfRangeValue& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 1;
  }
}
