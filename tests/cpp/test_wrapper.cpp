// Reference-shaped C++ tests over include/leuven_b200.hpp, mirroring cases of
// proj/tests/unit/test_backend.cpp and test_kernel.cpp. Exit code = failures.
#include <cstdio>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "leuven_b200.hpp"

using namespace leuven;
using namespace leuven::b200;

static int g_fail = 0;
#define CHECK(x)                                                 \
  do {                                                           \
    if (!(x)) {                                                  \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #x);    \
      ++g_fail;                                                  \
    }                                                            \
  } while (0)

template <typename E, typename F>
static bool throws(F f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static EncryptedString enc_ascii(GpuBackend& b, const std::string& s) {
  std::vector<int32_t> v;
  for (char c : s) {
    v.push_back(c & 15);
    v.push_back((c >> 4) & 7);
  }
  EncryptedString e;
  e.symbols = 2;
  if (!v.empty()) e.syms = b.encrypt(v);
  return e;
}

// One golden case per line (written by tests/test_gpu_cpp_wrapper.py from
// tests/golden/reference_runs.json): a, b, mode, ell, encoding, budget,
// key encoding, preprocess, the reference's report_json — tab-separated.
static std::vector<std::vector<std::string>> read_cases(const char* path) {
  std::vector<std::vector<std::string>> out;
  std::ifstream in(path);
  std::string line;
  while (std::getline(in, line)) {
    std::vector<std::string> f;
    std::stringstream ss(line);
    std::string x;
    while (std::getline(ss, x, '\t')) f.push_back(x);
    if (f.size() == 9) out.push_back(f);
  }
  return out;
}

static void pipeline_api(const char* cases_path) {
  using namespace leuven::b200::cli;
  {  // encoding.hpp builtins (encoding.cpp:78-96, 169-190)
    CHECK(AlphabetSpec::ascii7().charset().size() == 128);
    CHECK(AlphabetSpec::lower26().charset().size() == 26);
    CHECK(AlphabetSpec::dna4().charset().size() == 4);
    CHECK(AlphabetSpec::ascii7().symbol_count() == 2 && AlphabetSpec::ascii7().bit_width() == 7);
    CHECK(AlphabetSpec::dna4().code_of('G') == 2);
    CHECK(throws<CharNotInAlphabet>([] { AlphabetSpec::dna4().code_of('X'); }));
    CHECK(throws<InvalidParams>([] { AlphabetSpec::builtin("custom:x"); }));
    for (const AlphabetSpec* a : {&AlphabetSpec::ascii7(), &AlphabetSpec::lower26(), &AlphabetSpec::dna4()})
      for (char c : a->charset()) CHECK(decode_char(encode_char(c, *a), *a) == c);
    const EncodedChar e = encode_char('K', AlphabetSpec::ascii7());  // 75 = 0x4B -> (11, 4)
    CHECK(e.symbols.size() == 2 && e.symbols[0] == 11 && e.symbols[1] == 4);
  }
  GpuBackend be(4000.0, 5);
  {  // encrypt_string / decrypt_string round trip
    const EncryptedString x = encrypt_string("Hello, B200!", AlphabetSpec::ascii7(), be);
    CHECK(x.length() == 12 && x.symbols == 2);
    CHECK(decrypt_string(x, AlphabetSpec::ascii7(), be) == "Hello, B200!");
    CHECK(throws<CharNotInAlphabet>([&] { encrypt_string("ACGU", AlphabetSpec::dna4(), be); }));
  }
  {  // kernel::distance with an Eq9Provider + observer (kernel.hpp:162-199)
    const std::string a = "KID", b = "SIT";
    std::vector<Ct> eqs;
    size_t seen = 0;
    DistanceOptions opt;
    opt.observer = [&](const CellObservation& o) {
      ++seen;
      CHECK(o.key_variance > 0 && o.i >= 1 && o.j >= 1);
    };
    const DistanceRun r = distance(be, [&](size_t i, size_t j) {
      eqs.push_back(be.encrypt(a[i - 1] == b[j - 1] ? 9 : 0));
      return eqs.back();
    }, a.size(), b.size(), BandSpec::exact(3, 3), opt);
    CHECK(be.decrypt(r.score) == 2);
    CHECK(seen == 9 && eqs.size() == 9 && r.counters.kernel_pbs == 9 && r.counters.equality_pbs == 0);
  }
  {  // distance_batch == per-pair distance_encrypted
    const std::vector<std::pair<std::string, std::string>> ps = {{"kitten", "sitting"}, {"", "abc"},
                                                                 {"flaw", "lawn"}};
    std::vector<std::pair<EncryptedString, EncryptedString>> enc;
    std::vector<BandSpec> bands;
    for (const auto& p : ps) {
      enc.push_back({encrypt_string(p.first, AlphabetSpec::ascii7(), be),
                     encrypt_string(p.second, AlphabetSpec::ascii7(), be)});
      bands.push_back(BandSpec::exact(p.first.size(), p.second.size()));
    }
    const std::vector<DistanceRun> rs = distance_batch(be, enc, bands);
    CHECK(rs.size() == 3 && be.decrypt(rs[0].score) == 3 && be.decrypt(rs[1].score) == 3 &&
          be.decrypt(rs[2].score) == 2);
    CHECK(rs[0].counters.kernel_pbs == 42 && rs[0].counters.equality_pbs == 84);
  }
  {  // cli::compute_report / report_json on the compiled reference's cases
    const auto cases = read_cases(cases_path);
    CHECK(cases.size() >= 20);
    std::vector<std::pair<std::string, std::string>> batch_pairs;
    std::vector<std::string> batch_want;
    std::map<double, std::unique_ptr<GpuBackend>> by_budget;
    for (const auto& f : cases) {
      ComputeConfig c;
      c.a = f[0];
      c.b = f[1];
      c.mode = f[2];
      c.has_ell = c.mode == "approx";
      c.ell = std::stoull(f[3]);
      c.encoding = f[4];
      c.budget = std::stod(f[5]);
      c.key_encoding = f[6];
      c.preprocess = f[7] == "1";
      std::unique_ptr<GpuBackend>& b2 = by_budget[c.budget];  // one key set per budget
      if (!b2) b2.reset(new GpuBackend(c.budget, 9));
      const RunReport r = compute_report(c, b2.get());
      const std::string got = report_json(r, false);
      if (got != f[8]) std::printf("report %s | %s\n  got  %s\n  want %s\n", f[0].c_str(), f[1].c_str(),
                                   got.c_str(), f[8].c_str());
      CHECK(got == f[8]);
      CHECK(report_json(r, true).find("\"wall_time_ms\":") != std::string::npos);
      if (c.mode == "exact" && c.encoding == "ascii7" && c.budget == 4000.0 && !c.preprocess &&
          c.key_encoding == "negated") {
        batch_pairs.push_back({c.a, c.b});
        batch_want.push_back(f[8]);
      }
    }
    // the same cases through compute_batch: one wavefront, identical reports
    ComputeConfig base;
    const std::vector<RunReport> rs = compute_batch(batch_pairs, base, &be);
    CHECK(rs.size() == batch_pairs.size() && !rs.empty());
    for (size_t i = 0; i < rs.size(); ++i) CHECK(report_json(rs[i], false) == batch_want[i]);
    CHECK(human_report(compute_report({"KID", "SIT"}, &be)).rfind("distance: 2\n", 0) == 0);
    CHECK(classify_error_exit(BandTooNarrow("x")) == 3 && classify_error_exit(InvalidParams("x")) == 2);
  }
}

int main(int argc, char** argv) {
  if (argc > 1) pipeline_api(argv[1]);
  {
    // test_backend.cpp:202-219 (tight budget, Table-1 x-4 LUT)
    GpuBackend b(25.0);
    Lut16 lut{};
    for (int x = 0; x < 16; ++x) lut[x] = (x - 4 + 16) % 16;
    const Ct out = b.pbs(b.encrypt(5), lut);
    CHECK(b.decrypt(out) == 1);
    CHECK(b.variance(out) == 1);
    CHECK(b.stats().pbs_count == 1);
    Ct noisy = b.trivial(0);
    for (int k = 0; k < 25; ++k) noisy = b.add(noisy, b.encrypt(0));
    CHECK(b.variance(noisy) == 25);
    CHECK(!throws<NoiseBudgetExceeded>([&] { b.pbs(noisy, lut); }));
    noisy = b.add(noisy, b.encrypt(0));
    CHECK(throws<NoiseBudgetExceeded>([&] { b.pbs(noisy, lut); }));
    CHECK(throws<OutOfRangeValue>([&] { b.encrypt(32); }));
    CHECK(throws<ValueOutsideLutHalf>([&] { b.refresh(b.encrypt(16)); }));
  }
  {
    // test_kernel.cpp:230-249 worked examples
    GpuBackend b;
    const EncryptedString x = enc_ascii(b, "monday"), y = enc_ascii(b, "friday");
    const DistanceRun r = distance_encrypted(b, x, y, BandSpec::exact(6, 6));
    CHECK(b.decrypt(r.score) == 3);
    CHECK(r.counters.kernel_pbs == 36);
    CHECK(r.counters.visited_cells == 36);
    CHECK(r.counters.equality_pbs == 72);
    CHECK(r.counters.refreshes == 0);
    const DistanceRun kid = distance_encrypted(b, enc_ascii(b, "KID"), enc_ascii(b, "SIT"),
                                               BandSpec::exact(3, 3));
    CHECK(b.decrypt(kid.score) == 2);
    const DistanceRun same = distance_encrypted(b, enc_ascii(b, "zzzz"), enc_ascii(b, "zzzz"),
                                                BandSpec::skip(4, 4));
    CHECK(b.decrypt(same.score) == 0);
    CHECK(throws<BandTooNarrow>([&] {
      distance_encrypted(b, enc_ascii(b, "abcdef"), enc_ascii(b, "ab"), BandSpec::approx(2));
    }));
  }
  {
    // preprocessing, test_preprocess.cpp:119-134 shape (dna4 single symbol)
    GpuBackend b;
    EncryptedString xs;
    xs.symbols = 1;
    const std::string a = "ACGTTGCA";
    for (char c : a) xs.syms.push_back(b.encrypt(c == 'A' ? 0 : c == 'C' ? 1 : c == 'G' ? 2 : 3));
    uint64_t build = 0;
    EqTable* t = build_eq_table(b, xs, {{'A', {0}}, {'C', {1}}, {'G', {2}}, {'T', {3}}}, &build);
    CHECK(build == 4 * 8);
    CHECK(b.decrypt(t->lookup('G', 3)) == 9);
    CHECK(b.decrypt(t->lookup('G', 4)) == 0);
    CHECK(throws<PositionOutOfRange>([&] { t->lookup('A', 9); }));
    const DistanceRun r = distance_preprocessed(b, *t, "ACGTGCA", BandSpec::exact(8, 7));
    CHECK(b.decrypt(r.score) == 1);
    CHECK(r.counters.equality_pbs == 0);
    CHECK(r.counters.kernel_pbs == 56);
    const std::vector<DistanceRun> scan = distance_preprocessed_batch(
        b, *t, {"ACGTGCA", "ACGTACGT", "T"},
        {BandSpec::exact(8, 7), BandSpec::exact(8, 8), BandSpec::exact(8, 1)});
    CHECK(scan.size() == 3);
    CHECK(b.decrypt(scan[0].score) == 1);
    CHECK(scan[0].counters.kernel_pbs == 56);
    delete t;
  }
  {
    // client / server split: the server evaluates with exported keys only
    GpuBackend client(4000.0, 7);
    const GpuBackend::EvalKeys keys = client.export_keys();
    CHECK(keys.key_id != 7 && keys.key_id != 0);  // a public-key fingerprint, never the seed
    std::unique_ptr<GpuBackend> server = GpuBackend::evaluation(keys);
    CHECK(server->key_id() == keys.key_id);
    CHECK(throws<InvalidParams>([&] { server->encrypt(1); }));
    const std::vector<Ct> xs = client.encrypt(std::vector<int32_t>{3, 12, 20});
    std::vector<uint64_t> rows(xs.size() * 2049), back(xs.size() * 2049);
    check(lv_export(client.raw(), xs.data(), xs.size(), rows.data()));
    std::vector<Ct> on_server(xs.size()), out(xs.size());
    check(lv_import(server->raw(), rows.data(), rows.size() / 2049, on_server.data()));
    const Lut16 minus4 = {12, 13, 14, 15, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11};  // x - 4
    const uint32_t id = server->lut(minus4);
    std::vector<uint32_t> ids(xs.size(), id);
    check(lv_pbs_batch(server->raw(), on_server.data(), ids.data(), xs.size(), out.data()));
    check(lv_export(server->raw(), out.data(), out.size(), back.data()));
    std::vector<Ct> mine(xs.size());
    check(lv_import(client.raw(), back.data(), xs.size(), mine.data()));
    const std::vector<int32_t> got = client.decrypt(mine);
    CHECK(got.size() == 3 && got[0] == 15 && got[1] == 8 && got[2] == 0);  // negacyclic_eval(x - 4)
  }
  std::printf("%s: %d failures\n", g_fail ? "FAILED" : "OK", g_fail);
  return g_fail;
}
