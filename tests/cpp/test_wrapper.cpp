// Reference-shaped C++ tests over include/leuven_b200.hpp, mirroring cases of
// proj/tests/unit/test_backend.cpp and test_kernel.cpp. Exit code = failures.
#include <cstdio>
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

int main() {
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
