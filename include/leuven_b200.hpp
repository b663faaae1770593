// leuven_b200.hpp — header-only C++ face of the C ABI, shaped like the
// reference's leuven:: API (proj/include/leuven/{backend,kernel,preprocess,
// errors}.hpp) so reference-style code and tests port line for line:
//   leuven::Backend        -> leuven::b200::GpuBackend (handles, not values)
//   kernel::distance_encrypted / preprocess::build_eq_table /
//   preprocess::distance_preprocessed -> free functions below
//   leuven::Error hierarchy -> the same exception types, thrown from status codes
// Link: -L paper_2508_14568_b200/_build -lleuven_b200 (plus -lcudart).
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <memory>
#include <random>
#include <vector>

#include "leuven_b200.h"

namespace leuven {

// errors.hpp:8-39
struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct OutOfRangeValue : Error { using Error::Error; };
struct NoiseBudgetExceeded : Error { using Error::Error; };
struct ValueOutsideLutHalf : Error { using Error::Error; };
struct PackingViolation : Error { using Error::Error; };
struct CharNotInAlphabet : Error { using Error::Error; };
struct CharNotInSubset : Error { using Error::Error; };
struct PositionOutOfRange : Error { using Error::Error; };
struct BandTooNarrow : Error { using Error::Error; };
struct FormatError : Error { using Error::Error; };
struct InvalidParams : Error { using Error::Error; };
struct DeviceError : Error { using Error::Error; };

namespace b200 {

inline void check(int rc) {
  if (rc == LV_OK) return;
  const std::string m = lv_last_error();
  switch (rc) {
    case LV_ERR_OUT_OF_RANGE: throw OutOfRangeValue(m);
    case LV_ERR_NOISE_BUDGET: throw NoiseBudgetExceeded(m);
    case LV_ERR_VALUE_OUTSIDE_LUT_HALF: throw ValueOutsideLutHalf(m);
    case LV_ERR_PACKING: throw PackingViolation(m);
    case LV_ERR_CHAR_NOT_IN_ALPHABET: throw CharNotInAlphabet(m);
    case LV_ERR_CHAR_NOT_IN_SUBSET: throw CharNotInSubset(m);
    case LV_ERR_POSITION_OUT_OF_RANGE: throw PositionOutOfRange(m);
    case LV_ERR_BAND_TOO_NARROW: throw BandTooNarrow(m);
    case LV_ERR_FORMAT: throw FormatError(m);
    case LV_ERR_INVALID_PARAMS: throw InvalidParams(m);
    default: throw DeviceError(m);
  }
}

using Lut16 = std::array<int32_t, 16>;  // lut.hpp:22-24
using Ct = lv_ct;

struct StatsSnapshot {  // backend.hpp:36-40
  uint64_t pbs_count, refresh_count, linear_op_count;
};

// The GPU backend: same operations as leuven::Backend (backend.hpp:54-76),
// each also available in batched form.
// Key seeds default to OS entropy; pass a fixed seed only for tests and
// reproducible experiments (every secret derives from it).
inline uint64_t random_seed() {
  std::random_device rd;
  return ((uint64_t)rd() << 32) ^ rd();
}

class GpuBackend {
 public:
  // exact_mask_product: see lv_params (noise of exact products, 1.4x time)
  explicit GpuBackend(double budget = 4000.0, uint64_t seed = random_seed(),
                      bool exact_mask_product = false) {
    lv_params p;
    lv_default_params(&p);
    p.max_variance_budget = budget;
    p.exact_mask_product = exact_mask_product ? 1u : 0u;
    check(lv_ctx_create(&p, seed, &ctx_));
  }
  // key-set fingerprint (hash of the public KSK + parameters; lv_ctx_key_id)
  uint64_t key_id() const {
    uint64_t k = 0;
    check(lv_ctx_key_id(ctx_, &k));
    return k;
  }
  ~GpuBackend() { lv_ctx_destroy(ctx_); }
  GpuBackend(const GpuBackend&) = delete;
  GpuBackend& operator=(const GpuBackend&) = delete;

  // Client / server split: the evaluation keys of a secret-holding backend
  // (lv_keys_export) and a server backend built from them, which has no
  // secret key (encrypt/decrypt throw InvalidParams).
  struct EvalKeys {
    std::vector<uint64_t> bsk, ksk;
    uint64_t key_id = 0;
  };
  EvalKeys export_keys() const {
    lv_params p;
    check(lv_get_params(ctx_, &p));
    uint64_t nb = 0, nk = 0;
    check(lv_keys_size(&p, &nb, &nk));
    EvalKeys k;
    k.bsk.resize(nb);
    k.ksk.resize(nk);
    check(lv_keys_export(ctx_, k.bsk.data(), k.ksk.data(), &k.key_id));
    return k;
  }
  static std::unique_ptr<GpuBackend> evaluation(const EvalKeys& k, double budget = 4000.0,
                                                bool exact_mask_product = false) {
    lv_params p;
    lv_default_params(&p);
    p.max_variance_budget = budget;
    p.exact_mask_product = exact_mask_product ? 1u : 0u;
    uint64_t nb = 0, nk = 0;
    check(lv_keys_size(&p, &nb, &nk));
    if (k.bsk.size() != nb || k.ksk.size() != nk)
      throw InvalidParams("evaluation keys have the wrong size");
    lv_ctx* c = nullptr;
    check(lv_ctx_create_eval(&p, k.bsk.data(), k.ksk.data(), k.key_id, &c));
    return std::unique_ptr<GpuBackend>(new GpuBackend(c));
  }

  lv_ctx* raw() const { return ctx_; }

  Ct encrypt(int v) { return one(&lv_encrypt, v); }
  Ct trivial(int v) { return one(&lv_trivial, v); }
  int decrypt(Ct c) const {
    int32_t out;
    check(lv_decrypt(ctx_, &c, 1, &out));
    return out;
  }
  std::vector<Ct> encrypt(const std::vector<int32_t>& vs) {
    std::vector<Ct> out(vs.size());
    check(lv_encrypt(ctx_, vs.data(), vs.size(), out.data()));
    return out;
  }
  std::vector<int32_t> decrypt(const std::vector<Ct>& cs) const {
    std::vector<int32_t> out(cs.size());
    check(lv_decrypt(ctx_, cs.data(), cs.size(), out.data()));
    return out;
  }
  Ct add(Ct a, Ct b) { return two(&lv_add, a, b); }
  Ct sub(Ct a, Ct b) { return two(&lv_sub, a, b); }
  Ct scalar_mul(Ct a, int k) { return scal(&lv_scalar_mul, a, k); }
  Ct scalar_add(Ct a, int k) { return scal(&lv_scalar_add, a, k); }
  uint32_t lut(const Lut16& e) {
    uint32_t id;
    check(lv_lut_upload(ctx_, e.data(), &id));
    return id;
  }
  Ct pbs(Ct x, const Lut16& table) {
    const uint32_t id = lut(table);
    Ct out;
    check(lv_pbs_batch(ctx_, &x, &id, 1, &out));
    return out;
  }
  std::vector<Ct> pbs(const std::vector<Ct>& xs, const std::vector<uint32_t>& ids) {
    std::vector<Ct> out(xs.size());
    check(lv_pbs_batch(ctx_, xs.data(), ids.data(), xs.size(), out.data()));
    return out;
  }
  Ct refresh(Ct x) {
    Ct out;
    check(lv_refresh_batch(ctx_, &x, 1, &out));
    return out;
  }
  int64_t predict_variance(const std::vector<std::pair<Ct, int>>& terms) const {
    std::vector<Ct> c;
    std::vector<int32_t> k;
    for (const auto& t : terms) {
      c.push_back(t.first);
      k.push_back(t.second);
    }
    int64_t v;
    check(lv_predict_variance(ctx_, c.data(), k.data(), c.size(), &v));
    return v;
  }
  int64_t variance(Ct c) const {
    int64_t v;
    check(lv_ledger_variance(ctx_, &c, 1, &v));
    return v;
  }
  StatsSnapshot stats() const {
    lv_stats s;
    check(lv_get_stats(ctx_, &s));
    return {s.pbs_count, s.refresh_count, s.linear_op_count};
  }
  void release(const std::vector<Ct>& cs) { check(lv_release(ctx_, cs.data(), cs.size())); }

 private:
  explicit GpuBackend(lv_ctx* c) : ctx_(c) {}
  template <typename F>
  Ct one(F f, int v) {
    int32_t x = v;
    Ct out;
    check(f(ctx_, &x, 1, &out));
    return out;
  }
  template <typename F>
  Ct two(F f, Ct a, Ct b) {
    Ct out;
    check(f(ctx_, &a, &b, 1, &out));
    return out;
  }
  template <typename F>
  Ct scal(F f, Ct a, int k) {
    int32_t kk = k;
    Ct out;
    check(f(ctx_, &a, &kk, 1, &out));
    return out;
  }
  lv_ctx* ctx_ = nullptr;
};

// kernel.hpp:47-72 / 182-190
enum class KeyEncoding { original = LV_KEY_ORIGINAL, negated = LV_KEY_NEGATED };

struct BandSpec {
  lv_band b{};
  static BandSpec exact(uint64_t m, uint64_t n) { return make(LV_BAND_EXACT, 0, m, n); }
  static BandSpec skip(uint64_t m, uint64_t n) { return make(LV_BAND_SKIP, 0, m, n); }
  static BandSpec approx(uint64_t ell) { return make(LV_BAND_APPROX, ell, 0, 0); }

 private:
  static BandSpec make(int mode, uint64_t ell, uint64_t m, uint64_t n) {
    BandSpec s;
    check(lv_band_resolve(mode, ell, m, n, &s.b));
    return s;
  }
};

struct DistanceRun {
  Ct score;
  lv_run counters;
};

// An encrypted string: chars[i * symbols + k] = k-th symbol of char i
// (encoding.hpp:80-84, flattened).
struct EncryptedString {
  std::vector<Ct> syms;
  uint32_t symbols = 1;
  size_t length() const { return symbols ? syms.size() / symbols : 0; }
};

inline DistanceRun distance_encrypted(GpuBackend& be, const EncryptedString& a,
                                      const EncryptedString& b, const BandSpec& band,
                                      KeyEncoding enc = KeyEncoding::negated) {
  DistanceRun r{};
  check(lv_edit_distance_ee(be.raw(), a.syms.data(), a.length(), b.syms.data(), b.length(),
                            a.symbols, &band.b, static_cast<int32_t>(enc), &r.score, &r.counters));
  return r;
}

class EqTable {  // preprocess.hpp:18-39
 public:
  EqTable(GpuBackend& be, lv_eqtable* t) : be_(&be), t_(t) {}
  ~EqTable() { lv_eq_table_destroy(be_->raw(), t_); }
  EqTable(const EqTable&) = delete;
  EqTable& operator=(const EqTable&) = delete;
  Ct lookup(char c, uint64_t position) const {
    Ct out;
    check(lv_eq_table_lookup(be_->raw(), t_, c, position, &out));
    return out;
  }
  lv_eqtable* raw() const { return t_; }

 private:
  GpuBackend* be_;
  lv_eqtable* t_;
};

// rows: (character, its plaintext symbols) for every table row
inline EqTable* build_eq_table(GpuBackend& be, const EncryptedString& xs,
                               const std::vector<std::pair<char, std::vector<int32_t>>>& rows,
                               uint64_t* build_pbs = nullptr) {
  std::string chars;
  std::vector<int32_t> syms;
  for (const auto& r : rows) {
    chars.push_back(r.first);
    syms.insert(syms.end(), r.second.begin(), r.second.end());
  }
  lv_eqtable* t = nullptr;
  check(lv_eq_table_build(be.raw(), xs.syms.data(), xs.length(), xs.symbols, chars.data(),
                          syms.data(), rows.size(), &t, build_pbs));
  return new EqTable(be, t);
}

inline DistanceRun distance_preprocessed(GpuBackend& be, const EqTable& table,
                                         const std::string& plain, const BandSpec& band,
                                         KeyEncoding enc = KeyEncoding::negated) {
  DistanceRun r{};
  check(lv_edit_distance_pre(be.raw(), table.raw(), plain.data(), plain.size(), &band.b,
                             static_cast<int32_t>(enc), &r.score, &r.counters));
  return r;
}

// One table against many plaintext strings, all anti-diagonals batched
// (lv_edit_distance_pre_batch): the database-scan use of a preprocessed query.
inline std::vector<DistanceRun> distance_preprocessed_batch(
    GpuBackend& be, const EqTable& table, const std::vector<std::string>& plains,
    const std::vector<BandSpec>& bands, KeyEncoding enc = KeyEncoding::negated) {
  if (bands.size() != plains.size()) throw InvalidParams("one band per plaintext string");
  std::string data;
  std::vector<uint64_t> off(1, 0);
  std::vector<const lv_eqtable*> tables(plains.size(), table.raw());
  std::vector<lv_band> b;
  for (size_t p = 0; p < plains.size(); ++p) {
    data += plains[p];
    off.push_back(data.size());
    b.push_back(bands[p].b);
  }
  std::vector<lv_ct> scores(plains.size());
  std::vector<lv_run> runs(plains.size());
  check(lv_edit_distance_pre_batch(be.raw(), plains.size(), tables.data(), data.data(), off.data(),
                                   b.data(), static_cast<int32_t>(enc), scores.data(), runs.data()));
  std::vector<DistanceRun> out(plains.size());
  for (size_t p = 0; p < plains.size(); ++p) out[p] = DistanceRun{scores[p], runs[p]};
  return out;
}

}  // namespace b200
}  // namespace leuven
