// leuven_b200.hpp — header-only C++ face of the C ABI, shaped like the
// reference's leuven:: API (proj/include/leuven/{backend,encoding,kernel,
// preprocess,cli,errors}.hpp) so reference-style code and tests port line
// for line:
//   leuven::Backend        -> leuven::b200::GpuBackend (handles, not values)
//   AlphabetSpec / encode_char / encrypt_string / decrypt_string (builtins)
//   kernel::distance (Eq9Provider + observer), distance_encrypted,
//   distance_batch (all pairs in one wavefront)
//   preprocess::build_eq_table / distance_preprocessed(_batch)
//   cli::ComputeConfig / RunReport / compute_report / compute_batch /
//   report_json
//   leuven::Error hierarchy -> the same exception types, thrown from status codes
// Link: -L paper_2508_14568_b200/_build -lleuven_b200 (plus -lcudart).
#pragma once

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <stdexcept>
#include <string>
#include <string_view>
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

// ------------------------------------------------------------ encoding
// encoding.hpp:20-74: the three builtin alphabets (the spec-file parser,
// encoding.cpp:108-167, is out of scope). Codes split little-endian over
// the symbol widths.
class AlphabetSpec {
 public:
  static const AlphabetSpec& ascii7() {  // codes 0..127 as a 4-bit + a 3-bit symbol
    static const AlphabetSpec s = make("ascii7", {4, 3}, [](unsigned char u) { return u < 128 ? (int)u : -1; });
    return s;
  }
  static const AlphabetSpec& lower26() {  // 'a'..'z' -> 0..25 as 4-bit + 1-bit
    static const AlphabetSpec s =
        make("lower26", {4, 1}, [](unsigned char u) { return u >= 'a' && u <= 'z' ? u - 'a' : -1; });
    return s;
  }
  static const AlphabetSpec& dna4() {  // A, C, G, T -> 0..3 in one 2-bit symbol
    static const AlphabetSpec s = make("dna4", {2}, [](unsigned char u) {
      const char* a = "ACGT";
      for (int i = 0; i < 4; ++i)
        if (u == (unsigned char)a[i]) return i;
      return -1;
    });
    return s;
  }
  // cli.cpp resolve_alphabet: "ascii7" | "lower26" | "dna4"
  static const AlphabetSpec& builtin(const std::string& name) {
    if (name == "ascii7") return ascii7();
    if (name == "lower26") return lower26();
    if (name == "dna4") return dna4();
    throw InvalidParams("unknown encoding '" + name + "'");
  }
  const std::string& name() const { return name_; }
  const std::vector<int>& symbol_widths() const { return widths_; }
  int bit_width() const { return total_bits_; }
  size_t symbol_count() const { return widths_.size(); }
  bool contains(char c) const { return code_[(unsigned char)c] >= 0; }
  int code_of(char c) const {
    const int v = code_[(unsigned char)c];
    if (v < 0) throw CharNotInAlphabet(std::string("character not in alphabet '") + name_ + "'");
    return v;
  }
  char char_of(int code) const {
    for (char c : chars_)
      if (code_[(unsigned char)c] == code) return c;
    throw OutOfRangeValue("code not in alphabet '" + name_ + "'");
  }
  const std::vector<char>& charset() const { return chars_; }  // code order

 private:
  template <typename F>
  static AlphabetSpec make(std::string name, std::vector<int> widths, F code) {
    AlphabetSpec s;
    s.name_ = std::move(name);
    s.widths_ = std::move(widths);
    for (int w : s.widths_) s.total_bits_ += w;
    std::vector<std::pair<int, char>> by_code;
    for (int u = 0; u < 256; ++u) {
      s.code_[u] = code((unsigned char)u);
      if (s.code_[u] >= 0) by_code.push_back({s.code_[u], (char)u});
    }
    std::sort(by_code.begin(), by_code.end());
    for (const auto& p : by_code) s.chars_.push_back(p.second);
    return s;
  }
  std::string name_;
  std::vector<int> widths_;
  int total_bits_ = 0;
  std::array<int, 256> code_{};
  std::vector<char> chars_;
};

struct EncodedChar {  // encoding.hpp:76-79
  std::vector<int> symbols;
};
inline EncodedChar encode_char(char c, const AlphabetSpec& spec) {  // encoding.cpp:169-178
  int v = spec.code_of(c);
  EncodedChar e;
  for (int w : spec.symbol_widths()) {
    e.symbols.push_back(v & ((1 << w) - 1));
    v >>= w;
  }
  return e;
}
inline char decode_char(const EncodedChar& e, const AlphabetSpec& spec) {
  int v = 0, shift = 0;
  for (size_t k = 0; k < e.symbols.size() && k < spec.symbol_count(); ++k) {
    v |= e.symbols[k] << shift;
    shift += spec.symbol_widths()[k];
  }
  return spec.char_of(v);
}

// encoding.cpp:205-217, one batched encryption for the whole string
inline EncryptedString encrypt_string(std::string_view s, const AlphabetSpec& spec, GpuBackend& be) {
  std::vector<int32_t> v;
  v.reserve(s.size() * spec.symbol_count());
  for (char c : s)
    for (int x : encode_char(c, spec).symbols) v.push_back(x);
  EncryptedString e;
  e.symbols = static_cast<uint32_t>(spec.symbol_count());
  if (!v.empty()) e.syms = be.encrypt(v);
  return e;
}
inline std::string decrypt_string(const EncryptedString& enc, const AlphabetSpec& spec,
                                  const GpuBackend& be) {
  const std::vector<int32_t> v = enc.syms.empty() ? std::vector<int32_t>{} : be.decrypt(enc.syms);
  std::string out;
  for (size_t i = 0; i < enc.length(); ++i) {
    EncodedChar e;
    for (uint32_t k = 0; k < enc.symbols; ++k) e.symbols.push_back(v[i * enc.symbols + k]);
    out.push_back(decode_char(e, spec));
  }
  return out;
}

// ---------------------------------------------------------- traversals
// Every pair's same-index anti-diagonal in one launch (lv_edit_distance_batch).
inline std::vector<DistanceRun> distance_batch(
    GpuBackend& be, const std::vector<std::pair<EncryptedString, EncryptedString>>& pairs,
    const std::vector<BandSpec>& bands, KeyEncoding enc = KeyEncoding::negated) {
  if (bands.size() != pairs.size()) throw InvalidParams("one band per pair");
  uint32_t S = 0;
  for (const auto& p : pairs)
    for (const EncryptedString* e : {&p.first, &p.second}) {
      if (S && e->symbols != S) throw InvalidParams("equality operands must have the same nonzero symbol count");
      S = e->symbols;
    }
  std::vector<Ct> a, b;
  std::vector<uint64_t> aoff(1, 0), boff(1, 0);
  std::vector<lv_band> bb;
  for (size_t p = 0; p < pairs.size(); ++p) {
    a.insert(a.end(), pairs[p].first.syms.begin(), pairs[p].first.syms.end());
    b.insert(b.end(), pairs[p].second.syms.begin(), pairs[p].second.syms.end());
    aoff.push_back(pairs[p].first.length());
    boff.push_back(pairs[p].second.length());
    aoff.back() += aoff[aoff.size() - 2];
    boff.back() += boff[boff.size() - 2];
    bb.push_back(bands[p].b);
  }
  std::vector<lv_ct> scores(pairs.size());
  std::vector<lv_run> runs(pairs.size());
  check(lv_edit_distance_batch(be.raw(), pairs.size(), a.data(), aoff.data(), b.data(), boff.data(),
                               S ? S : 1, bb.data(), static_cast<int32_t>(enc), scores.data(),
                               runs.data()));
  std::vector<DistanceRun> out(pairs.size());
  for (size_t p = 0; p < pairs.size(); ++p) out[p] = DistanceRun{scores[p], runs[p]};
  return out;
}

// kernel.hpp:162-199. Eq9Provider supplies the encrypted 9*[a_i == b_j] of
// cell (i, j), 1-based; it is asked for every in-band cell in the
// reference's visiting order (diagonal, then i) before the wavefront runs.
// The observer sees each cell's schedule — (i, j), its eq9 handle, the
// predicted key variance and the refreshes in front of it — from the same
// symbolic plan the traversal executes; the running dv/dh operands stay on
// the device (updated in place), so they are not part of the observation.
using Eq9Provider = std::function<Ct(size_t, size_t)>;
struct CellObservation {
  size_t i, j;
  Ct eq9;
  int64_t key_variance;
  uint32_t refreshes;  // bit 0: dv refreshed, bit 1: dh refreshed
};
struct DistanceOptions {
  KeyEncoding encoding = KeyEncoding::negated;
  std::function<void(const CellObservation&)> observer;
};
inline DistanceRun distance(GpuBackend& be, const Eq9Provider& eq9_provider, size_t m, size_t n,
                            const BandSpec& band, const DistanceOptions& options = {}) {
  const uint64_t cap = (uint64_t)(m + 1) * (n + 1);
  std::vector<uint32_t> ij(2 * cap), rf(cap);
  std::vector<int64_t> kv(cap);
  uint64_t count = 0;
  lv_run totals{};
  lv_params p;
  check(lv_get_params(be.raw(), &p));
  check(lv_plan_trace(m, n, &band.b, static_cast<int32_t>(options.encoding), p.max_variance_budget,
                      cap, ij.data(), kv.data(), rf.data(), &count, &totals));
  std::vector<Ct> grid(std::max<size_t>(m * n, 1), 0);
  for (uint64_t c = 0; c < count; ++c) {
    const size_t i = ij[2 * c], j = ij[2 * c + 1];
    grid[(i - 1) * n + (j - 1)] = eq9_provider(i, j);
    if (options.observer) options.observer(CellObservation{i, j, grid[(i - 1) * n + (j - 1)], kv[c], rf[c]});
  }
  DistanceRun r{};
  check(lv_edit_distance_eq9(be.raw(), grid.data(), m, n, &band.b,
                             static_cast<int32_t>(options.encoding), &r.score, &r.counters));
  return r;
}

// build_eq_table over the whole alphabet (preprocess.cpp:38-60)
inline EqTable* build_eq_table(GpuBackend& be, const EncryptedString& xs, const AlphabetSpec& spec,
                               uint64_t* build_pbs = nullptr) {
  std::vector<std::pair<char, std::vector<int32_t>>> rows;
  for (char c : spec.charset()) {
    const EncodedChar e = encode_char(c, spec);
    rows.push_back({c, std::vector<int32_t>(e.symbols.begin(), e.symbols.end())});
  }
  return build_eq_table(be, xs, rows, build_pbs);
}

// ----------------------------------------------------------------- cli
namespace cli {

struct ComputeConfig {  // cli.hpp:10-21
  std::string a;
  std::string b;
  std::string mode = "exact";  // exact | skip | approx
  size_t ell = 0;
  bool has_ell = false;
  std::string encoding = "ascii7";  // ascii7 | lower26 | dna4
  double budget = 4000.0;
  std::string key_encoding = "negated";  // negated | original
  bool preprocess = false;
};

struct RunReport {  // cli.hpp:23-37
  int distance = 0;
  std::string mode;
  size_t half_width = 0;
  uint64_t visited_cells = 0;
  uint64_t pbs_total = 0;
  uint64_t pbs_equality = 0;
  uint64_t pbs_kernel = 0;
  uint64_t refresh_count = 0;
  uint64_t preprocessing_pbs = 0;
  int64_t max_key_variance = 0;
  double wall_time_ms = 0.0;
};

inline KeyEncoding resolve_key_encoding(const std::string& s) {
  if (s == "negated") return KeyEncoding::negated;
  if (s == "original") return KeyEncoding::original;
  throw InvalidParams("unknown key encoding '" + s + "'");
}
inline BandSpec resolve_band(const ComputeConfig& c, size_t m, size_t n) {  // cli.cpp:35-51
  if (c.mode == "exact") return BandSpec::exact(m, n);
  if (c.mode == "skip") return BandSpec::skip(m, n);
  if (c.mode == "approx") {
    if (!c.has_ell) throw InvalidParams("--mode approx requires --ell");
    return BandSpec::approx(c.ell);
  }
  throw InvalidParams("unknown mode '" + c.mode + "'");
}

// cli.cpp:53-91 on the GPU backend. `be` (optional) must have been made
// with config.budget; without it a backend with fresh keys is created.
inline RunReport compute_report(const ComputeConfig& config, GpuBackend* be = nullptr) {
  const AlphabetSpec& spec = AlphabetSpec::builtin(config.encoding);
  const BandSpec band = resolve_band(config, config.a.size(), config.b.size());
  const KeyEncoding ke = resolve_key_encoding(config.key_encoding);
  std::unique_ptr<GpuBackend> own;
  if (!be) {
    own.reset(new GpuBackend(config.budget));
    be = own.get();
  }
  const uint64_t pbs0 = be->stats().pbs_count;
  const auto t0 = std::chrono::steady_clock::now();
  DistanceRun run{};
  uint64_t pre = 0;
  std::vector<Ct> temps;
  if (config.preprocess) {
    const EncryptedString xs = encrypt_string(config.a, spec, *be);
    std::unique_ptr<EqTable> table(build_eq_table(*be, xs, spec, &pre));
    run = distance_preprocessed(*be, *table, config.b, band, ke);
    temps = xs.syms;
  } else {
    const EncryptedString xs = encrypt_string(config.a, spec, *be);
    const EncryptedString ys = encrypt_string(config.b, spec, *be);
    run = distance_encrypted(*be, xs, ys, band, ke);
    temps = xs.syms;
    temps.insert(temps.end(), ys.syms.begin(), ys.syms.end());
  }
  const auto t1 = std::chrono::steady_clock::now();
  RunReport r;
  r.distance = be->decrypt(run.score);
  r.mode = config.mode;
  r.half_width = band.b.half_width;
  r.visited_cells = run.counters.visited_cells;
  r.pbs_total = be->stats().pbs_count - pbs0;
  r.pbs_equality = run.counters.equality_pbs;
  r.pbs_kernel = run.counters.kernel_pbs;
  r.refresh_count = run.counters.refreshes;
  r.preprocessing_pbs = pre;
  r.max_key_variance = run.counters.max_key_variance;
  r.wall_time_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  temps.push_back(run.score);
  be->release(temps);
  return r;
}

// Many pairs sharing one config (mode, encoding, budget, key encoding; no
// preprocessing): every pair's anti-diagonals batched into the same
// launches (the batch subcommand's work, cli.cpp:164-210, in one
// wavefront instead of one thread per pair). Reports in input order.
inline std::vector<RunReport> compute_batch(const std::vector<std::pair<std::string, std::string>>& pairs,
                                            const ComputeConfig& base, GpuBackend* be = nullptr) {
  if (base.preprocess) throw InvalidParams("compute_batch: preprocessing runs per pair (compute_report)");
  const AlphabetSpec& spec = AlphabetSpec::builtin(base.encoding);
  const KeyEncoding ke = resolve_key_encoding(base.key_encoding);
  std::unique_ptr<GpuBackend> own;
  if (!be) {
    own.reset(new GpuBackend(base.budget));
    be = own.get();
  }
  std::vector<BandSpec> bands;
  for (const auto& p : pairs) bands.push_back(resolve_band(base, p.first.size(), p.second.size()));
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::pair<EncryptedString, EncryptedString>> enc;
  for (const auto& p : pairs) enc.push_back({encrypt_string(p.first, spec, *be), encrypt_string(p.second, spec, *be)});
  const std::vector<DistanceRun> runs = distance_batch(*be, enc, bands, ke);
  std::vector<Ct> scores;
  for (const auto& r : runs) scores.push_back(r.score);
  const std::vector<int32_t> d = scores.empty() ? std::vector<int32_t>{} : be->decrypt(scores);
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  std::vector<RunReport> out(pairs.size());
  for (size_t p = 0; p < pairs.size(); ++p) {
    const lv_run& c = runs[p].counters;
    RunReport& r = out[p];
    r.distance = d[p];
    r.mode = base.mode;
    r.half_width = bands[p].b.half_width;
    r.visited_cells = c.visited_cells;
    r.pbs_equality = c.equality_pbs;
    r.pbs_kernel = c.kernel_pbs;
    r.refresh_count = c.refreshes;
    r.pbs_total = c.equality_pbs + c.kernel_pbs + c.refreshes;
    r.max_key_variance = c.max_key_variance;
    r.wall_time_ms = ms;
  }
  std::vector<Ct> temps = scores;
  for (const auto& e : enc) {
    temps.insert(temps.end(), e.first.syms.begin(), e.first.syms.end());
    temps.insert(temps.end(), e.second.syms.begin(), e.second.syms.end());
  }
  be->release(temps);
  return out;
}

inline std::string json_escape(const std::string& s) {
  std::string o;
  for (unsigned char c : s) {
    if (c == '"' || c == '\\') {
      o.push_back('\\');
      o.push_back((char)c);
    } else if (c < 0x20) {
      char buf[8];
      std::snprintf(buf, sizeof buf, "\\u%04x", c);
      o += buf;
    } else {
      o.push_back((char)c);
    }
  }
  return o;
}

// cli.cpp:93-107: compact JSON, field order of the reference; timing
// excluded from batch lines so equal inputs serialise to equal bytes.
inline std::string report_json(const RunReport& r, bool include_timing) {
  std::string s = "{\"distance\":" + std::to_string(r.distance) + ",\"mode\":\"" + json_escape(r.mode) +
                  "\",\"half_width\":" + std::to_string(r.half_width) +
                  ",\"visited_cells\":" + std::to_string(r.visited_cells) +
                  ",\"pbs_total\":" + std::to_string(r.pbs_total) +
                  ",\"pbs_equality\":" + std::to_string(r.pbs_equality) +
                  ",\"pbs_kernel\":" + std::to_string(r.pbs_kernel) +
                  ",\"refresh_count\":" + std::to_string(r.refresh_count) +
                  ",\"preprocessing_pbs\":" + std::to_string(r.preprocessing_pbs) +
                  ",\"max_key_variance\":" + std::to_string(r.max_key_variance);
  if (include_timing) {
    char buf[40];  // shortest round-trip form, as the reference's JSON writer
    for (int prec = 1; prec <= 17; ++prec) {
      std::snprintf(buf, sizeof buf, "%.*g", prec, r.wall_time_ms);
      if (std::strtod(buf, nullptr) == r.wall_time_ms) break;
    }
    s += ",\"wall_time_ms\":" + std::string(buf);
  }
  return s + "}";
}

// cli.cpp:110-119
inline std::string human_report(const RunReport& r) {
  char buf[512];
  std::snprintf(buf, sizeof buf,
                "distance: %d\nmode: %s (half-width %zu)\nvisited cells: %llu\n"
                "bootstraps: total %llu (equality %llu, kernel %llu, refresh %llu, preprocessing %llu)\n"
                "max key variance: %lld eps^2\nwall time: %g ms\n",
                r.distance, r.mode.c_str(), r.half_width, (unsigned long long)r.visited_cells,
                (unsigned long long)r.pbs_total, (unsigned long long)r.pbs_equality,
                (unsigned long long)r.pbs_kernel, (unsigned long long)r.refresh_count,
                (unsigned long long)r.preprocessing_pbs, (long long)r.max_key_variance, r.wall_time_ms);
  return buf;
}

// cli.cpp:121-129
inline int classify_error_exit(const std::exception& e) {
  if (dynamic_cast<const BandTooNarrow*>(&e)) return 3;
  if (dynamic_cast<const CharNotInAlphabet*>(&e) || dynamic_cast<const CharNotInSubset*>(&e) ||
      dynamic_cast<const FormatError*>(&e) || dynamic_cast<const InvalidParams*>(&e) ||
      dynamic_cast<const OutOfRangeValue*>(&e))
    return 2;
  return 1;
}

}  // namespace cli

}  // namespace b200
}  // namespace leuven
