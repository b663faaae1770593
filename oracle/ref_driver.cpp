// TEST INFRASTRUCTURE ONLY — extern "C" driver over the reference's own
// simulated backend (/root/reference/proj/src, compiled in place by
// oracle/Makefile into oracle/_ref/libleuven_ref.so; sources are never
// copied). It is the decrypted-value / counter ground truth:
//   - ref_compute re-drives cli::compute_report (proj/src/cli.cpp:53-91),
//     whose translation unit needs the absent vendored CLI11, so the same
//     30 lines of orchestration are restated here over the real library.
//   - ref_trace exposes the per-cell observer hook (kernel.hpp:167-180).
//   - ref_sim_pbs times SimBackend::pbs (backend.cpp:61-70) for the
//     "simulation, no cryptography" CPU figure.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "leuven/backend.hpp"
#include "leuven/encoding.hpp"
#include "leuven/equality.hpp"
#include "leuven/errors.hpp"
#include "leuven/kernel.hpp"
#include "leuven/lut.hpp"
#include "leuven/oracle.hpp"
#include "leuven/preprocess.hpp"

using namespace leuven;

namespace {

thread_local std::string g_err;

int classify(const std::exception& e) {
  if (dynamic_cast<const OutOfRangeValue*>(&e)) return 1;
  if (dynamic_cast<const NoiseBudgetExceeded*>(&e)) return 2;
  if (dynamic_cast<const ValueOutsideLutHalf*>(&e)) return 3;
  if (dynamic_cast<const PackingViolation*>(&e)) return 4;
  if (dynamic_cast<const CharNotInAlphabet*>(&e)) return 5;
  if (dynamic_cast<const CharNotInSubset*>(&e)) return 6;
  if (dynamic_cast<const PositionOutOfRange*>(&e)) return 7;
  if (dynamic_cast<const BandTooNarrow*>(&e)) return 8;
  if (dynamic_cast<const FormatError*>(&e)) return 9;
  if (dynamic_cast<const InvalidParams*>(&e)) return 10;
  return 99;
}

const AlphabetSpec& alphabet(const char* name) {
  std::string s(name);
  if (s == "ascii7") return AlphabetSpec::ascii7();
  if (s == "lower26") return AlphabetSpec::lower26();
  if (s == "dna4") return AlphabetSpec::dna4();
  throw InvalidParams("unknown encoding '" + s + "'");
}

kernel::BandSpec band_of(const char* mode, std::size_t ell, std::size_t m, std::size_t n) {
  std::string s(mode);
  if (s == "exact") return kernel::BandSpec::exact(m, n);
  if (s == "skip") return kernel::BandSpec::skip(m, n);
  if (s == "approx") return kernel::BandSpec::approx(ell);
  throw InvalidParams("unknown mode '" + s + "'");
}

}  // namespace

extern "C" {

struct ref_report {
  int32_t distance;
  uint64_t half_width;
  uint64_t visited_cells;
  uint64_t pbs_total;
  uint64_t pbs_equality;
  uint64_t pbs_kernel;
  uint64_t refresh_count;
  uint64_t preprocessing_pbs;
  int64_t max_key_variance;
  uint64_t linear_ops;
  double wall_time_ms;
};

const char* ref_last_error() { return g_err.c_str(); }

int ref_compute(const char* a, const char* b, const char* mode, uint64_t ell,
                const char* encoding, double budget, int key_negated, int preprocess,
                ref_report* out) {
  try {
    const AlphabetSpec& spec = alphabet(encoding);
    const kernel::BandSpec band = band_of(mode, ell, std::strlen(a), std::strlen(b));
    SimBackend backend(NoiseParams{budget});
    kernel::DistanceOptions options;
    options.encoding = key_negated ? kernel::KeyEncoding::negated : kernel::KeyEncoding::original;
    const auto t0 = std::chrono::steady_clock::now();
    kernel::DistanceRun run;
    uint64_t pre = 0;
    if (preprocess) {
      const EncryptedString xs = encrypt_string(a, spec, backend);
      const StatsSnapshot before = backend.stats();
      const preprocess::EqTable table = preprocess::build_eq_table(backend, xs, spec);
      pre = backend.stats().pbs_count - before.pbs_count;
      run = preprocess::distance_preprocessed(backend, table, b, band, options);
    } else {
      const EncryptedString xs = encrypt_string(a, spec, backend);
      const EncryptedString ys = encrypt_string(b, spec, backend);
      run = kernel::distance_encrypted(backend, xs, ys, band, options);
    }
    const auto t1 = std::chrono::steady_clock::now();
    out->distance = backend.decrypt(run.score);
    out->half_width = band.half_width;
    out->visited_cells = run.visited_cells;
    out->pbs_total = backend.stats().pbs_count;
    out->pbs_equality = run.equality_pbs;
    out->pbs_kernel = run.kernel_pbs;
    out->refresh_count = run.refreshes;
    out->preprocessing_pbs = pre;
    out->max_key_variance = run.max_key_variance;
    out->linear_ops = backend.stats().linear_op_count;
    out->wall_time_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

// Per-cell trace of kernel::distance_encrypted: for every visited cell in
// visiting order, (i, j, key_variance, refreshes issued before it).
int ref_trace(const char* a, const char* b, const char* mode, uint64_t ell,
              const char* encoding, double budget, int key_negated, uint64_t cap,
              uint32_t* ij, int64_t* key_var, uint32_t* refreshes, uint64_t* count) {
  try {
    const AlphabetSpec& spec = alphabet(encoding);
    const kernel::BandSpec band = band_of(mode, ell, std::strlen(a), std::strlen(b));
    SimBackend backend(NoiseParams{budget});
    kernel::DistanceOptions options;
    options.encoding = key_negated ? kernel::KeyEncoding::negated : kernel::KeyEncoding::original;
    uint64_t k = 0;
    uint64_t last_refresh = 0;
    options.observer = [&](const kernel::CellObservation& cell) {
      const uint64_t now = backend.stats().refresh_count;
      if (k < cap) {
        ij[2 * k] = static_cast<uint32_t>(cell.i);
        ij[2 * k + 1] = static_cast<uint32_t>(cell.j);
        key_var[k] = cell.key_variance;
        refreshes[k] = static_cast<uint32_t>(now - last_refresh);
      }
      last_refresh = now;
      ++k;
    };
    const EncryptedString xs = encrypt_string(a, spec, backend);
    const EncryptedString ys = encrypt_string(b, spec, backend);
    (void)kernel::distance_encrypted(backend, xs, ys, band, options);
    *count = k;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

int ref_negacyclic_eval(const int32_t* entries, int32_t x, int32_t* out) {
  try {
    Lut16 lut;
    for (int i = 0; i < 16; ++i) lut.entries[static_cast<std::size_t>(i)] = entries[i];
    *out = negacyclic_eval(lut, x);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

int ref_lut(const char* which, int32_t arg, int32_t* out16) {
  try {
    std::string w(which);
    Lut16 lut;
    if (w == "minlut-original")
      lut = kernel::build_min_lut(kernel::KeyEncoding::original);
    else if (w == "minlut-negated")
      lut = kernel::build_min_lut(kernel::KeyEncoding::negated);
    else if (w == "eqlut")
      lut = equality::eq_lut(arg);
    else if (w == "identity")
      lut = identity_lut();
    else
      throw InvalidParams("unknown table");
    for (int i = 0; i < 16; ++i) out16[i] = lut.entries[static_cast<std::size_t>(i)];
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

int ref_wf_distance(const char* a, const char* b) { return oracle::wf_distance(a, b).distance; }

int ref_banded_distance(const char* a, const char* b, uint64_t hw, int32_t* out) {
  try {
    *out = oracle::banded_distance(a, b, hw);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

uint64_t ref_band_cell_count(uint64_t m, uint64_t ell) { return kernel::band_cell_count(m, ell); }

int ref_eq_cost(const char* technique, int32_t bits, int32_t* out) {
  try {
    const std::string t(technique);
    const equality::EqTechnique tech = t == "standard_2bit" ? equality::EqTechnique::standard_2bit
                                       : t == "ours_4bit"   ? equality::EqTechnique::ours_4bit
                                                            : equality::EqTechnique::combined;
    *out = equality::eq_cost(tech, bits);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  }
}

// cfg2 on the simulated backend: `count` fresh encryptions through
// SimBackend::pbs with the identity table, `threads` workers each with its
// own backend (the reference's batch model, cli.cpp:194-207). Returns the
// wall time in seconds and writes the decrypted outputs.
double ref_sim_pbs(const int32_t* values, uint64_t count, int threads, int32_t* out) {
  if (threads < 1) threads = 1;
  const Lut16 lut = identity_lut();
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      SimBackend backend;
      const uint64_t lo = count * t / threads, hi = count * (t + 1) / threads;
      for (uint64_t i = lo; i < hi; ++i)
        out[i] = backend.decrypt(backend.pbs(backend.encrypt(values[i]), lut));
    });
  }
  for (auto& th : pool) th.join();
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// A batch of compute_report calls (cfg5-style), one pair per worker thread
// like cli::run_batch (cli.cpp:164-210). Returns wall seconds.
double ref_compute_batch(const char* const* as, const char* const* bs, uint64_t count,
                         int threads, int32_t* distances) {
  if (threads < 1) threads = 1;
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      for (uint64_t i = t; i < count; i += threads) {
        ref_report r{};
        distances[i] = ref_compute(as[i], bs[i], "exact", 0, "ascii7", 4000.0, 1, 0, &r) == 0
                           ? r.distance
                           : -1;
      }
    });
  }
  for (auto& th : pool) th.join();
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // extern "C"
