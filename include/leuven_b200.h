/*
 * leuven_b200.h — C ABI of the B200-native TFHE PBS path behind Leuvenshtein.
 *
 * Drop-in boundary for the reference's leuven::Backend extension point
 * (proj/include/leuven/backend.hpp:45-77, "an adapter over a real scheme ...
 * would keep the same surface") and the traversal/preprocessing entry
 * points that consume it. The reference passes SimCiphertext by value
 * (backend.hpp:17-20); a real backend keeps ciphertexts resident in HBM, so
 * here a ciphertext is an opaque handle (lv_ct) into a device pool, with its
 * host-side NoiseLedger (proj/include/leuven/noise.hpp:19-51) tracked by the
 * library exactly as SimBackend tracks it.
 *
 * Every function returns an lv_status; LV_OK is 0 and the nonzero codes map
 * one-to-one onto the reference's exception types (errors.hpp:8-39). The
 * message of the last failure on the calling thread is lv_last_error().
 * Plain C types only; no torch, no C++ in the signatures.
 */
#ifndef LEUVEN_B200_H
#define LEUVEN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LV_ABI_VERSION 1

typedef enum {
  LV_OK = 0,
  LV_ERR_OUT_OF_RANGE = 1,            /* OutOfRangeValue        errors.hpp:13 */
  LV_ERR_NOISE_BUDGET = 2,            /* NoiseBudgetExceeded    errors.hpp:19 */
  LV_ERR_VALUE_OUTSIDE_LUT_HALF = 3,  /* ValueOutsideLutHalf    errors.hpp:22 */
  LV_ERR_PACKING = 4,                 /* PackingViolation       errors.hpp:26 */
  LV_ERR_CHAR_NOT_IN_ALPHABET = 5,    /* CharNotInAlphabet      errors.hpp:28 */
  LV_ERR_CHAR_NOT_IN_SUBSET = 6,      /* CharNotInSubset        errors.hpp:29 */
  LV_ERR_POSITION_OUT_OF_RANGE = 7,   /* PositionOutOfRange     errors.hpp:30 */
  LV_ERR_BAND_TOO_NARROW = 8,         /* BandTooNarrow          errors.hpp:33 */
  LV_ERR_FORMAT = 9,                  /* FormatError            errors.hpp:36 */
  LV_ERR_INVALID_PARAMS = 10,         /* InvalidParams          errors.hpp:39 */
  LV_ERR_CUDA = 20,                   /* device / driver failure (new)      */
  LV_ERR_INVALID_HANDLE = 21          /* unknown or released lv_ct (new)    */
} lv_status;

/* Parameter set. Only the cryptographic fields marked (fixed) must equal
 * the compiled kernel constants (N=2048, k=1, 2^23 x 1 BSK gadget, 2^3 x 5
 * KSK gadget); n, the noise bounds and the budget are free. */
typedef struct {
  uint32_t n;                 /* small LWE dimension (default 880)          */
  uint32_t N;                 /* (fixed) 2048                                */
  uint32_t k;                 /* (fixed) 1                                   */
  uint32_t pbs_base_log;      /* (fixed) 23                                  */
  uint32_t pbs_level;         /* (fixed) 1                                   */
  uint32_t ks_base_log;       /* (fixed) 3                                   */
  uint32_t ks_level;          /* (fixed) 5                                   */
  uint32_t lwe_noise_log2;    /* TUniform bound, small-key LWE (KSK) noise   */
  uint32_t glwe_noise_log2;   /* TUniform bound, GLWE / fresh big-key noise  */
  double max_variance_budget; /* NoiseParams::max_variance_budget, backend.hpp:23-34 */
  uint32_t exact_mask_product; /* 0: one f64 FFT product per external-product output
                                * (default); 1: the mask output splits the BSK as
                                * H 2^43 + Lo with an exactly rounded H product, so
                                * the FFT adds no key-amplified noise (phase-noise
                                * variance within 1.001x of exact integer products;
                                * 1.4x blind-rotation time). DESIGN.md §2.
                                * 2: noise measurement only — the reference's
                                * algorithm (TFHE-rs f64-FFT PBS): the BSK spectrum
                                * is the plain f64 transform of the rounded torus
                                * coefficients instead of our double-double one. */
  int32_t device;              /* CUDA device of the context; -1 (default): the
                                * calling thread's current device */
} lv_params;

typedef struct lv_ctx lv_ctx;
typedef uint32_t lv_ct;
typedef struct lv_eqtable lv_eqtable;

typedef struct {          /* StatsSnapshot, backend.hpp:36-40 */
  uint64_t pbs_count;
  uint64_t refresh_count;
  uint64_t linear_op_count;
} lv_stats;

typedef enum { LV_BAND_EXACT = 0, LV_BAND_SKIP = 1, LV_BAND_APPROX = 2 } lv_band_mode;
typedef enum { LV_KEY_ORIGINAL = 0, LV_KEY_NEGATED = 1 } lv_key_encoding;

typedef struct {          /* kernel::BandSpec, kernel.hpp:47-72 */
  int32_t mode;           /* lv_band_mode                              */
  uint64_t half_width;    /* resolved half width (see lv_band_resolve) */
} lv_band;

typedef struct {          /* kernel::DistanceRun, kernel.hpp:182-190 */
  uint64_t visited_cells;
  uint64_t equality_pbs;
  uint64_t kernel_pbs;
  uint64_t refreshes;
  int64_t max_key_variance;
  uint64_t waves;         /* new: anti-diagonal launches issued           */
} lv_run;

/* ---- lifecycle (new surface: the reference has no keys) ---------------- */
void lv_default_params(lv_params* out);
/* Generates secret keys, KSK and BSK on the device from `seed` (Philox). */
int lv_ctx_create(const lv_params* params, uint64_t seed, lv_ctx** out);
void lv_ctx_destroy(lv_ctx* ctx);
/* Client / server split (new surface). A context made by lv_ctx_create
 * holds the secret keys; lv_keys_export copies its evaluation keys to host
 * buffers of lv_keys_size words — the BSK in the standard domain,
 * [i < n][row < 2][poly < 2][N] u64 (GGSW rows of s_i under the GLWE key),
 * and the KSK [j < N][level < 5][n + 1] u64 — plus the key-set id that
 * LEQT tables carry: a fingerprint of the public KSK and the parameter set,
 * never the generating seed (a server given a non-zero key_id that does not
 * match the keys it received fails with LV_ERR_INVALID_PARAMS). lv_ctx_create_eval builds an
 * evaluation-only context from them (the Fourier BSK is computed on the
 * device): every homomorphic entry point works, while lv_encrypt,
 * lv_decrypt, lv_phase and the secret parts of lv_debug_keys fail with
 * LV_ERR_INVALID_PARAMS, and lv_refresh_batch skips the plaintext-range
 * check it cannot perform. Ciphertexts move between the two contexts with
 * lv_export / lv_import; results are bit-identical to the client's own. */
int lv_keys_size(const lv_params* params, uint64_t* bsk_count, uint64_t* ksk_count);
int lv_keys_export(lv_ctx* ctx, uint64_t* bsk, uint64_t* ksk, uint64_t* key_id);
int lv_ctx_create_eval(const lv_params* params, const uint64_t* bsk, const uint64_t* ksk,
                       uint64_t key_id, lv_ctx** out);
/* The key-set fingerprint of any context (client or server). */
int lv_ctx_key_id(lv_ctx* ctx, uint64_t* key_id);
const char* lv_last_error(void);
int lv_abi_version(void);

/* The product's own lookup tables (the ones it bootstraps with), for the
 * CLI `table` dump / pybind lut_dump (cli.cpp:212-228, module.cpp:97-106):
 * build_min_lut (kernel.cpp:64-72) in both key encodings and eq_lut(1|9)
 * (equality.cpp:31-36). */
typedef enum {
  LV_TABLE_MINLUT_ORIGINAL = 0,
  LV_TABLE_MINLUT_NEGATED = 1,
  LV_TABLE_EQLUT = 2,
  LV_TABLE_EQLUT9 = 3
} lv_table;
int lv_lut_table(int32_t which, int32_t* out16);

/* ---- Backend (backend.hpp:54-76) ---------------------------------------- */
int lv_encrypt(lv_ctx* ctx, const int32_t* values, size_t count, lv_ct* out);   /* encrypt :54 */
int lv_trivial(lv_ctx* ctx, const int32_t* values, size_t count, lv_ct* out);   /* trivial :55 */
int lv_decrypt(lv_ctx* ctx, const lv_ct* cts, size_t count, int32_t* out);      /* decrypt :56 */
int lv_add(lv_ctx* ctx, const lv_ct* a, const lv_ct* b, size_t count, lv_ct* out);       /* :58 */
int lv_sub(lv_ctx* ctx, const lv_ct* a, const lv_ct* b, size_t count, lv_ct* out);       /* :59 */
int lv_scalar_mul(lv_ctx* ctx, const lv_ct* a, const int32_t* k, size_t count, lv_ct* out); /* :60 */
int lv_scalar_add(lv_ctx* ctx, const lv_ct* a, const int32_t* k, size_t count, lv_ct* out); /* :61 */
/* Registers a Lut16 (lut.hpp:22-24); identical tables share one id. */
int lv_lut_upload(lv_ctx* ctx, const int32_t entries[16], uint32_t* lut_id);
/* Batched Backend::pbs (:63-65): out[i] = PBS(in[i], lut_ids[i]). Throws
 * (returns) LV_ERR_NOISE_BUDGET before any work if an input ledger exceeds
 * the budget, as SimBackend::pbs does per call (backend.cpp:61-67). */
int lv_pbs_batch(lv_ctx* ctx, const lv_ct* in, const uint32_t* lut_ids, size_t count, lv_ct* out);
/* Batched Backend::refresh (:69): identity PBS, values must be in [0,16). */
int lv_refresh_batch(lv_ctx* ctx, const lv_ct* in, size_t count, lv_ct* out);
/* Backend::predict_variance (:73): variance of sum coeffs[i]*cts[i]. */
int lv_predict_variance(lv_ctx* ctx, const lv_ct* cts, const int32_t* coeffs, size_t count,
                        int64_t* out);
int lv_get_stats(lv_ctx* ctx, lv_stats* out);                                    /* stats :75 */
int lv_get_params(lv_ctx* ctx, lv_params* out);                                  /* params :76 */

/* ---- handles and raw ciphertext I/O (new) ------------------------------- */
int lv_release(lv_ctx* ctx, const lv_ct* cts, size_t count);
int lv_ledger_variance(lv_ctx* ctx, const lv_ct* cts, size_t count, int64_t* out);
/* Raw big-key LWE rows, (N+1) u64 each (mask then body). */
int lv_export(lv_ctx* ctx, const lv_ct* cts, size_t count, uint64_t* host);
/* Imports rows as fresh ciphertexts (ledger = one new source). */
int lv_import(lv_ctx* ctx, const uint64_t* host, size_t count, lv_ct* out);
int lv_phase(lv_ctx* ctx, const lv_ct* cts, size_t count, uint64_t* out);

/* End-to-end batched PBS on HOST buffers (count rows of N+1 u64 in/out):
 * H2D, key switch, blind rotation, sample extract, D2H. Counts as `count`
 * bootstraps; no handles are created. */
int lv_pbs_batch_host(lv_ctx* ctx, const uint64_t* in, const uint32_t* lut_ids, size_t count,
                      uint64_t* out);

/* ---- traversal (kernel.hpp:197-212, preprocess.hpp:45-53) ------------- */
/* Resolves BandSpec::exact/skip/approx(ell) for lengths m, n. */
int lv_band_resolve(int32_t mode, uint64_t ell, uint64_t m, uint64_t n, lv_band* out);
/* distance_encrypted: a, b are m resp. n characters of `symbols` symbol
 * ciphertexts each (a[i*symbols + k] = k-th symbol of char i). The folded
 * equality circuit (equality.cpp:59-70) runs as a batched pre-pass per
 * anti-diagonal; every cell of a diagonal is one PBS launch. */
int lv_edit_distance_ee(lv_ctx* ctx, const lv_ct* a, size_t m, const lv_ct* b, size_t n,
                        uint32_t symbols, const lv_band* band, int32_t key_encoding,
                        lv_ct* score, lv_run* run);
/* Many independent pairs, all pairs' same-index diagonals in one launch
 * (the B200 form of cli.cpp:164-210 batch mode). Offsets are in characters:
 * pair p uses a[a_off[p]*symbols ...], length a_off[p+1]-a_off[p]. */
int lv_edit_distance_batch(lv_ctx* ctx, size_t pairs, const lv_ct* a, const uint64_t* a_off,
                           const lv_ct* b, const uint64_t* b_off, uint32_t symbols,
                           const lv_band* bands, int32_t key_encoding, lv_ct* scores,
                           lv_run* runs);
/* preprocess::build_eq_table (preprocess.cpp:38-60). rows x symbols plaintext
 * symbol values (row r = character chars[r]); one table row per character. */
int lv_eq_table_build(lv_ctx* ctx, const lv_ct* a, size_t m, uint32_t symbols,
                      const char* chars, const int32_t* char_symbols, size_t rows,
                      lv_eqtable** out, uint64_t* build_pbs);
int lv_eq_table_lookup(lv_ctx* ctx, const lv_eqtable* t, char c, uint64_t position, lv_ct* out);
/* LEQT v2 container (the reference's v1, preprocess.cpp:80-194, with real
 * LWE rows): meta = the caller's alphabet section, stored verbatim. Pass
 * buf = NULL to get the size. Loading checks magic/version (FormatError),
 * truncation (FormatError) and that the rows were encrypted under this
 * context's keyset (InvalidParams); ledgers get fresh source ids. */
int lv_eq_table_serialize(lv_ctx* ctx, const lv_eqtable* t, const uint8_t* meta, uint64_t meta_len,
                          uint8_t* buf, uint64_t cap, uint64_t* len);
int lv_eq_table_deserialize(lv_ctx* ctx, const uint8_t* buf, uint64_t len, lv_eqtable** out,
                            uint8_t* meta_out, uint64_t meta_cap, uint64_t* meta_len);
void lv_eq_table_destroy(lv_ctx* ctx, lv_eqtable* t);
/* preprocess::distance_preprocessed (preprocess.cpp:62-76). */
int lv_edit_distance_pre(lv_ctx* ctx, const lv_eqtable* t, const char* plain, size_t n,
                         const lv_band* band, int32_t key_encoding, lv_ct* score, lv_run* run);
/* Many plaintext strings against their tables in one wavefront (the
 * database-scan use of one preprocessed query):
 * string p = plains[plain_off[p] .. plain_off[p+1]) against tables[p]
 * (tables may repeat). Every pair's same-index anti-diagonal shares one
 * launch; scores/runs as lv_edit_distance_pre per pair. */
int lv_edit_distance_pre_batch(lv_ctx* ctx, size_t npairs, const lv_eqtable* const* tables,
                               const char* plains, const uint64_t* plain_off,
                               const lv_band* bands, int32_t key_encoding, lv_ct* scores,
                               lv_run* runs);

/* kernel::distance with a caller-supplied Eq9Provider (kernel.hpp:162-199):
 * eq9[(i-1) n + (j-1)] is the encrypted scaled equality bit of cell (i, j);
 * only the in-band cells' handles are read (and must be valid); they stay
 * owned by the caller. */
int lv_edit_distance_eq9(lv_ctx* ctx, const lv_ct* eq9, uint64_t m, uint64_t n,
                         const lv_band* band, int32_t key_encoding, lv_ct* score, lv_run* run);

/* Symbolic schedule of a traversal (no device work): per visited cell
 * (i, j, key variance, refreshes before it) — the observer hook of
 * kernel.hpp:167-180 for tests and planning. */
int lv_plan_trace(uint64_t m, uint64_t n, const lv_band* band, int32_t key_encoding,
                  double budget, uint64_t cap, uint32_t* ij, int64_t* key_var,
                  uint32_t* refreshes, uint64_t* count, lv_run* totals);

/* ---- parity / debug entry points --------------------------------------- */
/* Key material copied to host (sizes as in DESIGN.md §3). */
int lv_debug_keys(lv_ctx* ctx, uint8_t* sk_small, uint8_t* sk_glwe, uint64_t* ksk,
                  double* bskf_natural /* n*rows*(k+1)*N doubles, oracle order */);
/* Key switch only: count big LWE rows -> count small LWE rows (n+1 u64). */
int lv_debug_keyswitch(lv_ctx* ctx, const uint64_t* in, size_t count, uint64_t* out_small);
/* Blind rotation only, from modulus-switched inputs (count rows of n+1 u32)
 * -> extracted big LWE rows; glwe_out (nullable) also receives the whole
 * accumulator, count x (k+1) x N u64 (phase-noise measurements). */
int lv_debug_blind_rotate(lv_ctx* ctx, const uint32_t* ms, const uint32_t* lut_ids,
                          size_t count, uint64_t* out, uint64_t* glwe_out);
int lv_debug_fft(lv_ctx* ctx, const int64_t* poly, double* spec, uint64_t* roundtrip);

/* ---- timing helpers for bench.py (device-resident workloads) ----------- */
/* Runs `iters` batched PBS over device-resident inputs already in the pool
 * and returns per-iteration device milliseconds of the blind-rotation
 * kernel, the key-switch kernel and the whole step (CUDA events on the
 * launching stream). */
int lv_bench_pbs(lv_ctx* ctx, const lv_ct* in, const uint32_t* lut_ids, size_t count,
                 int iters, uint64_t flush_bytes, float* br_ms, float* ks_ms, float* step_ms);
/* Measured FP64 FMA throughput of this GPU (TFLOP/s, FMA = 2 flops): the
 * denominator of the blind-rotation roofline. */
int lv_bench_fp64_peak(float* tflops);

#ifdef __cplusplus
}
#endif
#endif
