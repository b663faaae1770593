/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement ("oracle") of the TFHE
 * programmable bootstrap that the B200 product implements.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * the timed CPU baseline. The product path never links it.
 *
 * What it restates
 *   The reference (/root/reference/proj) simulates TFHE: SimBackend::pbs
 *   (proj/src/backend.cpp:61-70) returns negacyclic_eval(lut, x)
 *   (proj/src/lut.cpp:9-16) and never touches a ciphertext. The real
 *   arithmetic lives in a third-party dependency that is NOT under
 *   /root/reference: TFHE-rs v0.7.2 (Rust; "4-bit message
 *   0-bit carry" parameters). This file restates TFHE-rs's published
 *   KS_PBS algorithm (key switch -> modulus switch -> blind rotation with
 *   an f64 negacyclic FFT external product -> sample extract) with a fully
 *   specified IEEE-754 operation order, so the GPU product can be checked
 *   for BIT-EXACT ciphertexts (every rounding is an explicit fma / mul /
 *   add that both CPU and GPU round identically).
 *
 *   The FFT network (radix-4/radix-2 stages, fft_dif / fft_dit_inverse),
 *   the double-double BSK spectrum computed at keygen, and the optional
 *   exact-mask-product split (orc_params.exact_mask_product) are part of
 *   that specification and mirrored by the GPU kernels.
 *
 *   A second blind-rotation mode multiplies polynomials exactly in
 *   Z_{2^64}[X]/(X^N+1) (schoolbook), independent of any FFT, so the FFT
 *   path's extra phase noise can be measured against an exact product
 *   (orc_fft_phase_error_var accounts it deterministically).
 *
 * Parity anchors (decrypted-value level): the reference's own tests and
 * the compiled reference SimBackend (oracle/_ref, tests/golden/).
 * Ciphertext-level parity is pinned only by this oracle ("parity unpinned"
 * against the reference, which has no ciphertexts) — see DESIGN.md.
 */
#ifndef LEUVEN_TFHE_ORACLE_H
#define LEUVEN_TFHE_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  uint32_t n;               /* small LWE dimension                         */
  uint32_t N;               /* GLWE polynomial size (power of two)         */
  uint32_t k;               /* GLWE dimension                              */
  uint32_t pbs_base_log;    /* gadget base log for the BSK                 */
  uint32_t pbs_level;
  uint32_t ks_base_log;     /* gadget base log for the KSK                 */
  uint32_t ks_level;
  uint32_t lwe_noise_log2;  /* TUniform bound log2 for small-key LWE noise */
  uint32_t glwe_noise_log2; /* TUniform bound log2 for GLWE / big-key noise*/
  /* 1: the mask output of every external product splits the BSK mask
   * coefficients b = H * 2^43 + Lo (|H| <= 2^20, |Lo| <= 2^42); the H
   * product is exact in f64 and rounded to an integer, so the FFT adds no
   * noise that the key amplifies. 0: one f64 product. */
  uint32_t exact_mask_product;
} orc_params;

typedef struct orc_ctx orc_ctx;

/* Counter-based generator shared (by specification, not by code) with the
 * product: Philox4x32-10, key = seed, counter = {idx_lo, idx_hi, domain, 0}. */
void orc_philox(uint64_t seed, uint32_t domain, uint64_t idx, uint32_t out[4]);
uint64_t orc_rand_u64(uint64_t seed, uint32_t domain, uint64_t idx);
int64_t orc_tuniform(uint64_t seed, uint32_t domain, uint64_t idx, uint32_t bound_log2);

orc_params orc_default_params(void);

/* Generates all keys deterministically from seed (threads <= 0: nproc). */
orc_ctx* orc_create(const orc_params* p, uint64_t seed, int threads);
void orc_destroy(orc_ctx* c);
const orc_params* orc_get_params(const orc_ctx* c);

/* Key material accessors (for bit-exact comparison with GPU keygen). */
const uint8_t* orc_sk_small(const orc_ctx* c);   /* n                     */
const uint8_t* orc_sk_glwe(const orc_ctx* c);    /* k*N                   */
const uint64_t* orc_ksk(const orc_ctx* c);       /* kN*ks_level*(n+1)     */
const uint64_t* orc_bsk(const orc_ctx* c);       /* n*rows*(k+1)*N        */
const double* orc_bskf(const orc_ctx* c);        /* n*rows*(k+1)*(N/2)*2 (re,im interleaved) */
const double* orc_bskf_hi(const orc_ctx* c);     /* exact_mask_product: n*rows*k*(N/2)*2     */
const double* orc_bskf_lo(const orc_ctx* c);     /* (NULL otherwise)                          */

/* Big-key LWE: kN mask coefficients followed by the body (kN+1 u64). */
void orc_encrypt_at(const orc_ctx* c, int32_t value, uint64_t counter, uint64_t* out);
void orc_trivial(const orc_ctx* c, int32_t value, uint64_t* out);
uint64_t orc_phase(const orc_ctx* c, const uint64_t* lwe_big);
int32_t orc_decrypt(const orc_ctx* c, const uint64_t* lwe_big);
/* Small-key LWE phase (n+1 u64). */
uint64_t orc_phase_small(const orc_ctx* c, const uint64_t* lwe_small);

/* Pieces of the PBS, exposed for stage-by-stage parity tests. */
void orc_keyswitch(const orc_ctx* c, const uint64_t* in_big, uint64_t* out_small);
void orc_modswitch(const orc_ctx* c, const uint64_t* in_small, uint32_t* out);
void orc_test_poly(const orc_ctx* c, const int32_t lut[16], uint64_t* tp);
/* mode 0: f64-FFT external product (bit-exact spec); 1: exact integer. */
void orc_blind_rotate(const orc_ctx* c, const uint32_t* ms, const uint64_t* tp,
                      uint64_t* glwe_out, int mode);
void orc_sample_extract(const orc_ctx* c, const uint64_t* glwe, uint64_t* out_big);
/* count blind rotations (ms rows of n+1, one test polynomial) over threads. */
void orc_blind_rotate_batch(const orc_ctx* c, size_t count, const uint32_t* ms,
                            const uint64_t* tp, uint64_t* glwe_out, int mode, int threads);
/* Sum over CMUX steps of the mean squared phase of (FFT - exact) external
 * product on the same input: the variance the f64 FFT adds (noise tests). */
double orc_fft_phase_error_var(const orc_ctx* c, const uint32_t* ms, const uint64_t* tp);

/* Whole PBS: KS -> MS -> BR -> SE. */
void orc_pbs(const orc_ctx* c, const uint64_t* in_big, const int32_t lut[16],
             uint64_t* out_big, int mode);
/* count independent PBS over `threads` host threads (<=0: nproc). luts is
 * count*16 entries. */
void orc_pbs_batch(const orc_ctx* c, size_t count, const uint64_t* in_big,
                   const int32_t* luts, uint64_t* out_big, int mode, int threads);
/* CPU-baseline build (AVX-512): the same PBS, 8 ciphertexts per vector lane
 * set, bit-identical outputs; returns -1 when built without AVX-512 or for
 * parameters it does not cover (pbs_level != 1, exact-mask keys). */
int orc_pbs_batch_simd(const orc_ctx* c, size_t count, const uint64_t* in_big,
                       const int32_t* luts, uint64_t* out_big, int threads);

/* Negacyclic f64 transform pieces, for unit tests of the FFT spec. */
void orc_fft_forward_i64(const orc_ctx* c, const int64_t* poly, double* spec);
void orc_fft_backward_torus(const orc_ctx* c, const double* spec, uint64_t* poly);

#ifdef __cplusplus
}
#endif
#endif
