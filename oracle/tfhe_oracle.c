/*
 * TEST INFRASTRUCTURE ONLY — see tfhe_oracle.h for scope and anchors.
 *
 * Compiled with -O2 -ffp-contract=off: every floating-point rounding below
 * is the one written (fma() is a single rounding, a*b and a+b are one each),
 * which is what makes the GPU comparison bit-exact.
 *
 * Algorithm anchors
 *  - plaintext space and LUT semantics: Lut16 / negacyclic_eval
 *    (proj/include/leuven/lut.hpp:9-24, proj/src/lut.cpp:9-16): values mod 32,
 *    inputs in [16,32) return -entries[x-16] mod 32. The test polynomial
 *    below realises exactly this, with Delta = 2^64/32.
 *  - decrypt = nearest multiple of Delta (SimBackend::decrypt returns the
 *    plaintext residue, proj/include/leuven/backend.hpp:93).
 *  - KS_PBS pipeline, gadget decomposition, GGSW external product, sample
 *    extract: TFHE-rs v0.7.2 published algorithm (not vendored; named in
 *    PAPER.md:1236), restated here with our own operation order.
 */
#include "tfhe_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

enum {
  D_SK_SMALL = 1,
  D_SK_GLWE = 2,
  D_BSK_MASK = 3,
  D_BSK_NOISE = 4,
  D_KSK_MASK = 5,
  D_KSK_NOISE = 6,
  D_ENC_MASK = 7,
  D_ENC_NOISE = 8,
};

struct orc_ctx {
  orc_params p;
  uint64_t seed;
  uint8_t* sk_small;
  uint8_t* sk_glwe;
  uint64_t* ksk;
  uint64_t* bsk;
  double* bskf;    /* interleaved (re, im) */
  double* bskf_hi; /* exact_mask_product: spectra of H and Lo of every mask */
  double* bskf_lo; /* polynomial, [(i * rows + r) * k + q][2M]             */
  double* fwd_lf;  /* forward twiddles (c, t), level s block b at 2^s - 1 + b */
  double* inv_lf;  /* inverse twiddles (c, t) of conj(W^k), k < M/2 */
  double* twist;   /* zeta^j = exp(i pi j / N), j < M */
  double* untwist; /* zeta^-j / M */
  double* tw_dd;   /* W[t], t < M/2, as (re.hi, re.lo, im.hi, im.lo) */
  double* twist_dd; /* zeta^j, j < M, same packing */
  uint32_t M;      /* N/2 */
  uint32_t logM;
};

/* ------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al., SC'11), the Random123 round function.  */

static inline void mulhilo32(uint32_t a, uint32_t b, uint32_t* hi, uint32_t* lo) {
  uint64_t p = (uint64_t)a * (uint64_t)b;
  *hi = (uint32_t)(p >> 32);
  *lo = (uint32_t)p;
}

void orc_philox(uint64_t seed, uint32_t domain, uint64_t idx, uint32_t out[4]) {
  uint32_t c0 = (uint32_t)idx, c1 = (uint32_t)(idx >> 32), c2 = domain, c3 = 0;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint32_t hi0, lo0, hi1, lo1;
    mulhilo32(0xD2511F53u, c0, &hi0, &lo0);
    mulhilo32(0xCD9E8D57u, c2, &hi1, &lo1);
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0;
    c1 = n1;
    c2 = n2;
    c3 = n3;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

uint64_t orc_rand_u64(uint64_t seed, uint32_t domain, uint64_t idx) {
  uint32_t o[4];
  orc_philox(seed, domain, idx, o);
  return ((uint64_t)o[1] << 32) | o[0];
}

/* TUniform(b): integers in [-2^b, 2^b], endpoints at half weight. */
int64_t orc_tuniform(uint64_t seed, uint32_t domain, uint64_t idx, uint32_t b) {
  uint64_t x = orc_rand_u64(seed, domain, idx) & ((UINT64_C(1) << (b + 2)) - 1);
  return (int64_t)(x >> 1) + (int64_t)(x & 1) - ((int64_t)1 << b);
}

orc_params orc_default_params(void) {
  orc_params p;
  p.n = 880;
  p.N = 2048;
  p.k = 1;
  p.pbs_base_log = 23;
  p.pbs_level = 1;
  p.ks_base_log = 3;
  p.ks_level = 5;
  p.lwe_noise_log2 = 44;
  p.glwe_noise_log2 = 17;
  p.exact_mask_product = 0;
  return p;
}

/* ------------------------------------------------------------------ */
/* threading helper                                                     */

typedef void (*range_fn)(void* arg, size_t lo, size_t hi);
typedef struct {
  range_fn fn;
  void* arg;
  size_t lo, hi;
} range_job;

static void* range_thread(void* a) {
  range_job* j = (range_job*)a;
  j->fn(j->arg, j->lo, j->hi);
  return NULL;
}

static int resolve_threads(int threads) {
  if (threads > 0) return threads;
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

static void parallel_for(size_t count, int threads, range_fn fn, void* arg) {
  threads = resolve_threads(threads);
  if ((size_t)threads > count) threads = (int)count;
  if (threads <= 1) {
    if (count) fn(arg, 0, count);
    return;
  }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  range_job* jobs = (range_job*)malloc(sizeof(range_job) * (size_t)threads);
  for (int t = 0; t < threads; ++t) {
    jobs[t].fn = fn;
    jobs[t].arg = arg;
    jobs[t].lo = count * (size_t)t / (size_t)threads;
    jobs[t].hi = count * (size_t)(t + 1) / (size_t)threads;
    pthread_create(&th[t], NULL, range_thread, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
}

/* ------------------------------------------------------------------ */
/* polynomial helpers over Z_{2^64}[X]/(X^N+1)                         */

/* out = X^e * in, e in [0, 2N) */
static void poly_rotate(const uint64_t* in, uint64_t* out, uint32_t N, uint32_t e) {
  for (uint32_t j = 0; j < N; ++j) {
    uint32_t t = (j + 2 * N - e) % (2 * N);
    out[j] = t < N ? in[t] : (uint64_t)0 - in[t - N];
  }
}

/* acc += a * s (negacyclic), s binary */
static void poly_mul_binary_acc(uint64_t* acc, const uint64_t* a, const uint8_t* s,
                                uint32_t N) {
  for (uint32_t t = 0; t < N; ++t) {
    if (!s[t]) continue;
    /* X^t * a */
    for (uint32_t j = 0; j < N; ++j) {
      if (j + t < N)
        acc[j + t] += a[j];
      else
        acc[j + t - N] -= a[j];
    }
  }
}

/* acc += d * b (negacyclic), d small signed, exact mod 2^64 */
static void poly_mul_small_acc(uint64_t* acc, const int64_t* d, const uint64_t* b,
                               uint32_t N) {
  for (uint32_t t = 0; t < N; ++t) {
    uint64_t dt = (uint64_t)d[t];
    if (!dt) continue;
    for (uint32_t j = 0; j < N; ++j) {
      uint64_t v = dt * b[j];
      if (j + t < N)
        acc[j + t] += v;
      else
        acc[j + t - N] -= v;
    }
  }
}

/* signed gadget decomposition, closest representable, digits in [-B/2, B/2),
 * level index 0 = most significant (weight q/B). */
static void decompose(uint64_t x, uint32_t base_log, uint32_t level, int64_t* digits) {
  const uint32_t shift = 64 - base_log * level;
  uint64_t v = (x + (UINT64_C(1) << (shift - 1))) >> shift;
  const uint64_t mask = (UINT64_C(1) << base_log) - 1;
  const int64_t half = (int64_t)1 << (base_log - 1);
  for (int l = (int)level - 1; l >= 0; --l) {
    int64_t d = (int64_t)(v & mask);
    v >>= base_log;
    if (d >= half) {
      d -= (int64_t)1 << base_log;
      v += 1;
    }
    digits[l] = d;
  }
}

/* ------------------------------------------------------------------ */
/* FFT specification                                                    */

static inline void cmul(double ar, double ai, double br, double bi, double* r, double* i) {
  double t1 = ai * bi;
  double t2 = ai * br;
  *r = fma(ar, br, -t1);
  *i = fma(ar, bi, t2);
}

/* The transform (M = N/2 complex points) is a fixed network of radix-2
 * Cooley-Tukey butterflies u +- w v, each in Linzer-Feig form: the twiddle
 * w = c (1 + i t) is stored as (c, t) = (cos, tan) of its angle, rounded
 * from long double, and the butterfly is six FMAs (ct_lf below).
 * forward (fft_fwd): negacyclic, natural order in, bit-reversed out —
 *   level s (half = M >> (s+1)), block b: w = zeta^e(s, b) with
 *   e(s, b) = (M >> (s+1)) (1 - 4 brv_s(b)) mod 2N, zeta = exp(i pi / N);
 *   the output is the spectrum of the twisted DFT (bin f = the polynomial
 *   at zeta^(1 - 4 brv(f))), so no separate twist is applied. Sibling
 *   blocks differ by w(s, 2b+1) = -i w(s, 2b): at the levels where the GPU
 *   holds the block's low bit in registers (4, 5, 7, 9; production size)
 *   an odd block uses its even sibling's (c, t) with the -i folded into
 *   the FMA operands (ct_lf_mi), so one twiddle serves both.
 * inverse (fft_inv): cyclic DIT, bit-reversed in, natural out — stage s =
 *   logM-1 .. 0, pair (j, j + half), w = conj(W^k), k = j << s, W = exp(-2
 *   pi i / M); the two stages with half <= 2 have w in {1, i} and are exact
 *   additions (ct_one, ct_i); at stages 0, 1, 3, 4, 6 a pair with k >= M/4
 *   uses conj(W^(k - M/4)) with the factor i folded in (ct_lf_i); the
 *   untwist follows in backward_torus.
 * Toy sizes (logM != 10) use the plain forms everywhere.
 * The GPU (csrc/fft.cuh) reorders data, never arithmetic. */
typedef struct {
  double re, im;
} cpx;
static inline cpx ld(const double* x, uint32_t i) { return (cpx){x[2 * i], x[2 * i + 1]}; }
static inline void st(double* x, uint32_t i, cpx v) {
  x[2 * i] = v.re;
  x[2 * i + 1] = v.im;
}

static inline void ct_lf(double* x, uint32_t iu, uint32_t iv, const double* w /* c, t */) {
  const cpx u = ld(x, iu), v = ld(x, iv);
  const double a = fma(-w[1], v.im, v.re);
  const double b = fma(w[1], v.re, v.im);
  st(x, iu, (cpx){fma(w[0], a, u.re), fma(w[0], b, u.im)});
  st(x, iv, (cpx){fma(-w[0], a, u.re), fma(-w[0], b, u.im)});
}
/* u +- (-i w) v with w = c (1 + i t): (-i w) v = c (b - i a) */
static inline void ct_lf_mi(double* x, uint32_t iu, uint32_t iv, const double* w) {
  const cpx u = ld(x, iu), v = ld(x, iv);
  const double a = fma(-w[1], v.im, v.re);
  const double b = fma(w[1], v.re, v.im);
  st(x, iu, (cpx){fma(w[0], b, u.re), fma(-w[0], a, u.im)});
  st(x, iv, (cpx){fma(-w[0], b, u.re), fma(w[0], a, u.im)});
}
/* u +- (i w) v: (i w) v = c (-b + i a) */
static inline void ct_lf_i(double* x, uint32_t iu, uint32_t iv, const double* w) {
  const cpx u = ld(x, iu), v = ld(x, iv);
  const double a = fma(-w[1], v.im, v.re);
  const double b = fma(w[1], v.re, v.im);
  st(x, iu, (cpx){fma(-w[0], b, u.re), fma(w[0], a, u.im)});
  st(x, iv, (cpx){fma(w[0], b, u.re), fma(-w[0], a, u.im)});
}
static inline void ct_one(double* x, uint32_t iu, uint32_t iv) { /* w = 1 */
  const cpx u = ld(x, iu), v = ld(x, iv);
  st(x, iu, (cpx){u.re + v.re, u.im + v.im});
  st(x, iv, (cpx){u.re - v.re, u.im - v.im});
}
static inline void ct_i(double* x, uint32_t iu, uint32_t iv) { /* w = i: u +- i v */
  const cpx u = ld(x, iu), v = ld(x, iv);
  st(x, iu, (cpx){u.re - v.im, u.im + v.re});
  st(x, iv, (cpx){u.re + v.im, u.im - v.re});
}

static void fft_fwd(const orc_ctx* c, double* x /* interleaved M */) {
  const uint32_t M = c->M;
  for (uint32_t s = 0; s < c->logM; ++s) {
    const uint32_t half = M >> (s + 1);
    const int sib = c->logM == 10 && (s == 4 || s == 5 || s == 7 || s == 9);
    for (uint32_t b = 0; b < (1u << s); ++b) {
      const int mi = sib && (b & 1u);
      const double* w = c->fwd_lf + 2 * ((1u << s) - 1 + (mi ? b - 1 : b));
      for (uint32_t j = 0; j < half; ++j) {
        if (mi)
          ct_lf_mi(x, 2 * half * b + j, 2 * half * b + j + half, w);
        else
          ct_lf(x, 2 * half * b + j, 2 * half * b + j + half, w);
      }
    }
  }
}

static void fft_inv(const orc_ctx* c, double* x) {
  const uint32_t M = c->M;
  for (int s = (int)c->logM - 1; s >= 0; --s) {
    const uint32_t half = M >> (s + 1);
    for (uint32_t blk = 0; blk < M; blk += 2 * half)
      for (uint32_t j = 0; j < half; ++j) {
        const uint32_t k = j << s;
        if (half <= 2) {
          if (k == 0)
            ct_one(x, blk + j, blk + j + half);
          else
            ct_i(x, blk + j, blk + j + half);
        } else if (c->logM == 10 && s != 2 && s != 5 && s != 7 && k >= M / 4) {
          ct_lf_i(x, blk + j, blk + j + half, c->inv_lf + 2 * (k - M / 4));
        } else {
          ct_lf(x, blk + j, blk + j + half, c->inv_lf + 2 * k);
        }
      }
  }
}

static inline uint64_t f64_to_torus(double y) {
  const double two64 = 18446744073709551616.0;
  const double inv64 = 0x1p-64;
  double r = rint(y * inv64);
  double d = y - r * two64;
  if (d >= 9223372036854775808.0) d -= two64;
  return (uint64_t)(int64_t)llrint(d);
}

static void forward_i64(const orc_ctx* c, const int64_t* a, double* out) {
  const uint32_t M = c->M;
  for (uint32_t j = 0; j < M; ++j) {
    out[2 * j] = (double)a[j];
    out[2 * j + 1] = (double)a[j + M];
  }
  fft_fwd(c, out);
}

static void backward_torus(const orc_ctx* c, double* spec /* destroyed */, uint64_t* out) {
  const uint32_t M = c->M;
  fft_inv(c, spec);
  for (uint32_t j = 0; j < M; ++j) {
    double re, im;
    cmul(spec[2 * j], spec[2 * j + 1], c->untwist[2 * j], c->untwist[2 * j + 1], &re, &im);
    out[j] = f64_to_torus(re);
    out[j + M] = f64_to_torus(im);
  }
}

/* Key-preparation transform of the BSK (keygen only): the same DIF network
 * in double-double arithmetic with double-double twist/twiddle tables,
 * rounded to double once at the end. Removes the f64 FFT's own rounding of
 * the BSK spectrum (a third of the external product's FFT error, DESIGN.md
 * §2). Operation order is a specification shared with bsk_fourier_dd_kernel
 * (csrc/kernels.cu). */
typedef struct {
  double hi, lo;
} dd_t;
typedef struct {
  dd_t re, im;
} cdd_t;

static inline dd_t dd_two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  const double e = (a - (s - bb)) + (b - bb);
  return (dd_t){s, e};
}
static inline dd_t dd_fast(double a, double b) {
  const double s = a + b;
  return (dd_t){s, b - (s - a)};
}
static inline dd_t dd_add(dd_t x, dd_t y) {
  const dd_t s = dd_two_sum(x.hi, y.hi);
  return dd_fast(s.hi, s.lo + (x.lo + y.lo));
}
static inline dd_t dd_sub(dd_t x, dd_t y) {
  const dd_t s = dd_two_sum(x.hi, -y.hi);
  return dd_fast(s.hi, s.lo + (x.lo - y.lo));
}
static inline dd_t dd_mul(dd_t x, dd_t y) {
  const double p = x.hi * y.hi;
  double e = fma(x.hi, y.hi, -p);
  e = fma(x.hi, y.lo, e);
  e = fma(x.lo, y.hi, e);
  return dd_fast(p, e);
}
static inline cdd_t cdd_mul(cdd_t a, cdd_t b) {
  return (cdd_t){dd_sub(dd_mul(a.re, b.re), dd_mul(a.im, b.im)),
                 dd_add(dd_mul(a.re, b.im), dd_mul(a.im, b.re))};
}
static inline dd_t dd_from_i64(int64_t a) {
  const double hi = (double)(int64_t)((uint64_t)a & ~UINT64_C(0x7FF)); /* <= 53 bits: exact */
  const double lo = (double)(int64_t)((uint64_t)a & UINT64_C(0x7FF));
  return dd_two_sum(hi, lo);
}
static inline cdd_t cdd_load(const double* t) { return (cdd_t){{t[0], t[1]}, {t[2], t[3]}}; }

static void forward_i64_dd(const orc_ctx* c, const int64_t* a, double* out, cdd_t* x) {
  const uint32_t M = c->M;
  for (uint32_t j = 0; j < M; ++j)
    x[j] = cdd_mul((cdd_t){dd_from_i64(a[j]), dd_from_i64(a[j + M])}, cdd_load(c->twist_dd + 4 * j));
  for (uint32_t s = 0; s < c->logM; ++s) {
    const uint32_t half = M >> (s + 1);
    for (uint32_t blk = 0; blk < M; blk += 2 * half)
      for (uint32_t j = 0; j < half; ++j) {
        const cdd_t u = x[blk + j], v = x[blk + j + half];
        x[blk + j] = (cdd_t){dd_add(u.re, v.re), dd_add(u.im, v.im)};
        x[blk + j + half] = cdd_mul((cdd_t){dd_sub(u.re, v.re), dd_sub(u.im, v.im)},
                                    cdd_load(c->tw_dd + 4 * ((size_t)j << s)));
      }
  }
  for (uint32_t f = 0; f < M; ++f) {
    out[2 * f] = x[f].re.hi + x[f].re.lo;
    out[2 * f + 1] = x[f].im.hi + x[f].im.lo;
  }
}

void orc_fft_forward_i64(const orc_ctx* c, const int64_t* poly, double* spec) {
  forward_i64(c, poly, spec);
}

void orc_fft_backward_torus(const orc_ctx* c, const double* spec, uint64_t* poly) {
  double* tmp = (double*)malloc(sizeof(double) * 2 * c->M);
  memcpy(tmp, spec, sizeof(double) * 2 * c->M);
  backward_torus(c, tmp, poly);
  free(tmp);
}

static void build_tables(orc_ctx* c) {
  const uint32_t N = c->p.N, M = N / 2;
  c->M = M;
  c->logM = 0;
  while ((1u << c->logM) < M) ++c->logM;
  const long double PI = 3.141592653589793238462643383279502884L;
  /* Linzer-Feig twiddles (c, t) = (cos, tan), rounded from long double */
  c->fwd_lf = (double*)malloc(sizeof(double) * 2 * M);
  for (uint32_t s = 0; s < c->logM; ++s)
    for (uint32_t b = 0; b < (1u << s); ++b) {
      uint32_t r = 0; /* brv_s(b) */
      for (uint32_t q = 0; q < s; ++q) r |= ((b >> q) & 1u) << (s - 1 - q);
      const int64_t e = ((int64_t)(M >> (s + 1)) * (1 - 4 * (int64_t)r)) % (int64_t)(2 * N);
      const long double ang = PI * (long double)(e < 0 ? e + 2 * N : e) / (long double)N;
      double* w = c->fwd_lf + 2 * ((1u << s) - 1 + b);
      w[0] = (double)cosl(ang);
      w[1] = (double)tanl(ang);
    }
  c->inv_lf = (double*)malloc(sizeof(double) * M);
  for (uint32_t k = 0; k < M / 2; ++k) {
    const long double ang = 2.0L * PI * (long double)k / (long double)M; /* conj(W^k) */
    c->inv_lf[2 * k] = (double)cosl(ang);
    c->inv_lf[2 * k + 1] = (double)tanl(ang);
  }
  /* twist zeta^j = exp(i pi j / N), j < M, is DEFINED as the product of a
   * fine table (j mod 128) and a coarse table (j div 128), each rounded from
   * long double: the GPU keeps only the 2 KB fine table hot in L1. */
  c->twist = (double*)malloc(sizeof(double) * 2 * M);
  c->untwist = (double*)malloc(sizeof(double) * 2 * M);
  const uint32_t FINE = 128, COARSE = M / FINE;
  double* fine = (double*)malloc(sizeof(double) * 2 * FINE);
  double* coarse = (double*)malloc(sizeof(double) * 2 * COARSE);
  for (uint32_t j = 0; j < FINE; ++j) {
    long double ang = PI * (long double)j / (long double)N;
    fine[2 * j] = (double)cosl(ang);
    fine[2 * j + 1] = (double)sinl(ang);
  }
  for (uint32_t k = 0; k < COARSE; ++k) {
    long double ang = PI * (long double)(k * FINE) / (long double)N;
    coarse[2 * k] = (double)cosl(ang);
    coarse[2 * k + 1] = (double)sinl(ang);
  }
  for (uint32_t j = 0; j < M; ++j) {
    double cr, ci;
    cmul(fine[2 * (j % FINE)], fine[2 * (j % FINE) + 1], coarse[2 * (j / FINE)],
         coarse[2 * (j / FINE) + 1], &cr, &ci);
    c->twist[2 * j] = cr;
    c->twist[2 * j + 1] = ci;
    c->untwist[2 * j] = cr / (double)M;
    c->untwist[2 * j + 1] = -ci / (double)M;
  }
  free(fine);
  free(coarse);
  /* double-double tables for the BSK transform: hi = rn(v), lo = rn(v - hi) */
  c->tw_dd = (double*)malloc(sizeof(double) * 4 * (M / 2));
  c->twist_dd = (double*)malloc(sizeof(double) * 4 * M);
  for (uint32_t t = 0; t < M / 2; ++t) {
    const long double ang = 2.0L * PI * (long double)t / (long double)M;
    const long double cr = cosl(ang), ci = -sinl(ang);
    double* e = c->tw_dd + 4 * t;
    e[0] = (double)cr;
    e[1] = (double)(cr - (long double)e[0]);
    e[2] = (double)ci;
    e[3] = (double)(ci - (long double)e[2]);
  }
  for (uint32_t j = 0; j < M; ++j) {
    const long double ang = PI * (long double)j / (long double)N;
    const long double cr = cosl(ang), ci = sinl(ang);
    double* e = c->twist_dd + 4 * j;
    e[0] = (double)cr;
    e[1] = (double)(cr - (long double)e[0]);
    e[2] = (double)ci;
    e[3] = (double)(ci - (long double)e[2]);
  }
}

/* ------------------------------------------------------------------ */
/* key generation                                                       */

static uint32_t rows_of(const orc_params* p) { return (p->k + 1) * p->pbs_level; }

typedef struct {
  orc_ctx* c;
} keygen_arg;

static void bsk_range(void* a, size_t lo, size_t hi) {
  orc_ctx* c = ((keygen_arg*)a)->c;
  const orc_params* p = &c->p;
  const uint32_t N = p->N, k = p->k, rows = rows_of(p), L = p->pbs_level;
  double* spec = (double*)malloc(sizeof(double) * 2 * c->M);
  int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * N);
  cdd_t* work = (cdd_t*)malloc(sizeof(cdd_t) * c->M);
  for (size_t i = lo; i < hi; ++i) {
    for (uint32_t r = 0; r < rows; ++r) {
      const uint32_t comp = r / L, lev = r % L + 1;
      uint64_t* row = c->bsk + (((size_t)i * rows + r) * (k + 1)) * N;
      uint64_t* body = row + (size_t)k * N;
      memset(body, 0, sizeof(uint64_t) * N);
      for (uint32_t q = 0; q < k; ++q) {
        uint64_t* mask = row + (size_t)q * N;
        for (uint32_t cc = 0; cc < N; ++cc)
          mask[cc] = orc_rand_u64(c->seed, D_BSK_MASK,
                                  (((uint64_t)i * rows + r) * k + q) * N + cc);
        poly_mul_binary_acc(body, mask, c->sk_glwe + (size_t)q * N, N);
      }
      for (uint32_t cc = 0; cc < N; ++cc)
        body[cc] += (uint64_t)orc_tuniform(c->seed, D_BSK_NOISE,
                                           ((uint64_t)i * rows + r) * N + cc,
                                           p->glwe_noise_log2);
      if (c->sk_small[i]) {
        const uint64_t g = UINT64_C(1) << (64 - p->pbs_base_log * lev);
        row[(size_t)comp * N] += g; /* constant coefficient of component comp */
      }
      for (uint32_t o = 0; o <= k; ++o) {
        const uint64_t* poly = row + (size_t)o * N;
        for (uint32_t cc = 0; cc < N; ++cc) tmp[cc] = (int64_t)poly[cc];
        forward_i64_dd(c, tmp, spec, work);
        memcpy(c->bskf + (((size_t)i * rows + r) * (k + 1) + o) * 2 * c->M, spec,
               sizeof(double) * 2 * c->M);
        if (p->exact_mask_product && o < k) {
          /* b = H * 2^43 + Lo, H = round(b / 2^43) (signed, mod 2^64) */
          int64_t* lo = (int64_t*)malloc(sizeof(int64_t) * N);
          for (uint32_t cc = 0; cc < N; ++cc) {
            const int64_t h = (int64_t)(poly[cc] + (UINT64_C(1) << 42)) >> 43;
            tmp[cc] = h;
            lo[cc] = (int64_t)(poly[cc] - ((uint64_t)h << 43));
          }
          const size_t slot = (((size_t)i * rows + r) * k + o) * 2 * c->M;
          forward_i64_dd(c, tmp, spec, work);
          memcpy(c->bskf_hi + slot, spec, sizeof(double) * 2 * c->M);
          forward_i64_dd(c, lo, spec, work);
          memcpy(c->bskf_lo + slot, spec, sizeof(double) * 2 * c->M);
          free(lo);
        }
      }
    }
  }
  free(spec);
  free(tmp);
  free(work);
}

static void ksk_range(void* a, size_t lo, size_t hi) {
  orc_ctx* c = ((keygen_arg*)a)->c;
  const orc_params* p = &c->p;
  const uint32_t n = p->n, L = p->ks_level;
  for (size_t j = lo; j < hi; ++j) {
    for (uint32_t l = 0; l < L; ++l) {
      uint64_t* row = c->ksk + ((size_t)j * L + l) * (n + 1);
      uint64_t b = 0;
      for (uint32_t cc = 0; cc < n; ++cc) {
        row[cc] = orc_rand_u64(c->seed, D_KSK_MASK, ((uint64_t)j * L + l) * n + cc);
        if (c->sk_small[cc]) b += row[cc];
      }
      b += (uint64_t)orc_tuniform(c->seed, D_KSK_NOISE, (uint64_t)j * L + l,
                                  p->lwe_noise_log2);
      if (c->sk_glwe[j]) b += UINT64_C(1) << (64 - p->ks_base_log * (l + 1));
      row[n] = b;
    }
  }
}

orc_ctx* orc_create(const orc_params* p, uint64_t seed, int threads) {
  orc_ctx* c = (orc_ctx*)calloc(1, sizeof(orc_ctx));
  c->p = *p;
  c->seed = seed;
  const uint32_t n = p->n, N = p->N, k = p->k, rows = rows_of(p);
  build_tables(c);
  c->sk_small = (uint8_t*)malloc(n);
  for (uint32_t i = 0; i < n; ++i) c->sk_small[i] = (uint8_t)(orc_rand_u64(seed, D_SK_SMALL, i) & 1);
  c->sk_glwe = (uint8_t*)malloc((size_t)k * N);
  for (uint32_t j = 0; j < k * N; ++j) c->sk_glwe[j] = (uint8_t)(orc_rand_u64(seed, D_SK_GLWE, j) & 1);
  c->bsk = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n * rows * (k + 1) * N);
  c->bskf = (double*)malloc(sizeof(double) * (size_t)n * rows * (k + 1) * N);
  if (p->exact_mask_product) {
    c->bskf_hi = (double*)malloc(sizeof(double) * (size_t)n * rows * k * N);
    c->bskf_lo = (double*)malloc(sizeof(double) * (size_t)n * rows * k * N);
  }
  c->ksk = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)k * N * p->ks_level * (n + 1));
  keygen_arg ka = {c};
  parallel_for(n, threads, bsk_range, &ka);
  parallel_for((size_t)k * N, threads, ksk_range, &ka);
  return c;
}

void orc_destroy(orc_ctx* c) {
  if (!c) return;
  free(c->sk_small);
  free(c->sk_glwe);
  free(c->bsk);
  free(c->bskf);
  free(c->bskf_hi);
  free(c->bskf_lo);
  free(c->ksk);
  free(c->fwd_lf);
  free(c->inv_lf);
  free(c->twist);
  free(c->untwist);
  free(c->tw_dd);
  free(c->twist_dd);
  free(c);
}

const orc_params* orc_get_params(const orc_ctx* c) { return &c->p; }
const uint8_t* orc_sk_small(const orc_ctx* c) { return c->sk_small; }
const uint8_t* orc_sk_glwe(const orc_ctx* c) { return c->sk_glwe; }
const uint64_t* orc_ksk(const orc_ctx* c) { return c->ksk; }
const uint64_t* orc_bsk(const orc_ctx* c) { return c->bsk; }
const double* orc_bskf(const orc_ctx* c) { return c->bskf; }
const double* orc_bskf_hi(const orc_ctx* c) { return c->bskf_hi; }
const double* orc_bskf_lo(const orc_ctx* c) { return c->bskf_lo; }

/* ------------------------------------------------------------------ */
/* encryption                                                           */

static inline uint64_t delta(void) { return UINT64_C(1) << 59; } /* 2^64 / 32 */

void orc_encrypt_at(const orc_ctx* c, int32_t value, uint64_t counter, uint64_t* out) {
  const uint32_t kN = c->p.k * c->p.N;
  uint64_t b = 0;
  for (uint32_t j = 0; j < kN; ++j) {
    out[j] = orc_rand_u64(c->seed, D_ENC_MASK, counter * kN + j);
    if (c->sk_glwe[j]) b += out[j];
  }
  b += (uint64_t)orc_tuniform(c->seed, D_ENC_NOISE, counter, c->p.glwe_noise_log2);
  b += (uint64_t)(int64_t)value * delta();
  out[kN] = b;
}

void orc_trivial(const orc_ctx* c, int32_t value, uint64_t* out) {
  const uint32_t kN = c->p.k * c->p.N;
  memset(out, 0, sizeof(uint64_t) * kN);
  out[kN] = (uint64_t)(int64_t)value * delta();
}

uint64_t orc_phase(const orc_ctx* c, const uint64_t* lwe) {
  const uint32_t kN = c->p.k * c->p.N;
  uint64_t s = 0;
  for (uint32_t j = 0; j < kN; ++j)
    if (c->sk_glwe[j]) s += lwe[j];
  return lwe[kN] - s;
}

uint64_t orc_phase_small(const orc_ctx* c, const uint64_t* lwe) {
  uint64_t s = 0;
  for (uint32_t j = 0; j < c->p.n; ++j)
    if (c->sk_small[j]) s += lwe[j];
  return lwe[c->p.n] - s;
}

int32_t orc_decrypt(const orc_ctx* c, const uint64_t* lwe) {
  uint64_t ph = orc_phase(c, lwe);
  return (int32_t)(((ph + (delta() >> 1)) >> 59) & 31);
}

/* ------------------------------------------------------------------ */
/* PBS pieces                                                           */

void orc_keyswitch(const orc_ctx* c, const uint64_t* in, uint64_t* out) {
  const orc_params* p = &c->p;
  const uint32_t kN = p->k * p->N, n = p->n, L = p->ks_level;
  int64_t dig[64];
  memset(out, 0, sizeof(uint64_t) * n);
  out[n] = in[kN];
  for (uint32_t j = 0; j < kN; ++j) {
    decompose(in[j], p->ks_base_log, L, dig);
    for (uint32_t l = 0; l < L; ++l) {
      if (!dig[l]) continue;
      const uint64_t d = (uint64_t)dig[l];
      const uint64_t* row = c->ksk + ((size_t)j * L + l) * (n + 1);
      for (uint32_t cc = 0; cc <= n; ++cc) out[cc] -= d * row[cc];
    }
  }
}

void orc_modswitch(const orc_ctx* c, const uint64_t* in, uint32_t* out) {
  uint32_t log2N2 = 1;
  while ((1u << log2N2) < 2 * c->p.N) ++log2N2;
  const uint32_t shift = 64 - log2N2;
  for (uint32_t j = 0; j <= c->p.n; ++j)
    out[j] = (uint32_t)(((in[j] + (UINT64_C(1) << (shift - 1))) >> shift) & ((1u << log2N2) - 1));
}

void orc_test_poly(const orc_ctx* c, const int32_t lut[16], uint64_t* tp) {
  const uint32_t N = c->p.N;
  const uint32_t box = N / 16, half = N / 32;
  for (uint32_t j = 0; j < N; ++j) {
    uint32_t t = j + half; /* tp = X^{-half} * aligned boxes */
    if (t < N)
      tp[j] = (uint64_t)(int64_t)lut[t / box] * delta();
    else
      tp[j] = (uint64_t)0 - (uint64_t)(int64_t)lut[(t - N) / box] * delta();
  }
}

/* acc += d * b per bin, the MAC's fixed FMA order (blind_rotate_kernel) */
static void mac_bins(double* acc, const double* d, const double* b, uint32_t M) {
  for (uint32_t f = 0; f < M; ++f) {
    double ar = acc[2 * f], ai = acc[2 * f + 1];
    const double dr = d[2 * f], di = d[2 * f + 1];
    const double br = b[2 * f], bi = b[2 * f + 1];
    ar = fma(dr, br, ar);
    ar = fma(-di, bi, ar);
    ai = fma(dr, bi, ai);
    ai = fma(di, br, ai);
    acc[2 * f] = ar;
    acc[2 * f + 1] = ai;
  }
}

static void external_product_fft(const orc_ctx* c, size_t i, const uint64_t* glwe_in,
                                 uint64_t* glwe_out, double* specs /* rows*2M */,
                                 double* acc /* 2M */, int64_t* dig /* L*N */) {
  const orc_params* p = &c->p;
  const uint32_t N = p->N, k = p->k, L = p->pbs_level, rows = rows_of(p), M = c->M;
  int64_t dl[64];
  for (uint32_t comp = 0; comp <= k; ++comp) {
    const uint64_t* poly = glwe_in + (size_t)comp * N;
    for (uint32_t j = 0; j < N; ++j) {
      decompose(poly[j], p->pbs_base_log, L, dl);
      for (uint32_t l = 0; l < L; ++l) dig[(size_t)l * N + j] = dl[l];
    }
    for (uint32_t l = 0; l < L; ++l)
      forward_i64(c, dig + (size_t)l * N, specs + (size_t)(comp * L + l) * 2 * M);
  }
  for (uint32_t o = 0; o <= k; ++o) {
    if (p->exact_mask_product && o < k) {
      /* mask output: 2^43 * round(sum d * H) + sum d * Lo */
      uint64_t* hi = (uint64_t*)malloc(sizeof(uint64_t) * N);
      for (int part = 0; part < 2; ++part) {
        memset(acc, 0, sizeof(double) * 2 * M);
        for (uint32_t rr = 0; rr < rows; ++rr) {
          const uint32_t r = (rr + o) % rows; /* output o: row o first */
          const double* d = specs + (size_t)r * 2 * M;
          const double* b = (part == 0 ? c->bskf_hi : c->bskf_lo) + ((i * rows + r) * k + o) * 2 * M;
          mac_bins(acc, d, b, M);
        }
        backward_torus(c, acc, part == 0 ? hi : glwe_out + (size_t)o * N);
      }
      for (uint32_t j = 0; j < N; ++j) glwe_out[(size_t)o * N + j] += hi[j] << 43;
      free(hi);
      continue;
    }
    memset(acc, 0, sizeof(double) * 2 * M);
    for (uint32_t rr = 0; rr < rows; ++rr) {
      const uint32_t r = (rr + o) % rows; /* output o: row o first */
      const double* d = specs + (size_t)r * 2 * M;
      const double* b = c->bskf + ((i * rows + r) * (k + 1) + o) * 2 * M;
      for (uint32_t f = 0; f < M; ++f) {
        double ar = acc[2 * f], ai = acc[2 * f + 1];
        const double dr = d[2 * f], di = d[2 * f + 1];
        const double br = b[2 * f], bi = b[2 * f + 1];
        ar = fma(dr, br, ar);
        ar = fma(-di, bi, ar);
        ai = fma(dr, bi, ai);
        ai = fma(di, br, ai);
        acc[2 * f] = ar;
        acc[2 * f + 1] = ai;
      }
    }
    backward_torus(c, acc, glwe_out + (size_t)o * N);
  }
}

static void external_product_exact(const orc_ctx* c, size_t i, const uint64_t* glwe_in,
                                   uint64_t* glwe_out, int64_t* dig) {
  const orc_params* p = &c->p;
  const uint32_t N = p->N, k = p->k, L = p->pbs_level, rows = rows_of(p);
  int64_t dl[64];
  memset(glwe_out, 0, sizeof(uint64_t) * (k + 1) * N);
  for (uint32_t comp = 0; comp <= k; ++comp) {
    const uint64_t* poly = glwe_in + (size_t)comp * N;
    for (uint32_t j = 0; j < N; ++j) {
      decompose(poly[j], p->pbs_base_log, L, dl);
      for (uint32_t l = 0; l < L; ++l) dig[(size_t)l * N + j] = dl[l];
    }
    for (uint32_t l = 0; l < L; ++l) {
      const uint32_t r = comp * L + l;
      for (uint32_t o = 0; o <= k; ++o)
        poly_mul_small_acc(glwe_out + (size_t)o * N, dig + (size_t)l * N,
                           c->bsk + ((i * rows + r) * (k + 1) + o) * N, N);
    }
  }
}

void orc_blind_rotate(const orc_ctx* c, const uint32_t* ms, const uint64_t* tp,
                      uint64_t* acc, int mode) {
  const orc_params* p = &c->p;
  const uint32_t N = p->N, k = p->k, n = p->n, M = c->M;
  const size_t glen = (size_t)(k + 1) * N;
  memset(acc, 0, sizeof(uint64_t) * (size_t)k * N);
  poly_rotate(tp, acc + (size_t)k * N, N, (2 * N - ms[n]) % (2 * N));
  uint64_t* diff = (uint64_t*)malloc(sizeof(uint64_t) * glen);
  uint64_t* ext = (uint64_t*)malloc(sizeof(uint64_t) * glen);
  double* specs = (double*)malloc(sizeof(double) * 2 * M * rows_of(p));
  double* facc = (double*)malloc(sizeof(double) * 2 * M);
  int64_t* dig = (int64_t*)malloc(sizeof(int64_t) * N * p->pbs_level);
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t a = ms[i];
    if (a == 0) continue;
    for (uint32_t comp = 0; comp <= k; ++comp) {
      poly_rotate(acc + (size_t)comp * N, diff + (size_t)comp * N, N, a);
      for (uint32_t j = 0; j < N; ++j) diff[(size_t)comp * N + j] -= acc[(size_t)comp * N + j];
    }
    if (mode == 0)
      external_product_fft(c, i, diff, ext, specs, facc, dig);
    else
      external_product_exact(c, i, diff, ext, dig);
    for (size_t j = 0; j < glen; ++j) acc[j] += ext[j];
  }
  free(diff);
  free(ext);
  free(specs);
  free(facc);
  free(dig);
}

/* Noise accounting (test infrastructure): one FFT-mode blind rotation in
 * which every external product is also computed exactly on the same input;
 * returns the sum over CMUX steps of the mean squared phase of
 * (FFT product - exact product), i.e. the variance the f64 FFT adds to the
 * accumulator phase, free of the run-to-run spread of a noise estimate. */
double orc_fft_phase_error_var(const orc_ctx* c, const uint32_t* ms, const uint64_t* tp) {
  const orc_params* p = &c->p;
  const uint32_t N = p->N, k = p->k, n = p->n, M = c->M;
  const size_t glen = (size_t)(k + 1) * N;
  uint64_t* acc = (uint64_t*)calloc(glen, sizeof(uint64_t));
  poly_rotate(tp, acc + (size_t)k * N, N, (2 * N - ms[n]) % (2 * N));
  uint64_t* diff = (uint64_t*)malloc(sizeof(uint64_t) * glen);
  uint64_t* ext = (uint64_t*)malloc(sizeof(uint64_t) * glen);
  uint64_t* ex2 = (uint64_t*)malloc(sizeof(uint64_t) * glen);
  uint64_t* ph = (uint64_t*)malloc(sizeof(uint64_t) * N);
  double* specs = (double*)malloc(sizeof(double) * 2 * M * rows_of(p));
  double* facc = (double*)malloc(sizeof(double) * 2 * M);
  int64_t* dig = (int64_t*)malloc(sizeof(int64_t) * N * p->pbs_level);
  double total = 0;
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t a = ms[i];
    if (a == 0) continue;
    for (uint32_t comp = 0; comp <= k; ++comp) {
      poly_rotate(acc + (size_t)comp * N, diff + (size_t)comp * N, N, a);
      for (uint32_t j = 0; j < N; ++j) diff[(size_t)comp * N + j] -= acc[(size_t)comp * N + j];
    }
    external_product_fft(c, i, diff, ext, specs, facc, dig);
    external_product_exact(c, i, diff, ex2, dig);
    for (size_t j = 0; j < glen; ++j) ex2[j] = ext[j] - ex2[j];
    /* phase = B - sum_q A_q * S_q */
    memcpy(ph, ex2 + (size_t)k * N, sizeof(uint64_t) * N);
    for (uint32_t q = 0; q < k; ++q) {
      uint64_t* neg = diff; /* reuse as scratch: -A_q */
      for (uint32_t j = 0; j < N; ++j) neg[j] = (uint64_t)0 - ex2[(size_t)q * N + j];
      poly_mul_binary_acc(ph, neg, c->sk_glwe + (size_t)q * N, N);
    }
    double s = 0;
    for (uint32_t j = 0; j < N; ++j) {
      const double e = (double)(int64_t)ph[j];
      s += e * e;
    }
    total += s / N;
    for (size_t j = 0; j < glen; ++j) acc[j] += ext[j];
  }
  free(acc);
  free(diff);
  free(ext);
  free(ex2);
  free(ph);
  free(specs);
  free(facc);
  free(dig);
  return total;
}

void orc_sample_extract(const orc_ctx* c, const uint64_t* glwe, uint64_t* out) {
  const uint32_t N = c->p.N, k = c->p.k;
  for (uint32_t q = 0; q < k; ++q) {
    const uint64_t* a = glwe + (size_t)q * N;
    out[(size_t)q * N] = a[0];
    for (uint32_t j = 1; j < N; ++j) out[(size_t)q * N + j] = (uint64_t)0 - a[N - j];
  }
  out[(size_t)k * N] = glwe[(size_t)k * N];
}

void orc_pbs(const orc_ctx* c, const uint64_t* in, const int32_t lut[16], uint64_t* out,
             int mode) {
  const orc_params* p = &c->p;
  uint64_t* small = (uint64_t*)malloc(sizeof(uint64_t) * (p->n + 1));
  uint32_t* ms = (uint32_t*)malloc(sizeof(uint32_t) * (p->n + 1));
  uint64_t* tp = (uint64_t*)malloc(sizeof(uint64_t) * p->N);
  uint64_t* acc = (uint64_t*)malloc(sizeof(uint64_t) * (p->k + 1) * p->N);
  orc_keyswitch(c, in, small);
  orc_modswitch(c, small, ms);
  orc_test_poly(c, lut, tp);
  orc_blind_rotate(c, ms, tp, acc, mode);
  orc_sample_extract(c, acc, out);
  free(small);
  free(ms);
  free(tp);
  free(acc);
}

typedef struct {
  const orc_ctx* c;
  const uint64_t* in;
  const int32_t* luts;
  uint64_t* out;
  int mode;
} pbs_batch_arg;

static void pbs_range(void* a, size_t lo, size_t hi) {
  pbs_batch_arg* b = (pbs_batch_arg*)a;
  const size_t len = (size_t)b->c->p.k * b->c->p.N + 1;
  for (size_t t = lo; t < hi; ++t)
    orc_pbs(b->c, b->in + t * len, b->luts + 16 * t, b->out + t * len, b->mode);
}

void orc_pbs_batch(const orc_ctx* c, size_t count, const uint64_t* in, const int32_t* luts,
                   uint64_t* out, int mode, int threads) {
  pbs_batch_arg a = {c, in, luts, out, mode};
  parallel_for(count, threads, pbs_range, &a);
}

typedef struct {
  const orc_ctx* c;
  const uint32_t* ms;
  const uint64_t* tp;
  uint64_t* out;
  int mode;
} br_batch_arg;

static void br_range(void* a, size_t lo, size_t hi) {
  br_batch_arg* b = (br_batch_arg*)a;
  const size_t n1 = b->c->p.n + 1, g = (size_t)(b->c->p.k + 1) * b->c->p.N;
  for (size_t t = lo; t < hi; ++t) orc_blind_rotate(b->c, b->ms + t * n1, b->tp, b->out + t * g, b->mode);
}

void orc_blind_rotate_batch(const orc_ctx* c, size_t count, const uint32_t* ms,
                            const uint64_t* tp, uint64_t* glwe_out, int mode, int threads) {
  br_batch_arg a = {c, ms, tp, glwe_out, mode};
  parallel_for(count, threads, br_range, &a);
}

/* ------------------------------------------------------------------ */
/* CPU-baseline build only: the same KS_PBS, 8 ciphertexts in lockstep, one */
/* per AVX-512 lane (the FFT, MAC and conversions vectorised across the     */
/* batch, the KSK streamed once per 8 ciphertexts). Every lane performs     */
/* exactly the scalar path's IEEE operations (vfmadd/vfnmadd are single-    */
/* rounding fma, the torus conversion is rint + fix-up + nearest-even), so  */
/* outputs are bit-identical to orc_pbs (checked by tests/test_oracle_     */
/* pins.py). FFT-spec mode (mode 0) and default-layout keys only.           */
#if defined(__AVX512F__) && defined(__AVX512DQ__)
#include <immintrin.h>
#define W8 8

typedef struct {
  __m512d re, im;
} v8c;

static inline void v_ct_lf(v8c* u, v8c* v, const double* w) {
  const __m512d c = _mm512_set1_pd(w[0]), t = _mm512_set1_pd(w[1]);
  const __m512d a = _mm512_fnmadd_pd(t, v->im, v->re); /* fma(-t, v.im, v.re) */
  const __m512d b = _mm512_fmadd_pd(t, v->re, v->im);
  const v8c U = *u;
  u->re = _mm512_fmadd_pd(c, a, U.re);
  u->im = _mm512_fmadd_pd(c, b, U.im);
  v->re = _mm512_fnmadd_pd(c, a, U.re);
  v->im = _mm512_fnmadd_pd(c, b, U.im);
}
static inline void v_ct_lf_mi(v8c* u, v8c* v, const double* w) { /* (-i w) v = c (b - i a) */
  const __m512d c = _mm512_set1_pd(w[0]), t = _mm512_set1_pd(w[1]);
  const __m512d a = _mm512_fnmadd_pd(t, v->im, v->re);
  const __m512d b = _mm512_fmadd_pd(t, v->re, v->im);
  const v8c U = *u;
  u->re = _mm512_fmadd_pd(c, b, U.re);
  u->im = _mm512_fnmadd_pd(c, a, U.im);
  v->re = _mm512_fnmadd_pd(c, b, U.re);
  v->im = _mm512_fmadd_pd(c, a, U.im);
}
static inline void v_ct_lf_i(v8c* u, v8c* v, const double* w) { /* (i w) v = c (-b + i a) */
  const __m512d c = _mm512_set1_pd(w[0]), t = _mm512_set1_pd(w[1]);
  const __m512d a = _mm512_fnmadd_pd(t, v->im, v->re);
  const __m512d b = _mm512_fmadd_pd(t, v->re, v->im);
  const v8c U = *u;
  u->re = _mm512_fnmadd_pd(c, b, U.re);
  u->im = _mm512_fmadd_pd(c, a, U.im);
  v->re = _mm512_fmadd_pd(c, b, U.re);
  v->im = _mm512_fnmadd_pd(c, a, U.im);
}

static void v_fft_fwd(const orc_ctx* c, v8c* x) {
  const uint32_t M = c->M;
  for (uint32_t s = 0; s < c->logM; ++s) {
    const uint32_t half = M >> (s + 1);
    const int sib = c->logM == 10 && (s == 4 || s == 5 || s == 7 || s == 9);
    for (uint32_t b = 0; b < (1u << s); ++b) {
      const int mi = sib && (b & 1u);
      const double* w = c->fwd_lf + 2 * ((1u << s) - 1 + (mi ? b - 1 : b));
      v8c* blk = x + 2 * half * b;
      for (uint32_t j = 0; j < half; ++j) {
        if (mi)
          v_ct_lf_mi(blk + j, blk + j + half, w);
        else
          v_ct_lf(blk + j, blk + j + half, w);
      }
    }
  }
}

static void v_fft_inv(const orc_ctx* c, v8c* x) {
  const uint32_t M = c->M;
  for (int s = (int)c->logM - 1; s >= 0; --s) {
    const uint32_t half = M >> (s + 1);
    for (uint32_t blk = 0; blk < M; blk += 2 * half)
      for (uint32_t j = 0; j < half; ++j) {
        const uint32_t k = j << s;
        v8c* u = x + blk + j;
        v8c* v = x + blk + j + half;
        if (half <= 2) {
          const v8c U = *u, V = *v;
          if (k == 0) {
            u->re = _mm512_add_pd(U.re, V.re);
            u->im = _mm512_add_pd(U.im, V.im);
            v->re = _mm512_sub_pd(U.re, V.re);
            v->im = _mm512_sub_pd(U.im, V.im);
          } else { /* u +- i v */
            u->re = _mm512_sub_pd(U.re, V.im);
            u->im = _mm512_add_pd(U.im, V.re);
            v->re = _mm512_add_pd(U.re, V.im);
            v->im = _mm512_sub_pd(U.im, V.re);
          }
        } else if (c->logM == 10 && s != 2 && s != 5 && s != 7 && k >= M / 4) {
          v_ct_lf_i(u, v, c->inv_lf + 2 * (k - M / 4));
        } else {
          v_ct_lf(u, v, c->inv_lf + 2 * k);
        }
      }
  }
}

/* f64_to_torus per lane: r = rint(y 2^-64), d = y - r 2^64 (exact), d >= 2^63
 * -> d - 2^64, then llrint (nearest-even, the default MXCSR mode). */
static inline __m512i v_f64_to_torus(__m512d y) {
  const __m512d two64 = _mm512_set1_pd(18446744073709551616.0);
  const __m512d r = _mm512_roundscale_pd(_mm512_mul_pd(y, _mm512_set1_pd(0x1p-64)),
                                         _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC);
  __m512d d = _mm512_sub_pd(y, _mm512_mul_pd(r, two64));
  const __mmask8 big = _mm512_cmp_pd_mask(d, _mm512_set1_pd(9223372036854775808.0), _CMP_GE_OQ);
  d = _mm512_mask_sub_pd(d, big, d, two64);
  return _mm512_cvtpd_epi64(d);
}

typedef struct {
  uint64_t* acc;   /* [(k+1) N][W8]: the 8 accumulators lane-interleaved */
  v8c* spec;       /* [rows][M] */
  v8c* facc;       /* [M] */
  uint64_t* small; /* [W8][n+1] */
  uint32_t* ms;    /* [W8][n+1] */
  uint64_t* tp;    /* [N] */
} v_scratch;

/* the 8 ciphertexts in[w] (count <= 8 real ones; the rest repeat lane 0) */
static void v_pbs8(const orc_ctx* c, const uint64_t* const* in, const int32_t* const* luts,
                   uint64_t* const* out, int count, v_scratch* sc) {
  const orc_params* p = &c->p;
  const uint32_t N = p->N, k = p->k, n = p->n, M = c->M, L = p->ks_level, rows = rows_of(p);
  const uint32_t kN = k * N;
  /* key switch: the KSK row of (j, l) serves all 8 ciphertexts */
  for (int w = 0; w < W8; ++w) {
    uint64_t* o = sc->small + (size_t)w * (n + 1);
    memset(o, 0, sizeof(uint64_t) * n);
    o[n] = in[w][kN];
  }
  int64_t dig[W8][64];
  for (uint32_t j = 0; j < kN; ++j) {
    for (int w = 0; w < W8; ++w) decompose(in[w][j], p->ks_base_log, L, dig[w]);
    for (uint32_t l = 0; l < L; ++l) {
      const uint64_t* row = c->ksk + ((size_t)j * L + l) * (n + 1);
      for (int w = 0; w < W8; ++w) {
        if (!dig[w][l]) continue;
        const __m512i d = _mm512_set1_epi64(dig[w][l]);
        uint64_t* o = sc->small + (size_t)w * (n + 1);
        uint32_t cc = 0;
        for (; cc + 8 <= n + 1; cc += 8) {
          const __m512i r = _mm512_loadu_si512((const void*)(row + cc));
          const __m512i v = _mm512_loadu_si512((const void*)(o + cc));
          _mm512_storeu_si512((void*)(o + cc), _mm512_sub_epi64(v, _mm512_mullo_epi64(d, r)));
        }
        for (; cc <= n; ++cc) o[cc] -= (uint64_t)dig[w][l] * row[cc];
      }
    }
  }
  /* ACC = X^{-b~} (0, TP), lane-interleaved */
  memset(sc->acc, 0, sizeof(uint64_t) * W8 * (size_t)k * N);
  for (int w = 0; w < W8; ++w) {
    orc_modswitch(c, sc->small + (size_t)w * (n + 1), sc->ms + (size_t)w * (n + 1));
    orc_test_poly(c, luts[w], sc->tp);
    const uint32_t e = (2 * N - sc->ms[(size_t)w * (n + 1) + n]) % (2 * N);
    for (uint32_t j = 0; j < N; ++j) {
      const uint32_t t = (j + 2 * N - e) % (2 * N);
      sc->acc[((size_t)k * N + j) * W8 + w] = t < N ? sc->tp[t] : (uint64_t)0 - sc->tp[t - N];
    }
  }
  const __m512i lane = _mm512_setr_epi64(0, 1, 2, 3, 4, 5, 6, 7);
  const __m512i half41 = _mm512_set1_epi64((int64_t)1 << 40);
  for (uint32_t i = 0; i < n; ++i) {
    /* per-lane rotation a_w: rotated difference, 1-level base-2^23 digit
     * (decompose: (x + 2^40) >> 41, centred), folded into the spectra */
    int64_t av[W8];
    for (int w = 0; w < W8; ++w) av[w] = sc->ms[(size_t)w * (n + 1) + i];
    const __m512i a = _mm512_loadu_si512((const void*)av);
    for (uint32_t comp = 0; comp <= k; ++comp) {
      const uint64_t* P = sc->acc + (size_t)comp * N * W8;
      double* sp = (double*)(sc->spec + (size_t)comp * M);
      for (uint32_t j = 0; j < N; ++j) {
        /* t = (j - a) mod 2N; rv = t < N ? P[t] : -P[t - N] */
        __m512i t = _mm512_sub_epi64(_mm512_set1_epi64(j + 2 * N), a);
        t = _mm512_and_si512(t, _mm512_set1_epi64(2 * N - 1));
        const __mmask8 wrap = _mm512_cmpge_epu64_mask(t, _mm512_set1_epi64(N));
        const __m512i src = _mm512_mask_sub_epi64(t, wrap, t, _mm512_set1_epi64(N));
        const __m512i idx = _mm512_add_epi64(_mm512_slli_epi64(src, 3), lane);
        __m512i rv = _mm512_i64gather_epi64(idx, (const void*)P, 8);
        rv = _mm512_mask_sub_epi64(rv, wrap, _mm512_setzero_si512(), rv);
        const __m512i x = _mm512_sub_epi64(rv, _mm512_loadu_si512((const void*)(P + (size_t)j * W8)));
        const __m512i v = _mm512_srli_epi64(_mm512_add_epi64(x, half41), 41);
        const __m512i d = _mm512_srai_epi64(_mm512_slli_epi64(v, 41), 41); /* centred 23-bit digit */
        const uint32_t jj = j < M ? j : j - M;
        _mm512_storeu_pd(sp + (size_t)jj * 16 + (j < M ? 0 : 8), _mm512_cvtepi64_pd(d));
      }
    }
    for (uint32_t r = 0; r < rows; ++r) v_fft_fwd(c, sc->spec + (size_t)r * M);
    for (uint32_t o = 0; o <= k; ++o) {
      for (uint32_t f = 0; f < M; ++f) {
        __m512d ar = _mm512_setzero_pd(), ai = _mm512_setzero_pd();
        for (uint32_t rr = 0; rr < rows; ++rr) {
          const uint32_t r = (rr + o) % rows;
          const v8c dd = sc->spec[(size_t)r * M + f];
          const double* b = c->bskf + ((i * rows + r) * (k + 1) + o) * 2 * M + 2 * f;
          const __m512d br = _mm512_set1_pd(b[0]), bi = _mm512_set1_pd(b[1]);
          ar = _mm512_fmadd_pd(dd.re, br, ar);
          ar = _mm512_fnmadd_pd(dd.im, bi, ar);
          ai = _mm512_fmadd_pd(dd.re, bi, ai);
          ai = _mm512_fmadd_pd(dd.im, br, ai);
        }
        sc->facc[f].re = ar;
        sc->facc[f].im = ai;
      }
      v_fft_inv(c, sc->facc);
      uint64_t* A = sc->acc + (size_t)o * N * W8;
      for (uint32_t j = 0; j < M; ++j) {
        const __m512d ur = _mm512_set1_pd(c->untwist[2 * j]), ui = _mm512_set1_pd(c->untwist[2 * j + 1]);
        const v8c z = sc->facc[j];
        const __m512d t1 = _mm512_mul_pd(z.im, ui), t2 = _mm512_mul_pd(z.im, ur);
        const __m512d re = _mm512_fmsub_pd(z.re, ur, t1); /* fma(ar, br, -t1) */
        const __m512d im = _mm512_fmadd_pd(z.re, ui, t2);
        uint64_t* a0 = A + (size_t)j * W8;
        uint64_t* a1 = A + (size_t)(j + M) * W8;
        _mm512_storeu_si512((void*)a0, _mm512_add_epi64(_mm512_loadu_si512((const void*)a0), v_f64_to_torus(re)));
        _mm512_storeu_si512((void*)a1, _mm512_add_epi64(_mm512_loadu_si512((const void*)a1), v_f64_to_torus(im)));
      }
    }
  }
  /* sample extract per lane */
  for (int w = 0; w < count; ++w) {
    uint64_t* o = out[w];
    for (uint32_t q = 0; q < k; ++q) {
      const uint64_t* A = sc->acc + (size_t)q * N * W8;
      o[(size_t)q * N] = A[w];
      for (uint32_t j = 1; j < N; ++j) o[(size_t)q * N + j] = (uint64_t)0 - A[(size_t)(N - j) * W8 + w];
    }
    o[(size_t)k * N] = sc->acc[(size_t)k * N * W8 + w];
  }
}

typedef struct {
  const orc_ctx* c;
  const uint64_t* in;
  const int32_t* luts;
  uint64_t* out;
  size_t count;
} v_batch_arg;

static void v_range(void* a, size_t lo, size_t hi) { /* lo, hi: group indices */
  v_batch_arg* b = (v_batch_arg*)a;
  const orc_params* p = &b->c->p;
  const size_t len = (size_t)p->k * p->N + 1;
  v_scratch sc;
  sc.acc = (uint64_t*)aligned_alloc(64, sizeof(uint64_t) * W8 * (p->k + 1) * p->N);
  sc.tp = (uint64_t*)malloc(sizeof(uint64_t) * p->N);
  sc.spec = (v8c*)aligned_alloc(64, sizeof(v8c) * rows_of(p) * b->c->M);
  sc.facc = (v8c*)aligned_alloc(64, sizeof(v8c) * b->c->M);
  sc.small = (uint64_t*)malloc(sizeof(uint64_t) * W8 * (p->n + 1));
  sc.ms = (uint32_t*)malloc(sizeof(uint32_t) * W8 * (p->n + 1));
  for (size_t g = lo; g < hi; ++g) {
    const uint64_t* in[W8];
    const int32_t* luts[W8];
    uint64_t* out[W8];
    const size_t base = g * W8;
    const int count = (int)(b->count - base < W8 ? b->count - base : W8);
    for (int w = 0; w < W8; ++w) {
      const size_t t = base + (size_t)(w < count ? w : 0);
      in[w] = b->in + t * len;
      luts[w] = b->luts + 16 * t;
      out[w] = b->out + t * len;
    }
    v_pbs8(b->c, in, luts, out, count, &sc);
  }
  free(sc.acc);
  free(sc.spec);
  free(sc.facc);
  free(sc.small);
  free(sc.ms);
  free(sc.tp);
}

int orc_pbs_batch_simd(const orc_ctx* c, size_t count, const uint64_t* in, const int32_t* luts,
                       uint64_t* out, int threads) {
  if (c->p.pbs_level != 1 || c->p.exact_mask_product) return -1;
  v_batch_arg a = {c, in, luts, out, count};
  parallel_for((count + W8 - 1) / W8, threads, v_range, &a);
  return 0;
}
#else
int orc_pbs_batch_simd(const orc_ctx* c, size_t count, const uint64_t* in, const int32_t* luts,
                       uint64_t* out, int threads) {
  (void)c, (void)count, (void)in, (void)luts, (void)out, (void)threads;
  return -1; /* built without AVX-512 */
}
#endif
