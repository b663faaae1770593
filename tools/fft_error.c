/* Experiment: error of the f64 negacyclic FFT external product
 * (2 digit polys x 2 BSK polys, N = 2048, base 2^23) against the exact
 * product mod 2^64, for FFT specification variants. Not test
 * infrastructure; used to choose the FFT spec.
 *   gcc -O2 -ffp-contract=off -o /tmp/fft_error tools/fft_error.c -lm */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define N 2048
#define M 1024
#define LOGM 10

typedef long double ld;
static double tw[2 * M], twist[2 * M], untw[2 * M];
static ld twl[2 * M], twistl[2 * M];
static int R8 = 0, R4 = 0;
static void dif4(double* X);
static void dit4(double* X);
static void dif8(double* X);
static void dit8(double* X);

static uint64_t s[2] = {0x1234567, 0x89abcdef};
static uint64_t rnd(void) {
  uint64_t s1 = s[0];
  const uint64_t s0 = s[1];
  s[0] = s0;
  s1 ^= s1 << 23;
  s[1] = s1 ^ s0 ^ (s1 >> 17) ^ (s0 >> 26);
  return s[1] + s0;
}

static inline void cmul(double ar, double ai, double br, double bi, double* r, double* i) {
  double t1 = ai * bi, t2 = ai * br;
  *r = fma(ar, br, -t1);
  *i = fma(ar, bi, t2);
}

static void tables(void) {
  const ld PI = 3.141592653589793238462643383279502884L;
  for (int t = 0; t < M; ++t) {
    ld a = 2.0L * PI * t / M;
    tw[2 * t] = (double)cosl(a);
    tw[2 * t + 1] = (double)-sinl(a);
    twl[2 * t] = cosl(a);
    twl[2 * t + 1] = -sinl(a);
  }
  for (int j = 0; j < M; ++j) {
    ld a = PI * j / N;
    twistl[2 * j] = cosl(a);
    twistl[2 * j + 1] = sinl(a);
    /* fine x coarse as the spec */
    double fr = (double)cosl(PI * (j % 128) / N), fi = (double)sinl(PI * (j % 128) / N);
    double cr = (double)cosl(PI * (j / 128 * 128) / N), ci = (double)sinl(PI * (j / 128 * 128) / N);
    double r, i;
    cmul(fr, fi, cr, ci, &r, &i);
    if (getenv("PRECISE_TWIST")) {
      r = (double)twistl[2 * j];
      i = (double)twistl[2 * j + 1];
    }
    twist[2 * j] = r;
    twist[2 * j + 1] = i;
    untw[2 * j] = r / M;
    untw[2 * j + 1] = -i / M;
  }
}

static void dif(double* x) {
  for (int s = 0; s < LOGM; ++s) {
    int half = M >> (s + 1);
    for (int b = 0; b < M; b += 2 * half)
      for (int j = 0; j < half; ++j) {
        double* u = x + 2 * (b + j);
        double* v = x + 2 * (b + j + half);
        const double* w = tw + 2 * (j << s);
        double sr = u[0] + v[0], si = u[1] + v[1], tr = u[0] - v[0], ti = u[1] - v[1];
        u[0] = sr;
        u[1] = si;
        cmul(tr, ti, w[0], w[1], &v[0], &v[1]);
      }
  }
}
static void dit(double* x) {
  for (int s = LOGM - 1; s >= 0; --s) {
    int half = M >> (s + 1);
    for (int b = 0; b < M; b += 2 * half)
      for (int j = 0; j < half; ++j) {
        double* p = x + 2 * (b + j);
        double* q = x + 2 * (b + j + half);
        const double* w = tw + 2 * (j << s);
        double qr, qi;
        cmul(q[0], q[1], w[0], -w[1], &qr, &qi);
        double pr = p[0], pi = p[1];
        p[0] = pr + qr;
        p[1] = pi + qi;
        q[0] = pr - qr;
        q[1] = pi - qi;
      }
  }
}
static void difl(ld* x) {
  for (int s = 0; s < LOGM; ++s) {
    int half = M >> (s + 1);
    for (int b = 0; b < M; b += 2 * half)
      for (int j = 0; j < half; ++j) {
        ld* u = x + 2 * (b + j);
        ld* v = x + 2 * (b + j + half);
        const ld* w = twl + 2 * (j << s);
        ld sr = u[0] + v[0], si = u[1] + v[1], tr = u[0] - v[0], ti = u[1] - v[1];
        u[0] = sr;
        u[1] = si;
        v[0] = tr * w[0] - ti * w[1];
        v[1] = tr * w[1] + ti * w[0];
      }
  }
}

static void fwd(const int64_t* a, double* out) {
  for (int j = 0; j < M; ++j) cmul((double)a[j], (double)a[j + M], twist[2 * j], twist[2 * j + 1], &out[2 * j], &out[2 * j + 1]);
  if (R4) dif4(out); else if (R8) dif8(out); else dif(out);
}
static void fwd_ld(const int64_t* a, double* out) {
  ld x[2 * M];
  for (int j = 0; j < M; ++j) {
    ld re = (ld)a[j], im = (ld)a[j + M];
    x[2 * j] = re * twistl[2 * j] - im * twistl[2 * j + 1];
    x[2 * j + 1] = re * twistl[2 * j + 1] + im * twistl[2 * j];
  }
  difl(x);
  for (int j = 0; j < 2 * M; ++j) out[j] = (double)x[j];
}
static void ditl(ld* x) {
  for (int s = LOGM - 1; s >= 0; --s) {
    int half = M >> (s + 1);
    for (int b = 0; b < M; b += 2 * half)
      for (int j = 0; j < half; ++j) {
        ld* p = x + 2 * (b + j);
        ld* q = x + 2 * (b + j + half);
        const ld* w = twl + 2 * (j << s);
        ld qr = q[0] * w[0] + q[1] * w[1], qi = q[1] * w[0] - q[0] * w[1];
        ld pr = p[0], pi = p[1];
        p[0] = pr + qr;
        p[1] = pi + qi;
        q[0] = pr - qr;
        q[1] = pi - qi;
      }
  }
}
static uint64_t f2t(double y) {
  double r = rint(y * 0x1p-64);
  double d = y - r * 18446744073709551616.0;
  if (d >= 9223372036854775808.0) d -= 18446744073709551616.0;
  return (uint64_t)(int64_t)llrint(d);
}
/* ---- radix-8 passes (8 x 8 x 8 x 2) ---- */
static const double C8 = 0.70710678118654752440;
static inline int brev3(int r) { return ((r & 1) << 2) | (r & 2) | ((r >> 2) & 1); }
typedef struct { double x, y; } c2;
static inline c2 add(c2 a, c2 b) { return (c2){a.x + b.x, a.y + b.y}; }
static inline c2 sub(c2 a, c2 b) { return (c2){a.x - b.x, a.y - b.y}; }
static inline c2 mulw(c2 a, const double* w) { c2 r; cmul(a.x, a.y, w[0], w[1], &r.x, &r.y); return r; }
static inline c2 mulwc(c2 a, const double* w) { c2 r; cmul(a.x, a.y, w[0], -w[1], &r.x, &r.y); return r; }
static inline c2 mul_mi(c2 a) { return (c2){a.y, -a.x}; }   /* * -i */
static inline c2 mul_pi(c2 a) { return (c2){-a.y, a.x}; }   /* * +i */
static inline c2 mul_w81(c2 a) { return (c2){(a.x + a.y) * C8, (a.y - a.x) * C8}; }
static inline c2 mul_w83(c2 a) { return (c2){(a.y - a.x) * C8, (a.x + a.y) * -C8}; }
static inline c2 mul_w81c(c2 a) { return (c2){(a.x - a.y) * C8, (a.x + a.y) * C8}; }
static inline c2 mul_w83c(c2 a) { return (c2){(a.x + a.y) * -C8, (a.x - a.y) * C8}; }
static void dft8(c2* a) {
  c2 b[8];
  for (int r = 0; r < 4; ++r) { b[r] = add(a[r], a[r + 4]); b[r + 4] = sub(a[r], a[r + 4]); }
  b[5] = mul_w81(b[5]); b[6] = mul_mi(b[6]); b[7] = mul_w83(b[7]);
  for (int r = 0; r < 8; r += 4) {
    c2 s0 = add(b[r], b[r + 2]), d0 = sub(b[r], b[r + 2]);
    c2 s1 = add(b[r + 1], b[r + 3]), d1 = mul_mi(sub(b[r + 1], b[r + 3]));
    a[r] = add(s0, s1); a[r + 1] = sub(s0, s1); a[r + 2] = add(d0, d1); a[r + 3] = sub(d0, d1);
  }
}
static void idft8(c2* a) {
  c2 b[8];
  for (int r = 0; r < 8; r += 4) {
    c2 s0 = add(a[r], a[r + 1]), d0 = sub(a[r], a[r + 1]);
    c2 s1 = add(a[r + 2], a[r + 3]), d1 = sub(a[r + 2], a[r + 3]);
    d1 = mul_pi(d1);
    b[r] = add(s0, s1); b[r + 2] = sub(s0, s1); b[r + 1] = add(d0, d1); b[r + 3] = sub(d0, d1);
  }
  b[5] = mul_w81c(b[5]); b[6] = mul_pi(b[6]); b[7] = mul_w83c(b[7]);
  for (int r = 0; r < 4; ++r) { a[r] = add(b[r], b[r + 4]); a[r + 4] = sub(b[r], b[r + 4]); }
}
static void dif8(double* X) {
  c2* x = (c2*)X;
  for (int p = 0; p < 3; ++p) {
    const int span = 128 >> (3 * p); /* 128, 16, 2 */
    for (int base = 0; base < M; base += 8 * span)
      for (int n1 = 0; n1 < span; ++n1) {
        c2 a[8];
        for (int r = 0; r < 8; ++r) a[r] = x[base + n1 + span * r];
        dft8(a);
        for (int r = 1; r < 8; ++r)
          if (n1) a[r] = mulw(a[r], tw + 2 * ((n1 * brev3(r)) << (3 * p)));
        for (int r = 0; r < 8; ++r) x[base + n1 + span * r] = a[r];
      }
  }
  for (int j = 0; j < M; j += 2) { c2 u = x[j], v = x[j + 1]; x[j] = add(u, v); x[j + 1] = sub(u, v); }
}
static void dit8(double* X) {
  c2* x = (c2*)X;
  for (int j = 0; j < M; j += 2) { c2 u = x[j], v = x[j + 1]; x[j] = add(u, v); x[j + 1] = sub(u, v); }
  for (int p = 2; p >= 0; --p) {
    const int span = 128 >> (3 * p);
    for (int base = 0; base < M; base += 8 * span)
      for (int n1 = 0; n1 < span; ++n1) {
        c2 a[8];
        for (int r = 0; r < 8; ++r) a[r] = x[base + n1 + span * r];
        for (int r = 1; r < 8; ++r)
          if (n1) a[r] = mulwc(a[r], tw + 2 * ((n1 * brev3(r)) << (3 * p)));
        idft8(a);
        for (int r = 0; r < 8; ++r) x[base + n1 + span * r] = a[r];
      }
  }
}

/* ---- radix-4 on stage pairs (0,1), (3,4), (6,7); radix-2 stages 2,5,8,9 ---- */

static void r2_dif_stage(c2* x, int s) {
  const int half = M >> (s + 1);
  for (int b = 0; b < M; b += 2 * half)
    for (int j = 0; j < half; ++j) {
      c2 u = x[b + j], v = x[b + j + half];
      x[b + j] = add(u, v);
      x[b + j + half] = (j << s) ? mulw(sub(u, v), tw + 2 * (j << s)) : sub(u, v);
    }
}
static void r4_dif_stages(c2* x, int s) {  /* stages s, s+1 */
  const int H = M >> (s + 2);
  for (int b = 0; b < M; b += 4 * H)
    for (int j = 0; j < H; ++j) {
      const int k = j << s;
      c2 x0 = x[b + j], x1 = x[b + j + H], x2 = x[b + j + 2 * H], x3 = x[b + j + 3 * H];
      c2 A = add(x0, x2), B = add(x1, x3), C = sub(x0, x2), D = mul_mi(sub(x1, x3));
      x[b + j] = add(A, B);
      x[b + j + H] = k ? mulw(sub(A, B), tw + 2 * (2 * k)) : sub(A, B);
      x[b + j + 2 * H] = k ? mulw(add(C, D), tw + 2 * k) : add(C, D);
      x[b + j + 3 * H] = k ? mulw(sub(C, D), tw + 2 * ((3 * k) % M)) : sub(C, D);
    }
}
static void dif4(double* X) {
  c2* x = (c2*)X;
  r4_dif_stages(x, 0); r2_dif_stage(x, 2);
  r4_dif_stages(x, 3); r2_dif_stage(x, 5);
  r4_dif_stages(x, 6); r2_dif_stage(x, 8);
  r2_dif_stage(x, 9);
}
static void r2_dit_stage(c2* x, int s) {
  const int half = M >> (s + 1);
  for (int b = 0; b < M; b += 2 * half)
    for (int j = 0; j < half; ++j) {
      c2 p = x[b + j], q = x[b + j + half];
      if (j << s) q = mulwc(q, tw + 2 * (j << s));
      x[b + j] = add(p, q);
      x[b + j + half] = sub(p, q);
    }
}
static void r4_dit_stages(c2* x, int s) {  /* stages s+1 then s */
  const int H = M >> (s + 2);
  for (int b = 0; b < M; b += 4 * H)
    for (int j = 0; j < H; ++j) {
      const int k = j << s;
      c2 x0 = x[b + j], x1 = x[b + j + H], x2 = x[b + j + 2 * H], x3 = x[b + j + 3 * H];
      c2 t1 = k ? mulwc(x1, tw + 2 * (2 * k)) : x1;
      c2 t2 = k ? mulwc(x2, tw + 2 * k) : x2;
      c2 t3 = k ? mulwc(x3, tw + 2 * ((3 * k) % M)) : x3;
      c2 A = add(x0, t1), B = sub(x0, t1), C = add(t2, t3), D = mul_pi(sub(t2, t3));
      x[b + j] = add(A, C);
      x[b + j + 2 * H] = sub(A, C);
      x[b + j + H] = add(B, D);
      x[b + j + 3 * H] = sub(B, D);
    }
}
static void dit4(double* X) {
  c2* x = (c2*)X;
  r2_dit_stage(x, 9);
  r2_dit_stage(x, 8); r4_dit_stages(x, 6);
  r2_dit_stage(x, 5); r4_dit_stages(x, 3);
  r2_dit_stage(x, 2); r4_dit_stages(x, 0);
}

static void bwd(double* x, uint64_t* out) {
  if (R4) dit4(x); else
  if (R8) dit8(x); else
  dit(x);
  for (int j = 0; j < M; ++j) {
    double re, im;
    cmul(x[2 * j], x[2 * j + 1], untw[2 * j], untw[2 * j + 1], &re, &im);
    out[j] = f2t(re);
    out[j + M] = f2t(im);
  }
}

static void bwd_ld(const double* xin, uint64_t* out) {
  ld x[2 * M];
  for (int j = 0; j < 2 * M; ++j) x[j] = xin[j];
  ditl(x);
  for (int j = 0; j < M; ++j) {
    ld re = (x[2 * j] * twistl[2 * j] + x[2 * j + 1] * twistl[2 * j + 1]) / M;
    ld im = (x[2 * j + 1] * twistl[2 * j] - x[2 * j] * twistl[2 * j + 1]) / M;
    ld r1 = rintl(re * 0x1p-64L), r2 = rintl(im * 0x1p-64L);
    out[j] = (uint64_t)(int64_t)llrintl(re - r1 * 18446744073709551616.0L);
    out[j + M] = (uint64_t)(int64_t)llrintl(im - r2 * 18446744073709551616.0L);
  }
}
static void exact(const int64_t* d, const uint64_t* b, uint64_t* acc) {
  for (int i = 0; i < N; ++i) {
    if (!d[i]) continue;
    uint64_t di = (uint64_t)d[i];
    for (int j = 0; j < N; ++j) {
      uint64_t p = di * b[j];
      int k = i + j;
      if (k < N) acc[k] += p;
      else acc[k - N] -= p;
    }
  }
}

int main(int argc, char** argv) {
  int trials = argc > 1 ? atoi(argv[1]) : 8;
  tables();
  R8 = getenv("R8") != NULL;
  R4 = getenv("R4") != NULL;
  if (R4) {
    static double a[2 * M], b2[2 * M];
    for (int j = 0; j < 2 * M; ++j) a[j] = b2[j] = (double)(int)(rnd() % 2001) - 1000;
    dif(a); dif4(b2);
    double e = 0; for (int j = 0; j < 2 * M; ++j) e = fmax(e, fabs(a[j] - b2[j]));
    printf("dif4 vs dif max diff %.3g\n", e);
    dit4(b2); dit(a);
    e = 0; for (int j = 0; j < 2 * M; ++j) e = fmax(e, fabs(a[j] - b2[j]));
    printf("dit4 vs dit max diff %.3g\n", e);
  }
  if (R8) { /* consistency: dif8 == dif up to rounding, dit8(dif8(x)) == M x */
    static double a[2 * M], b2[2 * M];
    for (int j = 0; j < 2 * M; ++j) a[j] = b2[j] = (double)(int)(rnd() % 2001) - 1000;
    dif(a); dif8(b2);
    double e = 0; for (int j = 0; j < 2 * M; ++j) e = fmax(e, fabs(a[j] - b2[j]));
    printf("dif8 vs dif max diff %.3g\n", e);
    dit8(b2); dit(a);
    e = 0; for (int j = 0; j < 2 * M; ++j) e = fmax(e, fabs(a[j] - b2[j]));
    printf("dit8 vs dit max diff %.3g\n", e);
  }
  static int64_t d[2][N];
  static uint64_t b[2][N], ex[N], out[N];
  static double D[2][2 * M], B[2][2 * M], A[2 * M];
  double var[8] = {0};
  long cnt = 0;
  for (int t = 0; t < trials; ++t) {
    for (int r = 0; r < 2; ++r)
      for (int j = 0; j < N; ++j) {
        d[r][j] = (int64_t)(rnd() & ((1u << 23) - 1)) - (1 << 22);
        b[r][j] = rnd();
      }
    memset(ex, 0, sizeof ex);
    for (int r = 0; r < 2; ++r) exact(d[r], b[r], ex);
    for (int v = 0; v < 4; ++v) {
      /* v bit0: BSK spectrum in long double; v bit1: digits spectrum + inverse in long double */
      for (int r = 0; r < 2; ++r) {
        if (v & 2) fwd_ld(d[r], D[r]); else fwd(d[r], D[r]);
        if (v & 1) fwd_ld((const int64_t*)b[r], B[r]);
        else fwd((const int64_t*)b[r], B[r]);
      }
      memset(A, 0, sizeof A);
      for (int r = 0; r < 2; ++r)
        for (int f = 0; f < M; ++f) {
          double ar = A[2 * f], ai = A[2 * f + 1];
          ar = fma(D[r][2 * f], B[r][2 * f], ar);
          ar = fma(-D[r][2 * f + 1], B[r][2 * f + 1], ar);
          ai = fma(D[r][2 * f], B[r][2 * f + 1], ai);
          ai = fma(D[r][2 * f + 1], B[r][2 * f], ai);
          A[2 * f] = ar;
          A[2 * f + 1] = ai;
        }
      if (v & 2) bwd_ld(A, out); else bwd(A, out);
      static int64_t errv[4][N], maskv[4][N];
      static uint8_t key[N];
      for (int j = 0; j < N; ++j) {
        errv[v][j] = (int64_t)(out[j] - ex[j]);
        double e = (double)errv[v][j];
        var[v] += e * e;
      }
      /* phase error of a GLWE whose mask error is the previous trial's and
       * body error this trial's: e_B - e_A * S (binary S), var per coeff */
      if (t & 1) {
        if (v == 0)
          for (int j = 0; j < N; ++j) key[j] = rnd() & 1;
        for (int j = 0; j < N; ++j) {
          int64_t acc = errv[v][j];
          for (int u = 0; u < N; ++u) {
            if (!key[u]) continue;
            acc -= (j >= u) ? maskv[v][j - u] : -maskv[v][j - u + N];
          }
          var[4 + v] += (double)acc * (double)acc;
        }
      } else {
        memcpy(maskv[v], errv[v], sizeof errv[v]);
      }
    }
    cnt += N;
  }
  for (int v = 0; v < 4; ++v)
    printf("variant %d: coefficient error std 2^%.3f, phase error std 2^%.3f\n", v,
           0.5 * log2(var[v] / cnt), 0.5 * log2(var[4 + v] / (cnt / 2)));
  return 0;
}
