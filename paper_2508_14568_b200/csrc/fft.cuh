// Negacyclic f64 FFT for N = 2048 (1024-point complex DIF forward, DIT
// inverse), 128 threads per transform, 8 complex values per thread, P
// polynomials processed in lockstep by the same threads.
//
// Bit-exactness contract with oracle/tfhe_oracle.c (fft_dif,
// fft_dit_inverse, forward_i64, backward_torus): every butterfly performs
// exactly the oracle's IEEE operations — __dadd_rn/__dsub_rn for sums,
// cmul() = {fma(a.x,b.x,-(a.y*b.y)), fma(a.x,b.y,(a.y*b.x))} for twiddles —
// with the same twiddle table entries. Only the data movement differs
// (registers, a swizzled shared buffer, lane shuffles), which cannot change
// a rounding. Multiplications by W[0] = (1,-0) are skipped: they are exact
// up to the sign of zero, which never reaches a nonzero result.
//
// Thread layouts (t = threadIdx.x in [0,128), r = register index 0..7):
//   fwd A  (stages 0-2) : x = t + 128 r
//   fwd B  (stages 3-5) : t = 16 b + u,   x = 128 b + u + 16 r
//   fwd C  (stages 6-8) : t = 2 c + v,    x = 16 c + v + 2 r
//   fwd stage 9 via shfl.xor 1 -> thread t owns spectrum bins 8t .. 8t+7
//   inv    (stages 9-7) : bins 8t + r
//   inv B' (stages 6-4) : t = 8 b + u,    x = 64 b + u + 8 r
//   inv A' (stages 3-1) : t = 32 w + 16 h + s, u = 16 w + s, x = 512 h + u + 64 r
//   inv stage 0 via shfl.xor 16
// Shared buffer index swizzle swz(x) keeps every one of these patterns
// free of bank conflicts (16-byte elements, 8 lanes per 128-byte wavefront).
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace lvb {

__device__ __forceinline__ uint32_t swz(uint32_t x) {
  return x ^ ((((x >> 3) & 7u) ^ (((x >> 9) & 1u) << 2)));
}

// Exchange through shared memory: one polynomial at a time through a
// single kM-entry buffer (16 KB) instead of all P at once, so the blind
// rotation fits 4 CTAs per SM. Set LVB_SPLIT_XCHG=0 for the P-buffer form.
#ifndef LVB_SPLIT_XCHG
#define LVB_SPLIT_XCHG 1
#endif
constexpr bool kSplitXchg = LVB_SPLIT_XCHG;
constexpr int kXchgBufs = kSplitXchg ? 1 : 2;

// Moves X from layout wr(r) to layout rd(r) (element indices x); the caller
// guarantees the buffer is free on entry.
template <int P, typename WR, typename RD>
__device__ __forceinline__ void xchg(double2 (&X)[P][8], double2* buf, WR wr, RD rd) {
#ifdef LVB_ABL_XCHG  // timing ablation only: results are wrong
  __syncthreads();
  return;
#endif
  if constexpr (!kSplitXchg || P == 1) {
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 8; ++r) buf[p * kM + swz(wr(r))] = X[p][r];
    __syncthreads();
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 8; ++r) X[p][r] = buf[p * kM + swz(rd(r))];
  } else {
#pragma unroll
    for (int p = 0; p < P; ++p) {
      if (p) __syncthreads();
#pragma unroll
      for (int r = 0; r < 8; ++r) buf[swz(wr(r))] = X[p][r];
      __syncthreads();
#pragma unroll
      for (int r = 0; r < 8; ++r) X[p][r] = buf[swz(rd(r))];
    }
  }
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  const double t1 = __dmul_rn(a.y, b.y);
  const double t2 = __dmul_rn(a.y, b.x);
  return make_double2(__fma_rn(a.x, b.x, -t1), __fma_rn(a.x, b.y, t2));
}

// a * conj(b), as the oracle computes cmul(q, (w.re, -w.im)).
__device__ __forceinline__ double2 cmul_conj(double2 a, double2 b) {
  const double nbi = -b.y;
  const double t1 = __dmul_rn(a.y, nbi);
  const double t2 = __dmul_rn(a.y, b.x);
  return make_double2(__fma_rn(a.x, b.x, -t1), __fma_rn(a.x, nbi, t2));
}

__device__ __forceinline__ void dif(double2& u, double2& v, double2 w) {
  const double2 s = make_double2(__dadd_rn(u.x, v.x), __dadd_rn(u.y, v.y));
  const double2 d = make_double2(__dsub_rn(u.x, v.x), __dsub_rn(u.y, v.y));
  u = s;
  v = cmul(d, w);
}

__device__ __forceinline__ void dif1(double2& u, double2& v) {  // w = W[0]
  const double2 s = make_double2(__dadd_rn(u.x, v.x), __dadd_rn(u.y, v.y));
  const double2 d = make_double2(__dsub_rn(u.x, v.x), __dsub_rn(u.y, v.y));
  u = s;
  v = d;
}

__device__ __forceinline__ void dit(double2& p, double2& q, double2 w) {
  const double2 qw = cmul_conj(q, w);
  const double2 a = make_double2(__dadd_rn(p.x, qw.x), __dadd_rn(p.y, qw.y));
  const double2 b = make_double2(__dsub_rn(p.x, qw.x), __dsub_rn(p.y, qw.y));
  p = a;
  q = b;
}

__device__ __forceinline__ void dit1(double2& p, double2& q) {  // w = W[0]
  const double2 a = make_double2(__dadd_rn(p.x, q.x), __dadd_rn(p.y, q.y));
  const double2 b = make_double2(__dsub_rn(p.x, q.x), __dsub_rn(p.y, q.y));
  p = a;
  q = b;
}

// Per-stage twiddle tables T_s[y] = W[y << s] (W[k] = exp(-2 pi i k / kM)),
// concatenated: T_s starts at kM - (kM >> s). Same values as W, laid out so
// every warp-wide twiddle load is contiguous.
__device__ __forceinline__ double2 tws(const double2* __restrict__ tw, int s, uint32_t y) {
#ifdef LVB_ABL_TW  // timing ablation only
  return make_double2(0.70710678118654757 + s * 1e-3, 0.70710678118654757 - y * 1e-9);
#endif
  return __ldg(tw + (kM - (kM >> s)) + y);
}

// Coarse twist factors zeta^(128 k), k < 8 (constant bank).
__constant__ double2 c_twist_coarse[8];  // defined here: fft.cuh has one includer (kernels.cu)

// zeta^x = fine[x & 127] * coarse[x >> 7] (oracle build_tables defines the
// twist this way); coarse[0] = 1 is an exact identity and is skipped.
__device__ __forceinline__ double2 twist_at(const double2* __restrict__ fine, uint32_t x) {
  const double2 f = __ldg(fine + (x & 127));
  return (x >> 7) == 0 ? f : cmul(f, c_twist_coarse[x >> 7]);
}

__device__ __forceinline__ double2 shfl_xor_d2(double2 v, int m) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
}

// ---------------------------------------------------------------- forward
// X[p][r] on entry: twisted inputs at x = t + 128 r. On exit: spectrum
// bins 8t + r. buf: P shared buffers of kM double2 each.
template <int P>
__device__ __forceinline__ void fft_forward(double2 (&X)[P][8], double2* buf,
                                            const double2* __restrict__ tw, uint32_t t) {
  // group A: stages 0,1,2
  {
    double2 w0[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) w0[r] = tws(tw, 0, t + 128 * r);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 4; ++r) dif(X[p][r], X[p][r + 4], w0[r]);
    const double2 w10 = tws(tw, 1, t), w11 = tws(tw, 1, t + 128);
#pragma unroll
    for (int p = 0; p < P; ++p) {
      dif(X[p][0], X[p][2], w10);
      dif(X[p][1], X[p][3], w11);
      dif(X[p][4], X[p][6], w10);
      dif(X[p][5], X[p][7], w11);
    }
    const double2 w2 = tws(tw, 2, t);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 8; r += 2) dif(X[p][r], X[p][r + 1], w2);
  }
  // A -> B
  {
    const uint32_t b = t >> 4, u = t & 15;
    xchg<P>(X, buf, [&](int r) { return t + 128 * r; },
            [&](int r) { return 128 * b + u + 16 * r; });
    double2 w3[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) w3[r] = tws(tw, 3, u + 16 * r);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 4; ++r) dif(X[p][r], X[p][r + 4], w3[r]);
    const double2 w40 = tws(tw, 4, u), w41 = tws(tw, 4, u + 16);
#pragma unroll
    for (int p = 0; p < P; ++p) {
      dif(X[p][0], X[p][2], w40);
      dif(X[p][1], X[p][3], w41);
      dif(X[p][4], X[p][6], w40);
      dif(X[p][5], X[p][7], w41);
    }
    const double2 w5 = tws(tw, 5, u);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 8; r += 2) dif(X[p][r], X[p][r + 1], w5);
    __syncthreads();
    const uint32_t c = t >> 1, v = t & 1;
    xchg<P>(X, buf, [&](int r) { return 128 * b + u + 16 * r; },
            [&](int r) { return 16 * c + v + 2 * r; });
  }
  {
    const uint32_t v = t & 1;
    double2 w6[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) w6[r] = tws(tw, 6, v + 2 * r);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 4; ++r) dif(X[p][r], X[p][r + 4], w6[r]);
    const double2 w70 = tws(tw, 7, v), w71 = tws(tw, 7, v + 2);
#pragma unroll
    for (int p = 0; p < P; ++p) {
      dif(X[p][0], X[p][2], w70);
      dif(X[p][1], X[p][3], w71);
      dif(X[p][4], X[p][6], w70);
      dif(X[p][5], X[p][7], w71);
    }
    const double2 w8 = tws(tw, 8, v);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 8; r += 2) dif(X[p][r], X[p][r + 1], w8);
    // stage 9: pairs (16c + 2r, 16c + 2r + 1) live in lanes (2c, 2c+1).
#pragma unroll
    for (int p = 0; p < P; ++p) {
      double2 Y[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) Y[q] = shfl_xor_d2(v ? X[p][q] : X[p][4 + q], 1);
      double2 F[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double2 e = v ? Y[q] : X[p][q];
        double2 o = v ? X[p][4 + q] : Y[q];
        dif1(e, o);
        F[2 * q] = e;
        F[2 * q + 1] = o;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) X[p][q] = F[q];
    }
  }
}

// ---------------------------------------------------------------- inverse
// X[p][r] on entry: spectrum bins 8t + r. On exit: for h = (t>>4)&1,
// u = 16 (t>>5) + (t&15), q = 0..3: X[p][q] = z at x = u + 64 (4h + q),
// X[p][4+q] = z at x + 512 (before untwist). Buffer reuse is guarded by the
// caller's __syncthreads before entry.
template <int P>
__device__ __forceinline__ void fft_inverse(double2 (&X)[P][8], double2* buf,
                                            const double2* __restrict__ tw, uint32_t t) {
  {
    // stage 9 (half 1), 8 (half 2), 7 (half 4) on the thread's 8 bins
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 8; r += 2) dit1(X[p][r], X[p][r + 1]);
    const double2 w81 = tws(tw, 8, 1);
#pragma unroll
    for (int p = 0; p < P; ++p) {
      dit1(X[p][0], X[p][2]);
      dit(X[p][1], X[p][3], w81);
      dit1(X[p][4], X[p][6]);
      dit(X[p][5], X[p][7], w81);
    }
    const double2 w71 = tws(tw, 7, 1), w72 = tws(tw, 7, 2), w73 = tws(tw, 7, 3);
#pragma unroll
    for (int p = 0; p < P; ++p) {
      dit1(X[p][0], X[p][4]);
      dit(X[p][1], X[p][5], w71);
      dit(X[p][2], X[p][6], w72);
      dit(X[p][3], X[p][7], w73);
    }
  }
  {
    const uint32_t b = t >> 3, u = t & 7;
    xchg<P>(X, buf, [&](int r) { return 8 * t + r; }, [&](int r) { return 64 * b + u + 8 * r; });
    const double2 w6 = tws(tw, 6, u);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 8; r += 2) dit(X[p][r], X[p][r + 1], w6);
    const double2 w50 = tws(tw, 5, u), w51 = tws(tw, 5, u + 8);
#pragma unroll
    for (int p = 0; p < P; ++p) {
      dit(X[p][0], X[p][2], w50);
      dit(X[p][1], X[p][3], w51);
      dit(X[p][4], X[p][6], w50);
      dit(X[p][5], X[p][7], w51);
    }
    double2 w4[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) w4[r] = tws(tw, 4, u + 8 * r);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 4; ++r) dit(X[p][r], X[p][r + 4], w4[r]);
    __syncthreads();
    const uint32_t h = (t >> 4) & 1, u2 = 16 * (t >> 5) + (t & 15);
    xchg<P>(X, buf, [&](int r) { return 64 * b + u + 8 * r; },
            [&](int r) { return 512 * h + u2 + 64 * r; });
  }
  {
    const uint32_t h = (t >> 4) & 1, u = 16 * (t >> 5) + (t & 15);
    const double2 w3 = tws(tw, 3, u);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 8; r += 2) dit(X[p][r], X[p][r + 1], w3);
    const double2 w20 = tws(tw, 2, u), w21 = tws(tw, 2, u + 64);
#pragma unroll
    for (int p = 0; p < P; ++p) {
      dit(X[p][0], X[p][2], w20);
      dit(X[p][1], X[p][3], w21);
      dit(X[p][4], X[p][6], w20);
      dit(X[p][5], X[p][7], w21);
    }
    double2 w1[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) w1[r] = tws(tw, 1, u + 64 * r);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 4; ++r) dit(X[p][r], X[p][r + 4], w1[r]);
    // stage 0 (half 512): lane pairs (t, t^16) hold x and x + 512.
    double2 w0[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) w0[q] = tws(tw, 0, u + 64 * (4 * h + q));
#pragma unroll
    for (int p = 0; p < P; ++p) {
      double2 Y[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) Y[q] = shfl_xor_d2(h ? X[p][q] : X[p][4 + q], 16);
      double2 Z[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double2 lo = h ? Y[q] : X[p][q];
        double2 hi = h ? X[p][4 + q] : Y[q];
        dit(lo, hi, w0[q]);
        Z[q] = lo;
        Z[4 + q] = hi;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) X[p][q] = Z[q];
    }
  }
}

// ------------------------------------------------ inverse, natural layout A
// Same arithmetic as fft_inverse (DIT stages 9..0), different data path:
//   stages 9,8,7 on the thread's bins 8t + r            (registers)
//   -> B' (t = 8b + u, x = 64b + u + 8r): stages 6,5,4  (shared exchange)
//   stage 3 (pairs x, x+64 in lanes t, t^8)             (shfl.xor 8)
//   -> A  (x = t + 128 r): stages 2,1,0                 (shared exchange)
// so the output lands in the layout fft_forward's input uses: each thread
// owns the same accumulator coefficients in both halves of a CMUX.
template <int P>
__device__ __forceinline__ void fft_inverse_a(double2 (&X)[P][8], double2* buf,
                                              const double2* __restrict__ tw, uint32_t t) {
  {
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 8; r += 2) dit1(X[p][r], X[p][r + 1]);
    const double2 w81 = tws(tw, 8, 1);
#pragma unroll
    for (int p = 0; p < P; ++p) {
      dit1(X[p][0], X[p][2]);
      dit(X[p][1], X[p][3], w81);
      dit1(X[p][4], X[p][6]);
      dit(X[p][5], X[p][7], w81);
    }
    const double2 w71 = tws(tw, 7, 1), w72 = tws(tw, 7, 2), w73 = tws(tw, 7, 3);
#pragma unroll
    for (int p = 0; p < P; ++p) {
      dit1(X[p][0], X[p][4]);
      dit(X[p][1], X[p][5], w71);
      dit(X[p][2], X[p][6], w72);
      dit(X[p][3], X[p][7], w73);
    }
  }
  const uint32_t b = t >> 3, u = t & 7, odd = b & 1;
  xchg<P>(X, buf, [&](int r) { return 8 * t + r; }, [&](int r) { return 64 * b + u + 8 * r; });
  {
    const double2 w6 = tws(tw, 6, u);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 8; r += 2) dit(X[p][r], X[p][r + 1], w6);
    const double2 w50 = tws(tw, 5, u), w51 = tws(tw, 5, u + 8);
#pragma unroll
    for (int p = 0; p < P; ++p) {
      dit(X[p][0], X[p][2], w50);
      dit(X[p][1], X[p][3], w51);
      dit(X[p][4], X[p][6], w50);
      dit(X[p][5], X[p][7], w51);
    }
    double2 w4[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) w4[r] = tws(tw, 4, u + 8 * r);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 4; ++r) dit(X[p][r], X[p][r + 4], w4[r]);
    // stage 3 (half 64): even b holds x, odd b holds x + 64; even lane
    // finishes r = 0..3, odd lane r = 4..7
    double2 w3[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) w3[q] = tws(tw, 3, u + 8 * (q + 4 * odd));
#pragma unroll
    for (int p = 0; p < P; ++p) {
      double2 Y[4];
      // even lane needs the odd lane's X[q] (upper of r=q); odd lane needs
      // the even lane's X[4+q] (lower of r=4+q)
#pragma unroll
      for (int q = 0; q < 4; ++q) Y[q] = shfl_xor_d2(odd ? X[p][q] : X[p][4 + q], 8);
      double2 Z[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double2 lo = odd ? Y[q] : X[p][q];
        double2 hi = odd ? X[p][4 + q] : Y[q];
        dit(lo, hi, w3[q]);
        Z[q] = lo;
        Z[4 + q] = hi;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) X[p][q] = Z[q];
    }
  }
  __syncthreads();
  xchg<P>(
      X, buf,
      [&](int r) { return 64 * (b & ~1u) + u + 8 * ((r & 3) + 4 * odd) + 64 * (r >> 2); },
      [&](int r) { return t + 128 * r; });
  {
    const double2 w2 = tws(tw, 2, t);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 8; r += 2) dit(X[p][r], X[p][r + 1], w2);
    const double2 w10 = tws(tw, 1, t), w11 = tws(tw, 1, t + 128);
#pragma unroll
    for (int p = 0; p < P; ++p) {
      dit(X[p][0], X[p][2], w10);
      dit(X[p][1], X[p][3], w11);
      dit(X[p][4], X[p][6], w10);
      dit(X[p][5], X[p][7], w11);
    }
    double2 w0[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) w0[r] = tws(tw, 0, t + 128 * r);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 4; ++r) dit(X[p][r], X[p][r + 4], w0[r]);
  }
}

// f64 -> Z_{2^64}, identical to oracle f64_to_torus. (An integer-pipe
// variant — exponent/mantissa shift for |y| >= 2^52 — measured slower on
// B200, 87-90 ms vs 82.5 ms per 4096 PBS, and was dropped.)
// Here r = floor(y 2^-64 + 1/2) (exact: |y 2^-64| < 2^32, so the sum keeps
// every bit) differs from the oracle's rint only on exact ties, where it
// yields d = -2^63 instead of +2^63 - 2^64 — the same residue — so no tie
// fix-up is needed, and d = y - r 2^64 is one exact FMA.
__device__ __forceinline__ uint64_t f64_to_torus(double y) {
  const double r = floor(__dadd_rn(__dmul_rn(y, 0x1p-64), 0.5));
  const double d = __fma_rn(-r, 18446744073709551616.0, y);
  return (uint64_t)__double2ll_rn(d);
}

}  // namespace lvb
