// Negacyclic f64 FFT for N = 2048 (1024-point complex DIF forward, DIT
// inverse), 128 threads per transform, 8 complex values per thread, P
// polynomials processed in lockstep by the same threads.
//
// Bit-exactness contract with oracle/tfhe_oracle.c (fft_dif,
// fft_dit_inverse, forward_i64, backward_torus): the network is fixed —
// forward: radix-4 DIF butterflies on the stage pairs (0,1), (3,4), (6,7),
// radix-2 stages 2, 5, 8, 9; inverse: radix-2 DIT stage 9, radix-4 (8,7),
// radix-2 6, radix-4 (5,4), radix-2 3 and 2, radix-4 (1,0) — and every
// butterfly performs exactly the oracle's IEEE operations (__dadd_rn /
// __dsub_rn for sums, cmul() = {fma(a.x,b.x,-(a.y*b.y)), fma(a.x,b.y,(a.y*b.x))}
// for twiddles, the same table entries). Only the data movement differs
// (registers, a swizzled shared buffer, lane shuffles), which cannot change
// a rounding. Multiplications by W^0 = (1,-0) that are static are skipped:
// they are exact up to the sign of zero, which never reaches a nonzero result.
// The radix-4 pairing saves a quarter of those stages' twiddle products
// (-8% FP64 instructions per transform) and rounds no more often
// (tools/fft_error.c: external-product error std 2^37.96 vs 2^38.00).
//
// Thread layouts (t = threadIdx.x in [0,128), r = register index 0..7):
//   fwd A  (stages 0-2) : x = t + 128 r
//   fwd B  (stages 3-5) : t = 16 b + u,   x = 128 b + u + 16 r
//   fwd C  (stages 6-8) : t = 2 c + v,    x = 16 c + v + 2 r
//   fwd stage 9 via shfl.xor 1 -> thread t owns spectrum bins 8t .. 8t+7
//   inv    (stages 9-7) : bins 8t + r
//   inv B' (stages 6-4) : t = 8 b + u,    x = 64 b + u + 8 r
//   inv stage 3 via shfl.xor 8
//   inv A  (stages 2-0) : x = t + 128 r
// In every group the radix-4 quadruples are the registers (r, r+2, r+4,
// r+6), r in {0, 1}, and the radix-2 pairs (r, r+1), r even.
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
// single kM-entry buffer (16 KB) instead of all P at once (smaller shared
// footprint). Set LVB_SPLIT_XCHG=0 for the P-buffer form.
#ifndef LVB_SPLIT_XCHG
#define LVB_SPLIT_XCHG 1
#endif
constexpr bool kSplitXchg = LVB_SPLIT_XCHG;
constexpr int kXchgBufs = kSplitXchg ? 1 : 2;
#ifndef LVB_TW_EARLY
#define LVB_TW_EARLY 1  // twiddles requested before the exchange that precedes their group
#endif

// Moves X from layout wr(r) to layout rd(r) (element indices x).
// kWarp: both layouts keep warp w inside the 256-point block w (x >> 8 = w;
// swz() preserves it), so only this warp reads or writes that part of the
// buffer and __syncwarp orders the exchange. Otherwise the exchange crosses
// warps: the caller guarantees no other warp still reads the addresses
// written (this warp's own earlier reads are ordered here).
template <int P, bool kWarp = false, typename WR, typename RD>
__device__ __forceinline__ void xchg(double2 (&X)[P][8], double2* buf, WR wr, RD rd) {
#ifdef LVB_ABL_XCHG  // timing ablation only: results are wrong
  __syncthreads();
  return;
#endif
  auto sync = [] {
    if constexpr (kWarp)
      __syncwarp();
    else
      __syncthreads();
  };
  __syncwarp();
  if constexpr (!kSplitXchg || P == 1) {
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 8; ++r) buf[p * kM + swz(wr(r))] = X[p][r];
    sync();
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 8; ++r) X[p][r] = buf[p * kM + swz(rd(r))];
  } else {
#pragma unroll
    for (int p = 0; p < P; ++p) {
      if (p) sync();
#pragma unroll
      for (int r = 0; r < 8; ++r) buf[swz(wr(r))] = X[p][r];
      sync();
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

__device__ __forceinline__ double2 add2(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
__device__ __forceinline__ double2 sub2(double2 a, double2 b) {
  return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
}

// radix-2 DIF (u + v, (u - v) w) and DIT (p + q conj(w), p - q conj(w))
__device__ __forceinline__ void dif(double2& u, double2& v, double2 w) {
  const double2 s = add2(u, v), d = sub2(u, v);
  u = s;
  v = cmul(d, w);
}
__device__ __forceinline__ void dif1(double2& u, double2& v) {  // w = W^0
  const double2 s = add2(u, v), d = sub2(u, v);
  u = s;
  v = d;
}
__device__ __forceinline__ void dit(double2& p, double2& q, double2 w) {
  const double2 qw = cmul_conj(q, w);
  const double2 a = add2(p, qw), b = sub2(p, qw);
  p = a;
  q = b;
}
__device__ __forceinline__ void dit1(double2& p, double2& q) {  // w = W^0
  const double2 a = add2(p, q), b = sub2(p, q);
  p = a;
  q = b;
}

// radix-4 DIF on (x0, x1, x2, x3) = positions j + {0, H, 2H, 3H} of stages
// s, s+1 (oracle r4_dif), w1 = W^k, w2 = W^2k, w3 = W^3k with k = j << s.
__device__ __forceinline__ void dif4(double2& x0, double2& x1, double2& x2, double2& x3,
                                     double2 w1, double2 w2, double2 w3) {
  const double2 A = add2(x0, x2), B = add2(x1, x3), C = sub2(x0, x2), d = sub2(x1, x3);
  const double2 D = make_double2(d.y, -d.x);  // (x1 - x3) * -i
  x0 = add2(A, B);
  x1 = cmul(sub2(A, B), w2);
  x2 = cmul(add2(C, D), w1);
  x3 = cmul(sub2(C, D), w3);
}
// radix-4 DIT on stages s+1 then s (oracle r4_dit).
__device__ __forceinline__ void dit4(double2& x0, double2& x1, double2& x2, double2& x3,
                                     double2 w1, double2 w2, double2 w3) {
  const double2 t1 = cmul_conj(x1, w2), t2 = cmul_conj(x2, w1), t3 = cmul_conj(x3, w3);
  const double2 A = add2(x0, t1), B = sub2(x0, t1), C = add2(t2, t3), d = sub2(t2, t3);
  const double2 D = make_double2(-d.y, d.x);  // (t2 - t3) * i
  x0 = add2(A, C);
  x2 = sub2(A, C);
  x1 = add2(B, D);
  x3 = sub2(B, D);
}
__device__ __forceinline__ void dit4_1(double2& x0, double2& x1, double2& x2, double2& x3) {
  const double2 A = add2(x0, x1), B = sub2(x0, x1), C = add2(x2, x3), d = sub2(x2, x3);
  const double2 D = make_double2(-d.y, d.x);
  x0 = add2(A, C);
  x2 = sub2(A, C);
  x1 = add2(B, D);
  x3 = sub2(B, D);
}

// Twiddle tables (one buffer, built by context.cu build_tables):
//   [0, kM): per-stage radix-2 tables T_s[y] = W[y << s] (W[k] =
//            exp(-2 pi i k / kM)) concatenated, T_s at kM - (kM >> s);
//   then per radix-4 pair s in {0, 3, 4, 6, 7}: three planes of H = kM >> (s+2)
//            entries, plane m (1..3) holding W[m (j << s)].
// Same values as the oracle's W table, laid out so every warp-wide load is
// contiguous or a broadcast.
__device__ __forceinline__ double2 tws(const double2* __restrict__ tw, int s, uint32_t y) {
#ifdef LVB_ABL_TW  // timing ablation only
  return make_double2(0.70710678118654757 + s * 1e-3, 0.70710678118654757 - y * 1e-9);
#endif
  return __ldg(tw + (kM - (kM >> s)) + y);
}
__device__ __forceinline__ double2 tw4(const double2* __restrict__ tw, int s, int m, uint32_t j) {
  return __ldg(tw + r4_base(s) + (m - 1) * (kM >> (s + 2)) + j);
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
// bins 8t + r. buf: the exchange buffer(s).
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};
// hook() runs once group C's data has arrived (the caller issues loads it
// needs right after the transform there, e.g. the first BSK row).
template <int P, typename Hook = NoHook>
__device__ __forceinline__ void fft_forward(double2 (&X)[P][8], double2* buf,
                                            const double2* __restrict__ tw, uint32_t t,
                                            Hook hook = Hook()) {
  // group A: radix-4 (0,1) with k = t + 128 r, radix-2 stage 2
  {
    double2 w[2][3];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int m = 0; m < 3; ++m) w[r][m] = tw4(tw, 0, m + 1, t + 128 * r);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 2; ++r)
        dif4(X[p][r], X[p][r + 2], X[p][r + 4], X[p][r + 6], w[r][0], w[r][1], w[r][2]);
    const double2 w2 = tws(tw, 2, t);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 8; r += 2) dif(X[p][r], X[p][r + 1], w2);
  }
  // A -> B: radix-4 (3,4) with j = u + 16 r, radix-2 stage 5
  {
    const uint32_t b = t >> 4, u = t & 15;
#if LVB_TW_EARLY
    double2 w[2][3];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int m = 0; m < 3; ++m) w[r][m] = tw4(tw, 3, m + 1, u + 16 * r);
    xchg<P>(X, buf, [&](int r) { return t + 128 * r; },
            [&](int r) { return 128 * b + u + 16 * r; });
#else
    xchg<P>(X, buf, [&](int r) { return t + 128 * r; },
            [&](int r) { return 128 * b + u + 16 * r; });
    double2 w[2][3];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int m = 0; m < 3; ++m) w[r][m] = tw4(tw, 3, m + 1, u + 16 * r);
#endif
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 2; ++r)
        dif4(X[p][r], X[p][r + 2], X[p][r + 4], X[p][r + 6], w[r][0], w[r][1], w[r][2]);
    const double2 w5 = tws(tw, 5, u);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 8; r += 2) dif(X[p][r], X[p][r + 1], w5);
#if LVB_TW_EARLY
    const uint32_t v0 = t & 1;
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int m = 0; m < 3; ++m) w[r][m] = tw4(tw, 6, m + 1, v0 + 2 * r);
#endif
    // B and C both keep warp w in block w (x >> 8 = t >> 5): warp-local
    const uint32_t c = t >> 1, v = t & 1;
    xchg<P, true>(X, buf, [&](int r) { return 128 * b + u + 16 * r; },
                  [&](int r) { return 16 * c + v + 2 * r; });
    hook();
#if LVB_TW_EARLY
    // group C continues in this scope (w already holds its twiddles)
#else
  }
  // C: radix-4 (6,7) with j = v + 2 r, radix-2 stage 8, stage 9 by shuffle
  {
    const uint32_t v = t & 1;
    double2 w[2][3];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int m = 0; m < 3; ++m) w[r][m] = tw4(tw, 6, m + 1, v + 2 * r);
#endif
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 2; ++r)
        dif4(X[p][r], X[p][r + 2], X[p][r + 4], X[p][r + 6], w[r][0], w[r][1], w[r][2]);
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

// ------------------------------------------------------------- inverse
// X[p][r] on entry: spectrum bins 8t + r. On exit: layout A (x = t + 128 r),
// the layout fft_forward's input uses, so each thread owns the same
// accumulator coefficients in both halves of a CMUX. The first exchange is
// warp-local, so the caller only has to order this warp's earlier buffer
// reads (__syncwarp).
template <int P>
__device__ __forceinline__ void fft_inverse_a(double2 (&X)[P][8], double2* buf,
                                              const double2* __restrict__ tw, uint32_t t) {
  // stage 9 (W^0), radix-4 (8,7): j = r, k = 128 r (r = 0: W^0)
  {
    const double2 w1 = tw4(tw, 7, 1, 1), w2 = tw4(tw, 7, 2, 1), w3 = tw4(tw, 7, 3, 1);
#pragma unroll
    for (int p = 0; p < P; ++p) {
#pragma unroll
      for (int r = 0; r < 8; r += 2) dit1(X[p][r], X[p][r + 1]);
      dit4_1(X[p][0], X[p][2], X[p][4], X[p][6]);
      dit4(X[p][1], X[p][3], X[p][5], X[p][7], w1, w2, w3);
    }
  }
  const uint32_t b = t >> 3, u = t & 7, odd = b & 1;
#if LVB_TW_EARLY
  const double2 w6 = tws(tw, 6, u);
  double2 w[2][3];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int m = 0; m < 3; ++m) w[r][m] = tw4(tw, 4, m + 1, u + 8 * r);
#endif
  // bins 8t + r and B' both keep warp w in block w: warp-local
  xchg<P, true>(X, buf, [&](int r) { return 8 * t + r; },
                [&](int r) { return 64 * b + u + 8 * r; });
  {
    // stage 6, radix-4 (5,4) with j = u + 8 r
#if !LVB_TW_EARLY
    const double2 w6 = tws(tw, 6, u);
#endif
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 8; r += 2) dit(X[p][r], X[p][r + 1], w6);
#if !LVB_TW_EARLY
    double2 w[2][3];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int m = 0; m < 3; ++m) w[r][m] = tw4(tw, 4, m + 1, u + 8 * r);
#endif
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 2; ++r)
        dit4(X[p][r], X[p][r + 2], X[p][r + 4], X[p][r + 6], w[r][0], w[r][1], w[r][2]);
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
#if LVB_TW_EARLY
  const double2 w2 = tws(tw, 2, t);
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int m = 0; m < 3; ++m) w[r][m] = tw4(tw, 0, m + 1, t + 128 * r);
#endif
  // B' -> A crosses warps; B' writes stay in this warp's block, which other
  // warps stopped reading at the (warp-local) exchange above
  xchg<P>(
      X, buf,
      [&](int r) { return 64 * (b & ~1u) + u + 8 * ((r & 3) + 4 * odd) + 64 * (r >> 2); },
      [&](int r) { return t + 128 * r; });
  {
    // stage 2, radix-4 (1,0) with j = t + 128 r
#if !LVB_TW_EARLY
    const double2 w2 = tws(tw, 2, t);
#endif
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 8; r += 2) dit(X[p][r], X[p][r + 1], w2);
#if !LVB_TW_EARLY
    double2 w[2][3];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int m = 0; m < 3; ++m) w[r][m] = tw4(tw, 0, m + 1, t + 128 * r);
#endif
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 2; ++r)
        dit4(X[p][r], X[p][r + 2], X[p][r + 4], X[p][r + 6], w[r][0], w[r][1], w[r][2]);
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
  const double r = floor(__fma_rn(y, 0x1p-64, 0.5));  // the product is exact
  const double d = __fma_rn(-r, 18446744073709551616.0, y);
  return (uint64_t)__double2ll_rn(d);
}

}  // namespace lvb
