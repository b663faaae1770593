// Shared device/host definitions for the B200 TFHE PBS path.
//
// Parameter set: q = 2^64, plaintext space Z_32 with the
// padding bit (proj/include/leuven/lut.hpp:9-13, kPlaintextModulus = 32),
// Delta = 2^59; GLWE k = 1, N = 2048; BSK gadget base 2^23, 1 level; KSK
// gadget base 2^3, 5 levels; small LWE dimension n (runtime, default 880).
// Everything is q = 2^64 integer arithmetic except the blind-rotation
// external product, which uses an f64 negacyclic FFT whose operation order
// is fixed (see fft.cuh) so results are bit-identical to the CPU oracle.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define LV_HD __host__ __device__ __forceinline__
#else
#define LV_HD inline
#endif

namespace lvb {

constexpr uint32_t kN = 2048;          // GLWE polynomial size
constexpr uint32_t kM = kN / 2;        // complex FFT size (negacyclic fold)
constexpr uint32_t kLogM = 10;
// FFT twiddle buffer (fft.cuh twf / twi): forward entries of level s at
// fwd_base(s) (the sibling levels 4, 5, 7, 9 keep only their even blocks),
// then kM/2 inverse entries from kM.
LV_HD constexpr bool fwd_sibling_level(int s) { return s == 4 || s == 5 || s == 7 || s == 9; }
LV_HD constexpr uint32_t fwd_base(int s) {
  uint32_t b = 0;
  for (int q = 0; q < s; ++q) b += fwd_sibling_level(q) ? (1u << q) >> 1 : (1u << q);
  return b;
}
constexpr uint32_t kTwEntries = kM + kM / 2;
// Spectrum layout of the blind rotation (fft.cuh L_D): register n of
// thread t = 32 w + L holds DIF output position spec_pos(t, n), bits
// (x0,x1,x6) = n, (x2,x3,x4,x5,x7) = L, (x8,x9) = w. The Fourier BSK is
// stored in this order; spec_slot is the inverse (t = slot >> 3, n = slot & 7).
LV_HD uint32_t spec_pos(uint32_t t, uint32_t n) {
  const uint32_t L = t & 31, w = t >> 5;
  return (n & 1) | ((n >> 1) & 1) << 1 | ((n >> 2) & 1) << 6 | (L & 1) << 2 | ((L >> 1) & 1) << 3 |
         ((L >> 2) & 1) << 4 | ((L >> 3) & 1) << 5 | ((L >> 4) & 1) << 7 | (w & 3) << 8;
}
LV_HD uint32_t spec_slot(uint32_t x) {
  const uint32_t n = (x & 1) | ((x >> 1) & 1) << 1 | ((x >> 6) & 1) << 2;
  const uint32_t L = ((x >> 2) & 1) | ((x >> 3) & 1) << 1 | ((x >> 4) & 1) << 2 | ((x >> 5) & 1) << 3 |
                     ((x >> 7) & 1) << 4;
  return ((((x >> 8) & 3) * 32 + L) << 3) | n;
}
constexpr uint32_t kK = 1;             // GLWE dimension
constexpr uint32_t kBig = kK * kN;     // big-key LWE mask length
constexpr uint32_t kBigStride = kBig + 8;  // pool row stride in u64 (16448 B, 64 B aligned)
constexpr uint32_t kPbsBaseLog = 23;
constexpr uint32_t kPbsLevel = 1;
constexpr uint32_t kRows = (kK + 1) * kPbsLevel;  // GGSW rows
constexpr uint32_t kKsBaseLog = 3;
constexpr uint32_t kKsLevel = 5;
constexpr uint32_t kLog2N2 = 12;       // log2(2N)
constexpr uint64_t kDelta = 1ull << 59;
constexpr uint32_t kMaxLweN = 4096;      // largest small-LWE dimension a context accepts

// Philox domains (shared by specification with the oracle).
enum Domain : uint32_t {
  kDomSkSmall = 1,
  kDomSkGlwe = 2,
  kDomBskMask = 3,
  kDomBskNoise = 4,
  kDomKskMask = 5,
  kDomKskNoise = 6,
  kDomEncMask = 7,
  kDomEncNoise = 8,
};

// Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11): key = seed,
// counter = {idx_lo, idx_hi, domain, 0}; returns words 0,1 as a u64.
LV_HD uint64_t philox_u64(uint64_t seed, uint32_t domain, uint64_t idx) {
  uint32_t c0 = (uint32_t)idx, c1 = (uint32_t)(idx >> 32), c2 = domain, c3 = 0;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    const uint32_t n1 = (uint32_t)p1;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    const uint32_t n3 = (uint32_t)p0;
    c0 = n0;
    c1 = n1;
    c2 = n2;
    c3 = n3;
  }
  return ((uint64_t)c1 << 32) | c0;
}

// TUniform(b): integers in [-2^b, 2^b] with half weight on the endpoints.
LV_HD int64_t tuniform(uint64_t seed, uint32_t domain, uint64_t idx, uint32_t b) {
  const uint64_t x = philox_u64(seed, domain, idx) & ((1ull << (b + 2)) - 1);
  return (int64_t)(x >> 1) + (int64_t)(x & 1) - ((int64_t)1 << b);
}

// Closest-representable signed gadget digit, 1 level (digits in [-B/2, B/2)).
LV_HD int64_t decomp1(uint64_t x, uint32_t base_log) {
  const uint32_t shift = 64 - base_log;
  const uint64_t v = (x + (1ull << (shift - 1))) >> shift;
  const int64_t half = (int64_t)1 << (base_log - 1);
  int64_t d = (int64_t)v;
  if (d >= half) d -= (int64_t)1 << base_log;
  return d;
}

// decomp1 for the blind-rotation gadget (base 2^23, one level) on 32-bit
// integer ops: adding 2^40 touches only the high word (2^40 = 2^8 * 2^32),
// and the arithmetic shift of (hi + 2^8) by 9 is the rounded digit already
// sign-folded into [-2^22, 2^22) — equal to decomp1(x, 23) for every x.
static_assert(kPbsBaseLog == 23 && kPbsLevel == 1, "decomp23 is the 2^23 x 1 gadget");
LV_HD int32_t decomp23(uint64_t x) {
  return (int32_t)((uint32_t)(x >> 32) + 256u) >> 9;
}

// Multi-level variant: digits[0] has weight q/B (most significant).
template <int L>
LV_HD void decomp(uint64_t x, uint32_t base_log, int64_t* digits) {
  const uint32_t shift = 64 - base_log * L;
  uint64_t v = (x + (1ull << (shift - 1))) >> shift;
  const uint64_t mask = (1ull << base_log) - 1;
  const int64_t half = (int64_t)1 << (base_log - 1);
#pragma unroll
  for (int l = L - 1; l >= 0; --l) {
    int64_t d = (int64_t)(v & mask);
    v >>= base_log;
    if (d >= half) {
      d -= (int64_t)1 << base_log;
      v += 1;
    }
    digits[l] = d;
  }
}

LV_HD uint32_t modswitch(uint64_t a) {
  constexpr uint32_t shift = 64 - kLog2N2;
  return (uint32_t)(((a + (1ull << (shift - 1))) >> shift) & ((1u << kLog2N2) - 1));
}

}  // namespace lvb
