// Negacyclic f64 FFT for N = 2048 (1024-point complex DIF forward, DIT
// inverse), 128 threads per transform, 8 complex values per thread, P
// polynomials processed in lockstep by the same threads.
//
// Bit-exactness contract with oracle/tfhe_oracle.c (fft_dif,
// fft_dit_inverse, forward_i64, backward_torus): the network is fixed —
// forward: radix-4 DIF butterflies on the stage pairs (0,1), (3,4), (6,7),
// (8,9) and radix-2 stages 2, 5; inverse (its DIT mirror): radix-4 (9,8),
// (7,6), radix-2 5, radix-4 (4,3), radix-2 2, radix-4 (1,0) — and every
// butterfly performs exactly the oracle's IEEE operations (__dadd_rn /
// __dsub_rn for sums, cmul() = {fma(a.x,b.x,-(a.y*b.y)), fma(a.x,b.y,(a.y*b.x))}
// for twiddles, the same table entries). Only the data movement differs
// (registers, a swizzled shared buffer, tensor memory), which cannot change
// a rounding. Multiplications by W^0 = (1,-0) that are static are skipped:
// they are exact up to the sign of zero, which never reaches a nonzero
// result (the (8,9) pair's twiddles are all W^0).
//
// Data movement per transform: one cross-warp exchange through shared
// memory and two warp-local exchanges through TENSOR MEMORY. A TMEM round
// trip — tcgen05.st with the 32x32b shape (thread = lane, registers =
// columns), tcgen05.ld with the 16x256b shape (thread t0 + 4 t1 <- lane
// t1 + 8h (+16 for the second load), 64-bit column t0 + 4k) — permutes the
// data between the warp's threads: it moves lane bits 3,4 into registers
// and register bits 0,1 into lanes. TMEM traffic runs on its own datapath,
// not the L1/shared-memory pipe that bounds this kernel (tools/
// tmem_xchg_bench.cu: a round trip of 2 x 4 KB per warp costs 271 SM-cycles
// per CTA vs 539 for the shared-memory exchange it replaces, and mixed
// with shared-memory traffic the two overlap completely). Complex points
// are stored planar (re of point r at 64-bit column r, im at 8 + r) so a
// 16x256b fragment keeps each point's two halves in one thread.
//
// Thread layouts (t = 32 w + L, w = warp, L = lane, r / n = register 0..7;
// x = position, bits x9..x0):
//   L_A (fwd pass A / inv pass A'): x = t + 128 r: regs (x7,x8,x9),
//        lanes (x0..x4), warps (x5,x6)
//   L_B : regs (x4,x5,x6), lanes (x7,x0,x1,x2,x3), warps (x8,x9)
//   L_C : regs (x2,x3,x6), lanes (x4,x5,x7,x0,x1)
//   L_D : regs (x0,x1,x6), lanes (x2,x3,x4,x5,x7)  — the spectrum layout
// L_A <-> L_B cross warps (shared memory); L_B -> L_C -> L_D are TMEM
// round trips (32x32b store, 16x256b load) and the inverse walks back with
// the inverse trips (16x256b store, 32x32b load).
#pragma once

#include <cuda_runtime.h>

#include <type_traits>

#include "common.cuh"

namespace lvb {

// Shared buffer index swizzle: both L_A (x0..x2 across an 8-lane phase,
// x7 fixed) and L_B (x7, x0, x1 across a phase, x2 fixed) hit 8 distinct
// 16-byte bank groups.
__device__ __forceinline__ uint32_t swz(uint32_t x) { return x ^ (((x >> 7) & 1u) << 2); }

// Barrier of the threads sharing one transform (the CTA).
struct CtaBar {
  __device__ __forceinline__ void sync() const { __syncthreads(); }
};

// Cross-warp exchanges go through NB shared 16 KB buffers (P polynomials in
// groups of NB). One buffer (default) costs two barriers per exchange but
// leaves 16 KB per CTA to L1: at 3 CTAs/SM the carveout drops from 228 to
// 164 KB and the twiddle tables stay L1-resident (59.4 -> 56.8 ms per 4096
// PBS; at 2 CTAs/SM it measured slower).
#ifndef LVB_XCHG_BUFS
#define LVB_XCHG_BUFS 1
#endif
constexpr int kXchgBufs = LVB_XCHG_BUFS;

// Moves X from layout wr(r) to layout rd(r) (element indices x) across
// warps. The caller guarantees no warp still reads the buffer.
template <int P, int NB, typename Bar, typename WR, typename RD>
__device__ __forceinline__ void xchg_cta(double2 (&X)[P][8], double2* buf, const Bar& bar, WR wr,
                                         RD rd) {
#ifdef LVB_ABL_XCHG  // timing ablation only: results are wrong
  bar.sync();
  return;
#endif
#pragma unroll
  for (int p0 = 0; p0 < P; p0 += NB) {
    if (p0) bar.sync();
#pragma unroll
    for (int p = p0; p < P && p < p0 + NB; ++p)
#pragma unroll
      for (int r = 0; r < 8; ++r) buf[(p - p0) * kM + swz(wr(r))] = X[p][r];
    bar.sync();
#pragma unroll
    for (int p = p0; p < P && p < p0 + NB; ++p)
#pragma unroll
      for (int r = 0; r < 8; ++r) X[p][r] = buf[(p - p0) * kM + swz(rd(r))];
  }
}

// Phase probes (diagnostic builds, -DLVB_PROBE): lane 0 of each warp of
// CTA 0 adds the SM clock at mark k; the host turns sums of timestamps into
// mean phase durations (lv_debug_probe). No-ops in the product.
#ifdef LVB_PROBE
__device__ unsigned long long g_probe[4][32];
__device__ __forceinline__ void probe_mark(int k) {
  if (blockIdx.x == 0 && (threadIdx.x & 31) == 0)
    atomicAdd(&g_probe[threadIdx.x >> 5][k], (unsigned long long)clock64());
}
#else
__device__ __forceinline__ void probe_mark(int) {}
#endif

// ---------------------------------------------------------------- TMEM
// Allocation: warp 0 allocates ncols columns (power of 2, >= 32) and
// writes the base address to *slot; every thread returns it.
__device__ __forceinline__ uint32_t tmem_alloc(uint32_t* slot, uint32_t ncols) {
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(slot)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  return *slot;
}
__device__ __forceinline__ void tmem_free(uint32_t base, uint32_t ncols) {
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(ncols));
}
// This warp's lane quarter of the CTA's allocation.
__device__ __forceinline__ uint32_t tmem_warp_base(uint32_t base) {
  return base + ((32u * ((threadIdx.x >> 5) & 3u)) << 16);
}
constexpr uint32_t kTmemColsPerPoly = 32;  // 8 complex points x 4 columns

__device__ __forceinline__ uint32_t d_lo(double v) { return (uint32_t)__double_as_longlong(v); }
__device__ __forceinline__ uint32_t d_hi(double v) {
  return (uint32_t)((unsigned long long)__double_as_longlong(v) >> 32);
}
__device__ __forceinline__ double d_mk(uint32_t l, uint32_t h) {
  return __longlong_as_double((long long)(((unsigned long long)h << 32) | l));
}

// tcgen05.wait::ld that also names the loaded registers as in/out
// operands, so the compiler cannot schedule a use of them above the wait.
#define LVB_TM_WAIT_LD16(a, b)                                                                    \
  asm volatile("tcgen05.wait::ld.sync.aligned;"                                                   \
               : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]),          \
                 "+r"(a[6]), "+r"(a[7]), "+r"(a[8]), "+r"(a[9]), "+r"(a[10]), "+r"(a[11]),        \
                 "+r"(a[12]), "+r"(a[13]), "+r"(a[14]), "+r"(a[15]), "+r"(b[0]), "+r"(b[1]),      \
                 "+r"(b[2]), "+r"(b[3]), "+r"(b[4]), "+r"(b[5]), "+r"(b[6]), "+r"(b[7]),          \
                 "+r"(b[8]), "+r"(b[9]), "+r"(b[10]), "+r"(b[11]), "+r"(b[12]), "+r"(b[13]),      \
                 "+r"(b[14]), "+r"(b[15])                                                         \
               :                                                                                  \
               : "memory")

// LVB_TM_FINE: one tcgen05 instruction per double (32x32b.x2) / per two
// doubles (16x256b.x1) instead of one per 8 points, so the operands need
// only aligned register pairs, not 16- or 32-register blocks (no moves).
#ifndef LVB_TM_FINE
#define LVB_TM_FINE 0
#endif
__device__ __forceinline__ void tm_st_32x32b(uint32_t a, const double2 (&X)[8]) {
#if LVB_TM_FINE
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(a + 2 * k),
                 "r"(d_lo(X[k].x)), "r"(d_hi(X[k].x))
                 : "memory");
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(a + 16 + 2 * k),
                 "r"(d_lo(X[k].y)), "r"(d_hi(X[k].y))
                 : "memory");
  }
  return;
#endif
  uint32_t r[32];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    r[2 * k] = d_lo(X[k].x);
    r[2 * k + 1] = d_hi(X[k].x);
    r[16 + 2 * k] = d_lo(X[k].y);
    r[17 + 2 * k] = d_hi(X[k].y);
  }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(a),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
      "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]),
      "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]),
      "r"(r[30]), "r"(r[31])
      : "memory");
}
// Issues the load; the caller waits (LVB_TM_WAIT_LD16(r, r + 16)) and unpacks.
__device__ __forceinline__ void tm_ld_32x32b(uint32_t a, uint32_t (&r)[32]) {
#if LVB_TM_FINE
#pragma unroll
  for (int k = 0; k < 16; ++k)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];"
                 : "=r"(r[2 * k]), "=r"(r[2 * k + 1])
                 : "r"(a + 2 * k)
                 : "memory");
  return;
#endif
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(a)
      : "memory");
}
__device__ __forceinline__ void unpack32(const uint32_t (&r)[32], double2 (&X)[8]) {
#pragma unroll
  for (int k = 0; k < 8; ++k)
    X[k] = make_double2(d_mk(r[2 * k], r[2 * k + 1]), d_mk(r[16 + 2 * k], r[17 + 2 * k]));
}
// 16x256b fragment of 16 lanes (the lane base is in the address) x 32
// columns: reg 4k + 2h (+1) = lane t1 + 8h, 64-bit column 4k + t0.
#if LVB_TM_FINE
#define LVB_TM_16x256b_LD(addr, a)                                                               \
  do {                                                                                           \
    _Pragma("unroll") for (int k_ = 0; k_ < 4; ++k_) asm volatile(                              \
        "tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"                            \
        : "=r"(a[4 * k_]), "=r"(a[4 * k_ + 1]), "=r"(a[4 * k_ + 2]), "=r"(a[4 * k_ + 3])         \
        : "r"((addr) + 8 * k_)                                                                   \
        : "memory");                                                                             \
  } while (0)
#define LVB_TM_16x256b_ST(addr, a)                                                               \
  do {                                                                                           \
    _Pragma("unroll") for (int k_ = 0; k_ < 4; ++k_) asm volatile(                              \
        "tcgen05.st.sync.aligned.16x256b.x1.b32 [%0], {%1,%2,%3,%4};" ::"r"((addr) + 8 * k_),    \
        "r"(a[4 * k_]), "r"(a[4 * k_ + 1]), "r"(a[4 * k_ + 2]), "r"(a[4 * k_ + 3])              \
        : "memory");                                                                             \
  } while (0)
#else
#define LVB_TM_16x256b_LD(addr, a)                                                                \
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12," \
               "%13,%14,%15}, [%16];"                                                              \
               : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]),           \
                 "=r"(a[6]), "=r"(a[7]), "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11]),         \
                 "=r"(a[12]), "=r"(a[13]), "=r"(a[14]), "=r"(a[15])                                \
               : "r"(addr)                                                                         \
               : "memory")
#define LVB_TM_16x256b_ST(addr, a)                                                                 \
  asm volatile("tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11," \
               "%12,%13,%14,%15,%16};" ::"r"(addr),                                                \
               "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]),        \
               "r"(a[7]), "r"(a[8]), "r"(a[9]), "r"(a[10]), "r"(a[11]), "r"(a[12]), "r"(a[13]),    \
               "r"(a[14]), "r"(a[15])                                                              \
               : "memory")
#endif
// Point index n of the 16x256b view: n = h + 2 g + 4 k' <-> (lane t1 + 8h +
// 16g, stored point t0 + 4k'); re at columns 4k', im at 4(k' + 2).
template <int G>
__device__ __forceinline__ void unpack16(const uint32_t (&a)[16], double2 (&X)[8]) {
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int k = 0; k < 2; ++k)
      X[h + 2 * G + 4 * k] = make_double2(d_mk(a[4 * k + 2 * h], a[4 * k + 2 * h + 1]),
                                          d_mk(a[4 * (k + 2) + 2 * h], a[4 * (k + 2) + 2 * h + 1]));
}
template <int G>
__device__ __forceinline__ void pack16(const double2 (&X)[8], uint32_t (&a)[16]) {
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double2 v = X[h + 2 * G + 4 * k];
      a[4 * k + 2 * h] = d_lo(v.x);
      a[4 * k + 2 * h + 1] = d_hi(v.x);
      a[4 * (k + 2) + 2 * h] = d_lo(v.y);
      a[4 * (k + 2) + 2 * h + 1] = d_hi(v.y);
    }
}

// Forward trip: lanes (l0..l4), regs (r0,r1,r2) -> lanes (r0,r1,l0,l1,l2),
// regs (l3,l4,r2). tm = this warp's lane-quarter base; polynomial p uses
// columns [32p, 32p + 32).
template <int P>
__device__ __forceinline__ void tm_trip_fwd(double2 (&X)[P][8], uint32_t tm) {
#ifdef LVB_ABL_TMEM  // timing ablation only
  return;
#endif
#pragma unroll
  for (int p = 0; p < P; ++p) tm_st_32x32b(tm + p * kTmemColsPerPoly, X[p]);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  uint32_t a[P][16], b[P][16];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    LVB_TM_16x256b_LD(tm + p * kTmemColsPerPoly, a[p]);
    LVB_TM_16x256b_LD(tm + p * kTmemColsPerPoly + (16u << 16), b[p]);
  }
#pragma unroll
  for (int p = 0; p < P; ++p) {
    LVB_TM_WAIT_LD16(a[p], b[p]);  // the first wait covers every load; the rest fence registers
    unpack16<0>(a[p], X[p]);
    unpack16<1>(b[p], X[p]);
  }
}
// Inverse trip (undoes tm_trip_fwd): lanes (l0..l4), regs (r0,r1,r2) ->
// lanes (l2,l3,l4,r0,r1), regs (l0,l1,r2).
template <int P>
__device__ __forceinline__ void tm_trip_inv(double2 (&X)[P][8], uint32_t tm) {
#ifdef LVB_ABL_TMEM
  return;
#endif
#pragma unroll
  for (int p = 0; p < P; ++p) {
    uint32_t a[16], b[16];
    pack16<0>(X[p], a);
    pack16<1>(X[p], b);
    LVB_TM_16x256b_ST(tm + p * kTmemColsPerPoly, a);
    LVB_TM_16x256b_ST(tm + p * kTmemColsPerPoly + (16u << 16), b);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  uint32_t r[P][32];
#pragma unroll
  for (int p = 0; p < P; ++p) tm_ld_32x32b(tm + p * kTmemColsPerPoly, r[p]);
#pragma unroll
  for (int p = 0; p < P; ++p) {
    LVB_TM_WAIT_LD16(r[p], (r[p] + 16));
    unpack32(r[p], X[p]);
  }
}

// ---------------------------------------------------------------- math
// int32 -> f64, exact: LVB_I2D_MAGIC builds 2^52 + 2^31 + d in the bits and
// subtracts it back (one DADD on the FP64 pipe instead of an XU conversion).
#ifndef LVB_I2D_MAGIC
#define LVB_I2D_MAGIC 0
#endif
__device__ __forceinline__ double i2d(int32_t d) {
#if LVB_I2D_MAGIC
  return __dadd_rn(__hiloint2double(0x43300000, (int)((uint32_t)d ^ 0x80000000u)), -4503601774854144.0);
#else
  return (double)d;
#endif
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

// Cooley-Tukey butterfly u +- w v in Linzer-Feig form (oracle ct_lf): the
// twiddle w = c (1 + i t) is held as (c, t) = (w.x, w.y), six FMAs.
__device__ __forceinline__ void ct(double2& u, double2& v, double2 w) {
  const double a = __fma_rn(-w.y, v.y, v.x);
  const double b = __fma_rn(w.y, v.x, v.y);
  const double2 U = u;
  u = make_double2(__fma_rn(w.x, a, U.x), __fma_rn(w.x, b, U.y));
  v = make_double2(__fma_rn(-w.x, a, U.x), __fma_rn(-w.x, b, U.y));
}
// u +- (-i w) v (oracle ct_lf_mi): an odd forward block from its even
// sibling's twiddle; (-i w) v = c (b - i a).
__device__ __forceinline__ void ct_mi(double2& u, double2& v, double2 w) {
  const double a = __fma_rn(-w.y, v.y, v.x);
  const double b = __fma_rn(w.y, v.x, v.y);
  const double2 U = u;
  u = make_double2(__fma_rn(w.x, b, U.x), __fma_rn(-w.x, a, U.y));
  v = make_double2(__fma_rn(-w.x, b, U.x), __fma_rn(w.x, a, U.y));
}
// u +- (i w) v (oracle ct_lf_i): an inverse pair with k >= kM/4 from the
// twiddle of k - kM/4; (i w) v = c (-b + i a).
__device__ __forceinline__ void ct_pi(double2& u, double2& v, double2 w) {
  const double a = __fma_rn(-w.y, v.y, v.x);
  const double b = __fma_rn(w.y, v.x, v.y);
  const double2 U = u;
  u = make_double2(__fma_rn(-w.x, b, U.x), __fma_rn(w.x, a, U.y));
  v = make_double2(__fma_rn(w.x, b, U.x), __fma_rn(-w.x, a, U.y));
}
// The inverse's first two stages (9, 8): w = 1 on (x0, x1), (x2, x3), then
// w = 1 on (x0, x2) and w = i on (x1, x3) — exact additions (oracle ct_one,
// ct_i).
__device__ __forceinline__ void dit4_1(double2& x0, double2& x1, double2& x2, double2& x3) {
  const double2 A = add2(x0, x1), B = sub2(x0, x1), C = add2(x2, x3), d = sub2(x2, x3);
  const double2 D = make_double2(-d.y, d.x);
  x0 = add2(A, C);
  x2 = sub2(A, C);
  x1 = add2(B, D);
  x3 = sub2(B, D);
}

// Twiddle buffer (context.cu build_tables), Linzer-Feig pairs (c, t):
//   [0, kFwdEntries): forward, the negacyclic root zeta^e of level s block b,
//            e = (kM >> (s+1)) (1 - 4 brv_s(b)) mod 2N, at fwd_base(s) + b —
//            at the sibling levels 4, 5, 7, 9 only the even blocks, at
//            fwd_base(s) + b/2 (odd blocks use -i x their even sibling);
//   [kM, kM + kM/2): inverse, conj(W^k) at kM + k.
// Compact so the tables (~19 KB touched) stay resident in L1 next to the
// shared-memory carveout. Levels 0-2 (pass A, blocks fixed by registers)
// also sit in the constant bank, so those butterflies take their twiddles
// as constant operands.
__constant__ double2 c_fwd_a[7];  // defined here: fft.cuh has one includer (kernels.cu)
__device__ __forceinline__ double2 twf(const double2* __restrict__ tw, int s, uint32_t b) {
#ifdef LVB_ABL_TW  // timing ablation only
  return make_double2(0.70710678118654757 + s * 1e-3, 0.9 - b * 1e-9);
#endif
  return __ldg(tw + fwd_base(s) + (fwd_sibling_level(s) ? b >> 1 : b));
}
__device__ __forceinline__ double2 twi(const double2* __restrict__ tw, uint32_t k) {
#ifdef LVB_ABL_TW
  return make_double2(0.70710678118654757, 0.9 - k * 1e-9);
#endif
  return __ldg(tw + kM + k);
}

// Coarse twist factors zeta^(128 k), k < 8 (constant bank).
__constant__ double2 c_twist_coarse[8];

// zeta^x = fine[x & 127] * coarse[x >> 7] (oracle build_tables defines the
// twist this way); coarse[0] = 1 is an exact identity and is skipped.
__device__ __forceinline__ double2 twist_at(const double2* __restrict__ fine, uint32_t x) {
  const double2 f = __ldg(fine + (x & 127));
  return (x >> 7) == 0 ? f : cmul(f, c_twist_coarse[x >> 7]);
}

// ------------------------------------------------------ twiddle sources
// Each thread needs the same 22 twiddles every CMUX (they depend only on
// its position in the layouts): 4 per forward pass B / C / D, 2 for inverse
// pass C', 4 for B' and A'. TwGlobal loads them from the L1-resident table
// at every use; TwTmem parks the thread's set in tensor memory once (88
// columns of its warp's lane quarter, fill()) and fetches a pass's set with
// one tcgen05.ld — for the latency kernels, where every L1 round trip sits
// on the critical path. Both give the same values, so results are
// bit-identical.
struct TwGlobal {
  const double2* __restrict__ tw;
  uint32_t t;
  __device__ __forceinline__ void fwdB(double2 (&w)[4]) const {
    const uint32_t L = t & 31, b3 = 2 * (t >> 5) + (L & 1);
    w[0] = twf(tw, 3, b3);
    w[1] = twf(tw, 4, 2 * b3);  // odd level-4 blocks: -i w4
#pragma unroll
    for (int q = 0; q < 2; ++q) w[2 + q] = twf(tw, 5, 4 * b3 + 2 * q);  // even level-5 blocks
  }
  __device__ __forceinline__ void fwdC(double2 (&w)[4]) const {
    const uint32_t L = t & 31;
    const uint32_t b6 = 16 * (t >> 5) + 8 * ((L >> 2) & 1) + 2 * ((L >> 1) & 1) + (L & 1);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      w[q] = twf(tw, 6, b6 + 4 * q);
      w[2 + q] = twf(tw, 7, 2 * (b6 + 4 * q));
    }
  }
  __device__ __forceinline__ void fwdD(double2 (&w)[4]) const {
    const uint32_t L = t & 31, b8 = 64 * (t >> 5) + 32 * (L >> 4) + (L & 15);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      w[q] = twf(tw, 8, b8 + 16 * q);
      w[2 + q] = twf(tw, 9, 2 * (b8 + 16 * q));
    }
  }
  __device__ __forceinline__ void invC(double2 (&v)[2]) const {
    const uint32_t j = (t & 31) >> 3;
    v[0] = twi(tw, j << 7);
    v[1] = twi(tw, j << 6);  // stage 6, x2 = 1: i v6
  }
  __device__ __forceinline__ void invB(double2 (&v)[4]) const {
    const uint32_t u = (t & 31) >> 1;
    v[0] = twi(tw, u << 5);
    v[1] = twi(tw, u << 4);  // stage 4, x4 = 1: i v4
#pragma unroll
    for (int q = 0; q < 2; ++q) v[2 + q] = twi(tw, (u << 3) + 128 * q);  // stage 3 per x4
  }
  __device__ __forceinline__ void invA(double2 (&v)[4]) const {
    v[0] = twi(tw, t << 2);
    v[1] = twi(tw, t << 1);  // stage 1, x7 = 1: i v1
#pragma unroll
    for (int q = 0; q < 2; ++q) v[2 + q] = twi(tw, t + 128 * q);  // stage 0 per x7
  }
  template <int K>
  __device__ __forceinline__ void ready(double2 (&)[K]) const {}
};

struct TwTmem {
  uint32_t cols;  // this warp's lane-quarter address of the 88 twiddle columns
  // column slots: fwd B 0, C 16, D 32, inv C' 48 (8), B' 56, A' 72
  template <int K>
  __device__ __forceinline__ void ld(uint32_t c, double2 (&w)[K]) const {
    uint32_t r[4 * K];
    if constexpr (K == 4)
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
          "%14,%15}, [%16];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
            "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(cols + c)
          : "memory");
    else
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                     "=r"(r[6]), "=r"(r[7])
                   : "r"(cols + c)
                   : "memory");
#pragma unroll
    for (int q = 0; q < K; ++q)
      w[q] = make_double2(d_mk(r[4 * q], r[4 * q + 1]), d_mk(r[4 * q + 2], r[4 * q + 3]));
  }
  __device__ __forceinline__ void fwdB(double2 (&w)[4]) const { ld(0, w); }
  __device__ __forceinline__ void fwdC(double2 (&w)[4]) const { ld(16, w); }
  __device__ __forceinline__ void fwdD(double2 (&w)[4]) const { ld(32, w); }
  __device__ __forceinline__ void invC(double2 (&v)[2]) const { ld(48, v); }
  __device__ __forceinline__ void invB(double2 (&v)[4]) const { ld(56, v); }
  __device__ __forceinline__ void invA(double2 (&v)[4]) const { ld(72, v); }
  // completes this thread's TMEM loads and fences the twiddle registers
  template <int K>
  __device__ __forceinline__ void ready(double2 (&w)[K]) const {
#pragma unroll
    for (int q = 0; q < K; ++q)
      asm volatile("tcgen05.wait::ld.sync.aligned;" : "+d"(w[q].x), "+d"(w[q].y) : : "memory");
  }
  // once per CTA: the thread's 22 twiddles from the global table into TMEM
  __device__ __forceinline__ void fill(const TwGlobal& g) const {
    double2 a[4];
    g.fwdB(a);
    st(0, a);
    g.fwdC(a);
    st(16, a);
    g.fwdD(a);
    st(32, a);
    double2 c[2];
    g.invC(c);
    st(48, c);
    g.invB(a);
    st(56, a);
    g.invA(a);
    st(72, a);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  template <int K>
  __device__ __forceinline__ void st(uint32_t c, const double2 (&w)[K]) const {
#pragma unroll
    for (int q = 0; q < K; ++q)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(cols + c + 4 * q),
                   "r"(d_lo(w[q].x)), "r"(d_hi(w[q].x)), "r"(d_lo(w[q].y)), "r"(d_hi(w[q].y))
                   : "memory");
  }
};
constexpr uint32_t kTwTmemCols = 88;

__device__ __forceinline__ TwGlobal tw_source(const double2* __restrict__ tw, uint32_t t) {
  return TwGlobal{tw, t};
}
__device__ __forceinline__ TwTmem tw_source(TwTmem s, uint32_t) { return s; }

// ---------------------------------------------------------------- forward
// Negacyclic forward transform (oracle fft_fwd): level s pairs bit x(9-s)
// of the position, block b = x >> (10 - s). X[p][r] on entry: the folded
// integer polynomial (d_x, d_{x+kM}) at x = t + 128 r (L_A), no twist. On
// exit: the spectrum in L_D (register n of thread t = position
// spec_pos(t, n)).
// buf: NB exchange buffers (no warp may still be reading them); tm: this
// warp's TMEM lane-quarter base.
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};
// hook() issues loads the caller needs right after the transform (the first
// BSK bin groups): LVB_HOOK_PASS 0 after the first TMEM trip, 1 (default)
// just before the second, 2 after it (55.86 / 55.55 / 55.56 ms per 4096).
#ifndef LVB_HOOK_PASS
#define LVB_HOOK_PASS 1
#endif
// kSyncFirst: buf aliases memory other warps may still be reading when the
// transform starts (the blind rotation's accumulator): one barrier before
// the first exchange write.
template <int P, int NB = kXchgBufs, typename Hook = NoHook, typename Bar = CtaBar,
          bool kSyncFirst = false, typename TW = const double2*>
__device__ __forceinline__ void fft_forward(double2 (&X)[P][8], double2* buf, TW twsrc, uint32_t t,
                                            uint32_t tm, Hook hook = Hook(), Bar bar = Bar()) {
  const uint32_t L = t & 31, w = t >> 5;
  // twiddles: the product's throughput kernel loads them from the L1-resident
  // table inline (TW = const double2*; the pre-policy code, register
  // allocation unchanged), the latency kernels fetch a pass's set from TMEM
  constexpr bool kTm = std::is_same<TW, TwTmem>::value;
  const auto tws = tw_source(twsrc, t);
  // pass A (L_A: regs (x7, x8, x9)): levels 0, 1, 2; every block index is
  // a register index, so the twiddles are constant-bank operands
#pragma unroll
  for (int p = 0; p < P; ++p)
#pragma unroll
    for (int r = 0; r < 4; ++r) ct(X[p][r], X[p][r + 4], c_fwd_a[0]);
#pragma unroll
  for (int p = 0; p < P; ++p)
#pragma unroll
    for (int r = 0; r < 8; r += (r & 1) ? 3 : 1) ct(X[p][r], X[p][r + 2], c_fwd_a[1 + (r >> 2)]);
#pragma unroll
  for (int p = 0; p < P; ++p)
#pragma unroll
    for (int r = 0; r < 8; r += 2) ct(X[p][r], X[p][r + 1], c_fwd_a[3 + (r >> 1)]);
  probe_mark(2);
  // L_A -> L_B (cross-warp); pass B (L_B: regs (x4, x5, x6), lanes (x7,
  // x0..x3), warps (x8, x9)): level 3 on x6, block b3 = x >> 7 = 2 w + L0;
  // level 4 on x5, block 2 b3 + x6; level 5 on x4, block 4 b3 + (x5, x6)
  const uint32_t u = L >> 1;  // x3..x0
  {
    double2 wB[4];  // w3, w4 (odd level-4 blocks: -i w4), w5 of the even level-5 blocks 4 b3 + 2 x6
    double2 w3, w4, w5[2];
    if constexpr (kTm) {
      tws.fwdB(wB);
    } else {
      const uint32_t b3 = 2 * w + (L & 1);
      w3 = twf(twsrc, 3, b3);
      w4 = twf(twsrc, 4, 2 * b3);
#pragma unroll
      for (int q = 0; q < 2; ++q) w5[q] = twf(twsrc, 5, 4 * b3 + 2 * q);
    }
    if constexpr (kSyncFirst) bar.sync();
    xchg_cta<P, NB>(X, buf, bar, [&](int r) { return t + 128u * r; },
                    [&](int r) { return 16u * r + 128u * (L & 1) + u + 256u * w; });
    if constexpr (kTm) {
      tws.ready(wB);
      w3 = wB[0];
      w4 = wB[1];
      w5[0] = wB[2];
      w5[1] = wB[3];
    }
    probe_mark(3);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 4; ++r) ct(X[p][r], X[p][r + 4], w3);
#pragma unroll
    for (int p = 0; p < P; ++p) {
      ct(X[p][0], X[p][2], w4);
      ct(X[p][1], X[p][3], w4);
      ct_mi(X[p][4], X[p][6], w4);
      ct_mi(X[p][5], X[p][7], w4);
    }
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 8; r += 4) {
        ct(X[p][r], X[p][r + 1], w5[r >> 2]);
        ct_mi(X[p][r + 2], X[p][r + 3], w5[r >> 2]);
      }
  }
  // L_B -> L_C (TMEM); pass C (L_C: regs (x2, x3, x6), lanes (x4, x5, x7,
  // x0, x1)): level 6 on x3, block x >> 4 = 16 w + 8 L2 + 4 x6 + 2 L1 + L0;
  // level 7 on x2, block 2 (x >> 4) + x3
  {
    double2 wC[4];  // w6 per x6; w7 per x6 (odd level-7 blocks, x3 = 1: -i w7)
    double2 w6[2], w7[2];
    if constexpr (kTm) {
      tws.fwdC(wC);
    } else {
      const uint32_t b6 = 16 * w + 8 * ((L >> 2) & 1) + 2 * ((L >> 1) & 1) + (L & 1);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        w6[q] = twf(twsrc, 6, b6 + 4 * q);
        w7[q] = twf(twsrc, 7, 2 * (b6 + 4 * q));
      }
    }
    probe_mark(4);
    tm_trip_fwd<P>(X, tm);
    if constexpr (kTm) {
      tws.ready(wC);
      w6[0] = wC[0];
      w6[1] = wC[1];
      w7[0] = wC[2];
      w7[1] = wC[3];
    }
    probe_mark(5);
#if LVB_HOOK_PASS == 0
    hook();
#endif
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int n = 0; n < 8; n += (n & 1) ? 3 : 1) ct(X[p][n], X[p][n + 2], w6[n >> 2]);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int n = 0; n < 8; n += 4) {
        ct(X[p][n], X[p][n + 1], w7[n >> 2]);
        ct_mi(X[p][n + 2], X[p][n + 3], w7[n >> 2]);
      }
  }
  // L_C -> L_D (TMEM); pass D (L_D: regs (x0, x1, x6), lanes (x2, x3, x4,
  // x5, x7)): level 8 on x1, block x >> 2 = 64 w + 32 L4 + 16 x6 + (L & 15);
  // level 9 on x0, block 2 (x >> 2) + x1
  {
    double2 wD[4];  // w8 per x6; w9 per x6 (odd level-9 blocks, x1 = 1: -i w9)
    double2 w8[2], w9[2];
    if constexpr (kTm) {
      tws.fwdD(wD);
    } else {
      const uint32_t b8 = 64 * w + 32 * (L >> 4) + (L & 15);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        w8[q] = twf(twsrc, 8, b8 + 16 * q);
        w9[q] = twf(twsrc, 9, 2 * (b8 + 16 * q));
      }
    }
    probe_mark(6);
#if LVB_HOOK_PASS == 1
    hook();
#endif
    tm_trip_fwd<P>(X, tm);
#if LVB_HOOK_PASS == 2
    hook();
#endif
    if constexpr (kTm) {
      tws.ready(wD);
      w8[0] = wD[0];
      w8[1] = wD[1];
      w9[0] = wD[2];
      w9[1] = wD[3];
    }
    probe_mark(7);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int n = 0; n < 8; n += (n & 1) ? 3 : 1) ct(X[p][n], X[p][n + 2], w8[n >> 2]);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int n = 0; n < 8; n += 4) {
        ct(X[p][n], X[p][n + 1], w9[n >> 2]);
        ct_mi(X[p][n + 2], X[p][n + 3], w9[n >> 2]);
      }
  }
}

// ------------------------------------------------------------- inverse
// Cyclic DIT inverse (oracle fft_inv): stage s pairs bit x(9-s), j = x mod
// 2^(9-s), twiddle conj(W^(j << s)). X[p][r] on entry: the spectrum in
// L_D. On exit: L_A (x = t + 128 r), the layout fft_forward's input uses,
// so each thread owns the same accumulator coefficients in both halves of
// a CMUX. The cross-warp exchange starts with a CTA barrier (other warps
// may still read buf). The untwist is the caller's.
template <int P, int NB = kXchgBufs, typename Bar = CtaBar, typename TW = const double2*>
__device__ __forceinline__ void fft_inverse_a(double2 (&X)[P][8], double2* buf, TW twsrc,
                                              uint32_t t, uint32_t tm, Bar bar = Bar()) {
  const uint32_t L = t & 31, w = t >> 5;
  constexpr bool kTm = std::is_same<TW, TwTmem>::value;
  const auto tws = tw_source(twsrc, t);
  // pass D': stages 9, 8 on (x0, x1) = regs (n0, n1): w in {1, i}
#pragma unroll
  for (int p = 0; p < P; ++p)
#pragma unroll
    for (int n = 0; n < 8; n += 4) dit4_1(X[p][n], X[p][n + 1], X[p][n + 2], X[p][n + 3]);
  // L_D -> L_C (TMEM); pass C': stage 7 on x2 = n0 (j = (x0, x1) = L >> 3),
  // stage 6 on x3 = n1 (j = (L >> 3) + 4 x2)
  {
    double2 vC[2];  // v7, v6 (stage 6, x2 = 1: i v6)
    double2 v7, v6;
    if constexpr (kTm) {
      tws.invC(vC);
    } else {
      const uint32_t j = L >> 3;
      v7 = twi(twsrc, j << 7);
      v6 = twi(twsrc, j << 6);
    }
    probe_mark(10);
    tm_trip_inv<P>(X, tm);
    if constexpr (kTm) {
      tws.ready(vC);
      v7 = vC[0];
      v6 = vC[1];
    }
    probe_mark(11);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int n = 0; n < 8; n += 2) ct(X[p][n], X[p][n + 1], v7);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int n = 0; n < 8; n += 4) {
        ct(X[p][n], X[p][n + 2], v6);
        ct_pi(X[p][n + 1], X[p][n + 3], v6);
      }
  }
  // L_C -> L_B (TMEM); pass B': stage 5 on x4 = r0 (j = u), stage 4 on
  // x5 = r1 (j = u + 16 x4), stage 3 on x6 = r2 (j = u + 16 (x4, x5))
  const uint32_t u = L >> 1;
  {
    double2 vB[4];  // v5, v4 (stage 4, x4 = 1: i v4), v3 per x4 (x5 = 1: i v3)
    double2 v5, v4, v3[2];
    if constexpr (kTm) {
      tws.invB(vB);
    } else {
      v5 = twi(twsrc, u << 5);
      v4 = twi(twsrc, u << 4);
#pragma unroll
      for (int q = 0; q < 2; ++q) v3[q] = twi(twsrc, (u << 3) + 128 * q);
    }
    probe_mark(12);
    tm_trip_inv<P>(X, tm);
    if constexpr (kTm) {
      tws.ready(vB);
      v5 = vB[0];
      v4 = vB[1];
      v3[0] = vB[2];
      v3[1] = vB[3];
    }
    probe_mark(13);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 8; r += 2) ct(X[p][r], X[p][r + 1], v5);
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 8; r += 4) {
        ct(X[p][r], X[p][r + 2], v4);
        ct_pi(X[p][r + 1], X[p][r + 3], v4);
      }
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        ct(X[p][r], X[p][r + 4], v3[r]);
        ct_pi(X[p][r + 2], X[p][r + 6], v3[r]);
      }
  }
  // L_B -> L_A (cross-warp); pass A': stage 2 on x7 = r0 (j = t), stage 1
  // on x8 = r1 (j = t + 128 x7), stage 0 on x9 = r2 (j = t + 128 (x7, x8))
  double2 vA[4];  // v2, v1 (stage 1, x7 = 1: i v1), v0 per x7 (x8 = 1: i v0)
  double2 v2, v1, v0[2];
  if constexpr (kTm) {
    tws.invA(vA);
  } else {
    v2 = twi(twsrc, t << 2);
    v1 = twi(twsrc, t << 1);
#pragma unroll
    for (int q = 0; q < 2; ++q) v0[q] = twi(twsrc, t + 128 * q);
  }
  probe_mark(14);
  bar.sync();
  xchg_cta<P, NB>(X, buf, bar, [&](int r) { return 16u * r + 128u * (L & 1) + u + 256u * w; },
                  [&](int r) { return t + 128u * r; });
  if constexpr (kTm) {
    tws.ready(vA);
    v2 = vA[0];
    v1 = vA[1];
    v0[0] = vA[2];
    v0[1] = vA[3];
  }
  probe_mark(15);
#pragma unroll
  for (int p = 0; p < P; ++p)
#pragma unroll
    for (int r = 0; r < 8; r += 2) ct(X[p][r], X[p][r + 1], v2);
#pragma unroll
  for (int p = 0; p < P; ++p)
#pragma unroll
    for (int r = 0; r < 8; r += 4) {
      ct(X[p][r], X[p][r + 2], v1);
      ct_pi(X[p][r + 1], X[p][r + 3], v1);
    }
#pragma unroll
  for (int p = 0; p < P; ++p)
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      ct(X[p][r], X[p][r + 4], v0[r]);
      ct_pi(X[p][r + 2], X[p][r + 6], v0[r]);
    }
}

// f64 -> Z_{2^64}, identical to oracle f64_to_torus. (An integer-pipe
// variant — exponent/mantissa shift for |y| >= 2^52 — measured slower on
// B200, 87-90 ms vs 82.5 ms per 4096 PBS, and was dropped.)
// Here r = floor(y 2^-64 + 1/2) (exact: |y 2^-64| < 2^32, so the sum keeps
// every bit) differs from the oracle's rint only on exact ties, where it
// yields d = -2^63 instead of +2^63 - 2^64 — the same residue — so no tie
// fix-up is needed, and d = y - r 2^64 is one exact FMA.
#ifndef LVB_FLOOR_MAGIC
#define LVB_FLOOR_MAGIC 0
#endif
__device__ __forceinline__ uint64_t f64_to_torus(double y) {
#if LVB_FLOOR_MAGIC  // floor by a round-down add of 1.5 * 2^52 (FP64 pipe instead of XU): exact
  const double C = 6755399441055744.0;
  const double r = __dadd_rn(__dadd_rd(__fma_rn(y, 0x1p-64, 0.5), C), -C);
#else
  const double r = floor(__fma_rn(y, 0x1p-64, 0.5));  // the product is exact
#endif
  const double d = __fma_rn(-r, 18446744073709551616.0, y);
  return (uint64_t)__double2ll_rn(d);
}

}  // namespace lvb
