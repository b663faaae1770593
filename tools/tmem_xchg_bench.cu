// Design microbenchmark (not part of the product): can TMEM round trips
// (tcgen05.st 32x32b -> tcgen05.ld 16x256b) take the warp-local FFT
// exchanges off the shared-memory data path?
//   1. checks the 16x256b fragment mapping used by the blind rotation
//      (thread t0 + 4 t1 <- lane t1 + 8h (+16g), 64-bit column t0 + 4k);
//   2. times, at 3 CTAs x 128 threads per SM and P = 2 polynomials per
//      thread, an emulated transform pass structure:
//        cur : [W] xchg(cross-warp smem) [W] xchg(warp smem) [W] shfl stage [W]
//        tmem: [W] xchg(cross-warp smem) [W] trip            [W] trip       [W]
//      where W is a radix-4 + radix-2 butterfly group on the 8 points;
//   3. pure exchange loops (no FP64) for each mechanism, alone and mixed.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_xchg_bench tools/tmem_xchg_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kM = 1024;

__device__ __forceinline__ uint32_t swz(uint32_t x) {
  return x ^ ((((x >> 3) & 7u) ^ (((x >> 9) & 1u) << 2)));
}
__device__ __forceinline__ double2 add2(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 sub2(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  const double t1 = __dmul_rn(a.y, b.y);
  const double t2 = __dmul_rn(a.y, b.x);
  return make_double2(__fma_rn(a.x, b.x, -t1), __fma_rn(a.x, b.y, t2));
}
__device__ __forceinline__ void dif4(double2& x0, double2& x1, double2& x2, double2& x3, double2 w1,
                                     double2 w2, double2 w3) {
  const double2 A = add2(x0, x2), B = add2(x1, x3), C = sub2(x0, x2), d = sub2(x1, x3);
  const double2 D = make_double2(d.y, -d.x);
  x0 = add2(A, B);
  x1 = cmul(sub2(A, B), w2);
  x2 = cmul(add2(C, D), w1);
  x3 = cmul(sub2(C, D), w3);
}
template <int P>
__device__ __forceinline__ void work(double2 (&X)[P][8], double2 w1, double2 w2, double2 w3) {
#pragma unroll
  for (int p = 0; p < P; ++p) {
#pragma unroll
    for (int r = 0; r < 2; ++r) dif4(X[p][r], X[p][r + 2], X[p][r + 4], X[p][r + 6], w1, w2, w3);
#pragma unroll
    for (int r = 0; r < 8; r += 2) {
      const double2 s = add2(X[p][r], X[p][r + 1]), d = sub2(X[p][r], X[p][r + 1]);
      X[p][r] = s;
      X[p][r + 1] = cmul(d, w2);
    }
  }
}

// ---- TMEM helpers (planar: re of point r at 64-bit column r, im at 8 + r)
__device__ __forceinline__ uint32_t lo(double v) { return (uint32_t)__double_as_longlong(v); }
__device__ __forceinline__ uint32_t hi(double v) { return (uint32_t)(__double_as_longlong(v) >> 32); }
__device__ __forceinline__ double mk(uint32_t l, uint32_t h) {
  return __longlong_as_double(((long long)h << 32) | l);
}

__device__ __forceinline__ void st_32x32b(uint32_t addr, const double2 (&X)[8]) {
  uint32_t r[32];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    r[2 * k] = lo(X[k].x);
    r[2 * k + 1] = hi(X[k].x);
    r[16 + 2 * k] = lo(X[k].y);
    r[16 + 2 * k + 1] = hi(X[k].y);
  }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(addr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
      "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]),
      "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]),
      "r"(r[30]), "r"(r[31])
      : "memory");
}
#define LD16(addr, a)                                                                              \
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12," \
               "%13,%14,%15}, [%16];"                                                              \
               : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]),           \
                 "=r"(a[6]), "=r"(a[7]), "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11]),         \
                 "=r"(a[12]), "=r"(a[13]), "=r"(a[14]), "=r"(a[15])                                \
               : "r"(addr)                                                                         \
               : "memory")
// X[h + 2g + 4k'] = (lane t1 + 8h + 16g, point t0 + 4k') of the stored array
__device__ __forceinline__ void ld_16x256b(uint32_t addr, double2 (&X)[8]) {
  uint32_t a[16], b[16];
  LD16(addr, a);
  LD16(addr + (16u << 16), b);
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      // re: regs 4*kk + 2h (+1); im: regs 4*(kk+2) + 2h (+1)
      X[h + 4 * kk] = make_double2(mk(a[4 * kk + 2 * h], a[4 * kk + 2 * h + 1]),
                                   mk(a[4 * (kk + 2) + 2 * h], a[4 * (kk + 2) + 2 * h + 1]));
      X[h + 2 + 4 * kk] = make_double2(mk(b[4 * kk + 2 * h], b[4 * kk + 2 * h + 1]),
                                       mk(b[4 * (kk + 2) + 2 * h], b[4 * (kk + 2) + 2 * h + 1]));
    }
}
template <int P>
__device__ __forceinline__ void trip(double2 (&X)[P][8], uint32_t base) {
#pragma unroll
  for (int p = 0; p < P; ++p) st_32x32b(base + p * 32, X[p]);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
#pragma unroll
  for (int p = 0; p < P; ++p) ld_16x256b(base + p * 32, X[p]);
}

template <int P, bool kWarp>
__device__ __forceinline__ void xchg(double2 (&X)[P][8], double2* buf, uint32_t t) {
  const uint32_t b = t >> 4, u = t & 15, c = t >> 1, v = t & 1;
#pragma unroll
  for (int p = 0; p < P; ++p) {
    if (kWarp) __syncwarp(); else __syncthreads();
#pragma unroll
    for (int r = 0; r < 8; ++r)
      buf[swz(kWarp ? 128 * b + u + 16 * r : t + 128 * r)] = X[p][r];
    if (kWarp) __syncwarp(); else __syncthreads();
#pragma unroll
    for (int r = 0; r < 8; ++r)
      X[p][r] = buf[swz(kWarp ? 16 * c + v + 2 * r : 128 * b + u + 16 * r)];
  }
}
template <int P>
__device__ __forceinline__ void shfl_stage(double2 (&X)[P][8], uint32_t t) {
  const uint32_t v = t & 1;
#pragma unroll
  for (int p = 0; p < P; ++p) {
    double2 Y[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double2 s = v ? X[p][q] : X[p][4 + q];
      Y[q] = make_double2(__shfl_xor_sync(~0u, s.x, 1), __shfl_xor_sync(~0u, s.y, 1));
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double2 e = v ? Y[q] : X[p][q], o = v ? X[p][4 + q] : Y[q];
      X[p][2 * q] = add2(e, o);
      X[p][2 * q + 1] = sub2(e, o);
    }
  }
}

__device__ uint32_t tmem_alloc(uint32_t* slot, uint32_t ncols) {
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(slot)), "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  return *slot;
}
__device__ void tmem_free(uint32_t base, uint32_t ncols) {
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(ncols));
}

// 1. mapping check
__global__ void k_check(int* bad) {
  __shared__ uint32_t slot;
  const uint32_t base0 = tmem_alloc(&slot, 32);
  const uint32_t t = threadIdx.x, w = t >> 5, L = t & 31;
  const uint32_t base = base0 + ((32u * w) << 16);
  double2 X[1][8];
#pragma unroll
  for (int r = 0; r < 8; ++r) X[0][r] = make_double2(L * 8 + r, -(double)(L * 8 + r) - 0.5);
  trip<1>(X, base);
  const uint32_t t0 = L & 3, t1 = L >> 2;
  int nb = 0;
#pragma unroll
  for (int n = 0; n < 8; ++n) {
    const uint32_t h = n & 1, g = (n >> 1) & 1, kk = n >> 2;
    const double e = (t1 + 8 * h + 16 * g) * 8 + t0 + 4 * kk;
    if (X[0][n].x != e || X[0][n].y != -e - 0.5) ++nb;
  }
  atomicAdd(bad, nb);
  tmem_free(base0, 32);
}

// 2. emulated transform passes. mode 0: current, 1: tmem
template <int kMode>
__global__ void __launch_bounds__(128, 3) k_pass(double* out, int iters) {
  __shared__ __align__(16) double2 buf[kM];
  __shared__ uint32_t slot;
  const uint32_t t = threadIdx.x;
  uint32_t base0 = 0, base = 0;
  if (kMode == 1) {
    base0 = tmem_alloc(&slot, 64);
    base = base0 + ((32u * (t >> 5)) << 16);
  }
  double2 X[2][8];
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int r = 0; r < 8; ++r) X[p][r] = make_double2(t + r + p, t - r);
  const double2 w1 = make_double2(0.7, 0.1 + t * 1e-4), w2 = make_double2(0.5, -0.3),
                w3 = make_double2(-0.2, 0.9);
  for (int it = 0; it < iters; ++it) {
    work<2>(X, w1, w2, w3);
    xchg<2, false>(X, buf, t);
    work<2>(X, w1, w2, w3);
    if (kMode == 0) {
      xchg<2, true>(X, buf, t);
      work<2>(X, w1, w2, w3);
      shfl_stage<2>(X, t);
    } else {
      trip<2>(X, base);
      work<2>(X, w1, w2, w3);
      trip<2>(X, base);
    }
    work<2>(X, w1, w2, w3);
  }
  double s = 0;
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int r = 0; r < 8; ++r) s += X[p][r].x + X[p][r].y;
  if (s == 1.2345) out[0] = s;
  if (kMode == 1) tmem_free(base0, 64);
}

// 3. pure exchange loops. mode 0 warp smem exchange, 1 tmem trip,
// 2 even warps smem / odd warps tmem, 3 only even warps (smem), 4 only odd (tmem)
__global__ void __launch_bounds__(128, 3) k_pure(double* out, int iters, int mode) {
  __shared__ __align__(16) double2 buf[kM];
  __shared__ uint32_t slot;
  const uint32_t t = threadIdx.x, w = t >> 5;
  const uint32_t base0 = tmem_alloc(&slot, 64);
  const uint32_t base = base0 + ((32u * w) << 16);
  double2 X[2][8];
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int r = 0; r < 8; ++r) X[p][r] = make_double2(t + r + p, t - r);
  const bool use_tmem = mode == 1 || ((mode == 2 || mode == 4) && (w & 1));
  const bool idle = (mode == 3 && (w & 1)) || (mode == 4 && !(w & 1));
  if (!idle) {
    for (int it = 0; it < iters; ++it) {
      if (use_tmem)
        trip<2>(X, base);
      else
        xchg<2, true>(X, buf, t);
      X[0][0].x += 1.0;
    }
  }
  double s = 0;
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int r = 0; r < 8; ++r) s += X[p][r].x + X[p][r].y;
  if (s == 1.2345) out[0] = s;
  tmem_free(base0, 64);
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaEventRecord(a);
  f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  int* bad;
  double* d;
  cudaMalloc(&bad, 4);
  cudaMalloc(&d, 64);
  cudaMemset(bad, 0, 4);
  k_check<<<1, 128>>>(bad);
  int hb = -1;
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
  printf("mapping check: err=%s mismatches=%d (of 1024)\n", cudaGetErrorString(e), hb);
  const int grid = sms * 3, iters = 2000;
  // per CTA-iteration: 1 "transform pair" (P=2) pass structure
  const double cta_iters = (double)grid * iters;
  float ms0 = timeit([&] { k_pass<0><<<grid, 128>>>(d, iters); });
  float ms1 = timeit([&] { k_pass<1><<<grid, 128>>>(d, iters); });
  printf("emulated transform (P=2, 3 CTAs/SM): current %.3f ms (%.0f SM-cyc per CTA-iter), tmem %.3f ms (%.0f) err=%s\n",
         ms0, ms0 * 1e-3 * clk * 1e3 * sms / cta_iters * 1.0, ms1,
         ms1 * 1e-3 * clk * 1e3 * sms / cta_iters, cudaGetErrorString(cudaGetLastError()));
  const char* nm[5] = {"warp smem xchg", "tmem trip", "half smem + half tmem", "half smem only",
                       "half tmem only"};
  for (int m = 0; m < 5; ++m) {
    float ms = timeit([&] { k_pure<<<grid, 128>>>(d, iters, m); });
    printf("pure %-24s %.3f ms  (%.0f SM-cyc per CTA-iter of P=2 exchange) err=%s\n", nm[m], ms,
           ms * 1e-3 * clk * 1e3 * sms / cta_iters, cudaGetErrorString(cudaGetLastError()));
  }
  printf("clock attr %d kHz, %d SMs\n", clk, sms);
  return 0;
}
