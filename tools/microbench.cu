// Throughput microbenchmarks for design decisions (not part of the product):
// LDS.128 / STS.128, SHFL, tcgen05.ld/st (TMEM), DFMA. Prints per-SM rates.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lds(double2* out, int iters) {
  __shared__ double2 buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_double2(i, i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  unsigned idx = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      double2 v = buf[(idx + k * 128) & 2047];
      acc.x += v.x;
      acc.y += v.y;
    }
    idx += 32;
  }
  if (acc.x == -1) out[0] = acc;
}

__global__ void k_sts(double2* out, int iters) {
  __shared__ double2 buf[2048];
  unsigned idx = threadIdx.x;
  double2 v = make_double2(threadIdx.x, 1);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) buf[(idx + k * 128) & 2047] = v;
    idx += 32;
    v.x += 1;
  }
  __syncthreads();
  if (buf[threadIdx.x].x == -1) out[0] = buf[0];
}

__global__ void k_shfl(double* out, int iters) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = __shfl_xor_sync(0xffffffffu, a[k], 1 + (k & 7));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == -1) out[0] = s;
}

__global__ void k_dfma(double* out, int iters) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = __fma_rn(a[k], 0.99999, 1e-9);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == -1) out[0] = s;
}

// LDS.128 and SHFL in the same SM: even warps run the k_lds loop, odd
// warps the k_shfl loop (does SHFL share the shared-memory data pipe?)
__global__ void k_mix(double* out, int iters, int mode) {
  __shared__ double2 buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_double2(i, i);
  __syncthreads();
  const int w = threadIdx.x / 32;
  const bool lds = mode == 0 ? true : mode == 1 ? false : (w & 1) == 0;
  if ((mode == 3 && (w & 1)) ) return;  // mode 3: only the even (LDS) half runs
  if ((mode == 4 && !(w & 1))) return;  // mode 4: only the odd (SHFL) half runs
  double s = 0;
  if (mode == 3 || (mode == 2 && lds) || mode == 0) {
    double2 acc = make_double2(0, 0);
    unsigned idx = threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        double2 v = buf[(idx + k * 128) & 2047];
        acc.x += v.x;
        acc.y += v.y;
      }
      idx += 32;
    }
    s = acc.x + acc.y;
  } else {
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x + k;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = __shfl_xor_sync(0xffffffffu, a[k], 1 + (k & 7));
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
  }
  if (s == -1) out[0] = s;
}

// TMEM: each warp stores/loads 32 lanes x 32 columns (x32) repeatedly.
__global__ void k_tmem(unsigned* out, int iters, int do_load) {
  __shared__ unsigned taddr_s;
  const unsigned warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned base = taddr_s + ((warp * 32) << 16);
  unsigned r[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) r[k] = threadIdx.x * 7 + k;
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
    const unsigned col = (it & 3) * 32;
    if (do_load) {
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
            "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
            "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
            "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(base + col));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int k = 0; k < 32; ++k) acc += r[k];  // static indices (no local-memory copy)
    } else {
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
          "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(base + col),
          "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
          "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
          "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
          "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
          "r"(r[29]), "r"(r[30]), "r"(r[31]));
#pragma unroll
      for (int k = 0; k < 32; ++k) r[k] += 1;
    }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(taddr_s));
  if (acc == 12345) out[0] = acc;
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
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* d;
  cudaMalloc(&d, 64);
  const int blocks = sms * 4, threads = 128, iters = 4096;
  float ms;
  ms = timeit([&] { k_lds<<<blocks, threads>>>((double2*)d, iters); });
  double ops = (double)blocks * threads / 32 * iters * 8;  // warp-instructions
  printf("LDS.128: %.3f warp-instr/clk/SM (%.1f B/clk/SM)\n", ops / (ms * 1e-3) / sms / (clk * 1e3),
         ops * 512 / (ms * 1e-3) / sms / (clk * 1e3));
  ms = timeit([&] { k_sts<<<blocks, threads>>>((double2*)d, iters); });
  printf("STS.128: %.3f warp-instr/clk/SM\n", ops / (ms * 1e-3) / sms / (clk * 1e3));
  ms = timeit([&] { k_shfl<<<blocks, threads>>>(d, iters); });
  ops = (double)blocks * threads / 32 * iters * 8 * 2;  // double shuffle = 2 SHFL
  printf("SHFL.32: %.3f warp-instr/clk/SM\n", ops / (ms * 1e-3) / sms / (clk * 1e3));
  ms = timeit([&] { k_dfma<<<blocks, threads>>>(d, iters); });
  ops = (double)blocks * threads / 32 * iters * 8;
  printf("DFMA: %.3f warp-instr/clk/SM\n", ops / (ms * 1e-3) / sms / (clk * 1e3));
  for (int ld = 0; ld < 2; ++ld) {
    ms = timeit([&] { k_tmem<<<sms * 4, 128>>>((unsigned*)d, iters, ld); });
    ops = (double)sms * 4 * 4 * iters;  // warp-instructions, each 32 lanes x 32 cols x 4 B = 4 KB
    printf("tcgen05.%s 32x32b.x32: %.3f warp-instr/clk/SM = %.1f B/clk/SM (err=%s)\n", ld ? "ld" : "st",
           ops / (ms * 1e-3) / sms / (clk * 1e3), ops * 4096 / (ms * 1e-3) / sms / (clk * 1e3),
           cudaGetErrorString(cudaGetLastError()));
  }
  {
    const char* nm[5] = {"all LDS", "all SHFL", "half LDS + half SHFL", "half LDS only",
                         "half SHFL only"};
    for (int m = 0; m < 5; ++m) {
      ms = timeit([&] { k_mix<<<sms * 4, 256>>>(d, iters, m); });
      printf("mix %-22s %.3f ms\n", nm[m], ms);
    }
  }
  printf("clock %d kHz (nominal attr)\n", clk);
  return 0;
}
