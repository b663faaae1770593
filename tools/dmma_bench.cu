// Does the FP64 tensor path (mma.sync m8n8k4 f64) add throughput on top of
// the FP64 vector pipe on B200? Measures DMMA alone, DFMA alone and both
// issued by different warps of the same CTAs. Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_bench tools/dmma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

// mode 0: all warps DMMA; 1: all warps DFMA; 2: even warps DMMA, odd warps DFMA
__global__ void k(double* out, int mode) {
  const int warp = threadIdx.x >> 5;
  const bool use_mma = mode == 0 || (mode == 2 && (warp & 1) == 0);
  double r = 0;
  if (use_mma) {
    double acc[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = threadIdx.x * 1e-3 + j;
    const double a = 1.0000001, b = 0.9999999;
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
      for (int j = 0; j < 8; ++j) dmma(acc[j], a, b);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) r += acc[j][0] + acc[j][1];
  } else {
    double x[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = threadIdx.x * 1e-3 + j;
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
      for (int j = 0; j < 16; ++j) x[j] = __fma_rn(x[j], 1.0000001, 0.5);
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) r += x[j];
  }
  if (r == -1.0) out[0] = r;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[3] = {"DMMA only", "DFMA only", "DMMA + DFMA (alternate warps)"};
  for (int mode = 0; mode < 3; ++mode) {
    const int blocks = sms * 4, threads = 256;
    k<<<blocks, threads>>>(d, mode);
    cudaEventRecord(e0);
    k<<<blocks, threads>>>(d, mode);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = (double)blocks * threads / 32;
    double mma_warps = mode == 0 ? warps : (mode == 2 ? warps / 2 : 0);
    double fma_warps = mode == 1 ? warps : (mode == 2 ? warps / 2 : 0);
    // m8n8k4: 8*8*4 FMAs = 512 flops per warp instruction; DFMA 32 FMAs = 64 flops
    const double flops = mma_warps * kIters * 8 * 512.0 + fma_warps * kIters * 16 * 64.0;
    printf("%-32s %8.3f ms  %7.2f TFLOP/s  (err=%s)\n", names[mode], ms, flops / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
