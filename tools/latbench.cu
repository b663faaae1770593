// Latency microbenchmarks (not part of the product): dependent-chain FP64
// latencies, CTA / cluster barrier round trips, shared and distributed
// shared memory load latency. Cycles via clock64() inside one kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o latbench tools/latbench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;
constexpr int kIters = 4096;

__global__ void k_chain(long long* out, double seed) {
  double a = seed, b = seed * 0.5;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < kIters; ++i) a = __dadd_rn(a, b);
  long long t1 = clock64();
#pragma unroll 16
  for (int i = 0; i < kIters; ++i) b = __fma_rn(b, 0.999, a);
  long long t2 = clock64();
  if (threadIdx.x == 0) {
    out[0] = t1 - t0;
    out[1] = t2 - t1;
  }
  if (a == b) out[7] = 1;
}

__global__ void k_sync(long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < kIters; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[2] = t1 - t0;
}

__global__ void __cluster_dims__(2, 1, 1) k_csync(long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < kIters; ++i) cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[3] = t1 - t0;
}

__global__ void __cluster_dims__(2, 1, 1) k_lds_chain(long long* out) {
  __shared__ unsigned nxt[1024];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) nxt[i] = (i * 37 + 11) & 1023;
  cl.sync();
  unsigned* remote = cl.map_shared_rank(nxt, cl.block_rank() ^ 1);
  unsigned p = threadIdx.x, q = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < kIters; ++i) p = nxt[p];
  long long t1 = clock64();
  for (int i = 0; i < kIters; ++i) q = remote[q];
  long long t2 = clock64();
  cl.sync();
  if (threadIdx.x == 0 && cl.block_rank() == 0) {
    out[4] = t1 - t0;
    out[5] = t2 - t1;
  }
  if (p == 12345678u && q == 1u) out[7] = 2;
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  cudaMemset(d, 0, 8 * sizeof(long long));
  long long h[8];
  k_chain<<<1, 32>>>(d, 1.000001);
  k_sync<<<1, 128>>>(d);
  k_csync<<<2, 128>>>(d);
  k_lds_chain<<<2, 32>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("err=%s\n", cudaGetErrorString(e));
  printf("DADD dependent latency: %.1f cyc\n", (double)h[0] / kIters);
  printf("DFMA dependent latency: %.1f cyc\n", (double)h[1] / kIters);
  printf("__syncthreads (128 thr): %.1f cyc\n", (double)h[2] / kIters);
  printf("cluster.sync (2 x 128 thr): %.1f cyc\n", (double)h[3] / kIters);
  printf("LDS dependent latency: %.1f cyc\n", (double)h[4] / kIters);
  printf("DSMEM dependent latency: %.1f cyc\n", (double)h[5] / kIters);
  return 0;
}
