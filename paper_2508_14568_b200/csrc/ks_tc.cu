// Key switch on the 5th-generation tensor cores (tcgen05.mma kind::i8).
//
// The batched LWE key switch (big key kN -> small key n) is a dense integer
// contraction: for B items, K = kN * ks_level = 10240 digits and n+1 = 881
// output coefficients,
//     out[m][c] = sum_k -d[m][k] * KSK[k][c]        (mod 2^64)
// With unsigned digits u = d + 4 in [0, 8) (bias repaid by ksk_bias, see
// keyswitch_kernel) and the u64 KSK split into 8 byte limbs, it becomes 8
// exact u8 x u8 -> s32 GEMMs (max accumulator 10240 * 7 * 255 < 2^31):
//     sum_k u K = sum_b 2^(8b) * (sum_k u * K_b)     (mod 2^64)
// A   = digits  [M_pad][K]   u8, K-major (written by ks_digits_kernel)
// B^T = KSK limbs [896*8][K] u8, K-major, row n = c*8 + b (keygen transposes)
// One CTA: M = 128 items x N = 256 limb-columns (32 output coefficients),
// accumulator in TMEM (256 columns), K streamed in 128-byte blocks through a
// double-buffered cp.async pipeline; one elected thread issues 4 MMAs
// (K = 32 each) per block and commits to an mbarrier; the epilogue reads TMEM
// (tcgen05.ld 32x32b), recombines the limbs and applies bias, body and the
// modulus switch. Bit-identical to the CUDA-core keyswitch_kernel.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "kernels.cuh"

namespace lvb {

constexpr uint32_t kKsK = kBig * kKsLevel;  // 10240
constexpr uint32_t kTcM = 128;
constexpr uint32_t kTcN = 256;              // limb columns per CTA (32 coefficients)
constexpr uint32_t kTcKB = 128;             // K bytes per pipeline stage
constexpr uint32_t kTcNumKB = kKsK / kTcKB;  // 80
constexpr uint32_t kTcCols = kTcN / 8;      // output coefficients per CTA

__device__ __forceinline__ uint64_t lin_coef_tc(const LinDesc& d, const uint64_t* pool,
                                                uint32_t stride, uint32_t j) {
  uint64_t v = 0;
  for (int q = 0; q < d.nterms; ++q)
    v += (uint64_t)(int64_t)d.coef[q] * pool[(size_t)d.slot[q] * stride + j];
  if (j == kBig) v += (uint64_t)(int64_t)d.body_const * kDelta;
  return v;
}

// digits[m][l * kN + j] = decomposition level l of input coefficient j, +4.
__global__ void ks_digits_kernel(const LinDesc* desc, const uint64_t* pool, uint32_t pool_stride,
                                 uint32_t count, uint8_t* digits, uint64_t* body) {
  const uint32_t m = blockIdx.y;
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  uint8_t* row = digits + (size_t)m * kKsK;
  if (m >= count) {
    if (j < kBig)
      for (int l = 0; l < (int)kKsLevel; ++l) row[l * kBig + j] = 4;
    return;
  }
  const LinDesc d = desc[m];
  if (j < kBig) {
    const uint64_t v = lin_coef_tc(d, pool, pool_stride, j);
    int64_t dd[kKsLevel];
    decomp<kKsLevel>(v, kKsBaseLog, dd);
#pragma unroll
    for (int l = 0; l < (int)kKsLevel; ++l) row[l * kBig + j] = (uint8_t)(dd[l] + 4);
  } else if (j == kBig) {
    body[m] = lin_coef_tc(d, pool, pool_stride, kBig);
  }
}

// Transposed byte limbs of the KSK: bt[(c*8 + b) * K + l*kN + j] = byte b of
// ksk[j][l][c]; rows for c > n are zero.
__global__ void ksk_limbs_kernel(const uint64_t* ksk, uint32_t n, uint8_t* bt) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;  // l * kN + j
  const uint32_t c = blockIdx.y;
  if (k >= kKsK) return;
  const uint32_t l = k / kBig, j = k % kBig;
  const uint64_t v = c <= n ? ksk[((size_t)j * kKsLevel + l) * (n + 1) + c] : 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) bt[((size_t)c * 8 + b) * kKsK + k] = (uint8_t)(v >> (8 * b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// UMMA shared-memory descriptor, K-major, no swizzle: core matrices of 8
// rows x 16 bytes; SBO = byte distance between 8-row groups, LBO = between
// the two 16-byte K chunks of one K=32 MMA. version = 1 (Blackwell).
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n\t"
      "DONE:\n\t}" ::"r"(bar),
      "r"(parity), "r"(0x989680u)
      : "memory");
}

// Epilogue shared by both GEMM forms: warp w reads TMEM lanes 32w..32w+31
// (its items), 32 columns (4 output coefficients x 8 limbs) at a time,
// recombines the limbs mod 2^64, repays the +4 digit bias, adds the body
// and stores the modulus-switched coefficient.
__device__ __forceinline__ void ks_epilogue(uint32_t tmem, uint32_t warp, uint32_t item,
                                            uint32_t nt, const uint64_t* __restrict__ bias,
                                            const uint64_t* __restrict__ body, uint32_t n,
                                            uint32_t count, uint16_t* ms, uint32_t ms_stride,
                                            uint64_t* small_out) {
  const uint32_t lane_base = (warp * 32) << 16;
#pragma unroll 1
  for (uint32_t ch = 0; ch < kTcN / 32; ++ch) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
        "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(tmem + lane_base + ch * 32));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (item < count) {
#pragma unroll
      for (uint32_t i = 0; i < 4; ++i) {
        const uint32_t c = nt * kTcCols + ch * 4 + i;
        if (c > n) continue;
        uint64_t s = 0;
#pragma unroll
        for (uint32_t b = 0; b < 8; ++b) s += (uint64_t)r[i * 8 + b] << (8 * b);
        uint64_t v = bias[c] - s;
        if (c == n) v += body[item];
        if (small_out) small_out[(size_t)item * (n + 1) + c] = v;
        ms[(size_t)item * ms_stride + c] = (uint16_t)modswitch(v);
      }
    }
  }
}

constexpr size_t kTcSmemA = kTcM * kTcKB;  // 16 KB
constexpr size_t kTcSmemB = kTcN * kTcKB;  // 32 KB
constexpr size_t kTcSmem = 2 * (kTcSmemA + kTcSmemB) + 1024;

__global__ void __launch_bounds__(128, 1)
ks_mma_kernel(const uint8_t* __restrict__ digits, const uint8_t* __restrict__ bt,
              const uint64_t* __restrict__ bias, const uint64_t* __restrict__ body, uint32_t n,
              uint32_t count, uint16_t* ms, uint32_t ms_stride, uint64_t* small_out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sA = smem;                      // [2][16 KB]
  unsigned char* sB = smem + 2 * kTcSmemA;       // [2][32 KB]
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t taddr_s;

  const uint32_t t = threadIdx.x, warp = t >> 5;
  const uint32_t m0 = blockIdx.y * kTcM;
  const uint32_t nt = blockIdx.x;  // limb rows [nt*256, nt*256+256)

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&taddr_s)),
                 "r"(kTcN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = taddr_s;

  // global sources of this CTA's tiles
  const uint8_t* gA = digits + (size_t)(m0 + t) * kKsK;              // row t of the A tile
  const uint8_t* gB0 = bt + ((size_t)nt * kTcN + t) * kKsK;          // rows t, t+128 of B
  const uint8_t* gB1 = bt + ((size_t)nt * kTcN + t + 128) * kKsK;

  auto load_stage = [&](uint32_t kb, uint32_t s) {
    const uint32_t a = smem_u32(sA + s * kTcSmemA), b = smem_u32(sB + s * kTcSmemB);
    const uint32_t ko = kb * kTcKB;
#pragma unroll
    for (uint32_t c = 0; c < kTcKB / 16; ++c) {
      cp_async16(a + c * (kTcM * 16) + t * 16, gA + ko + c * 16);
      cp_async16(b + c * (kTcN * 16) + t * 16, gB0 + ko + c * 16);
      cp_async16(b + c * (kTcN * 16) + (t + 128) * 16, gB1 + ko + c * 16);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  // instruction descriptor: S32 accumulate, A/B unsigned 8-bit, K-major,
  // N = 256 (n_dim = N >> 3), M = 128 (m_dim = M >> 4)
  const uint32_t idesc = (2u << 4) | (0u << 7) | (0u << 10) | ((kTcN >> 3) << 17) | ((kTcM >> 4) << 24);

  load_stage(0, 0);
  for (uint32_t kb = 0; kb < kTcNumKB; ++kb) {
    const uint32_t s = kb & 1;
    asm volatile("cp.async.wait_all;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (t == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a = smem_u32(sA + s * kTcSmemA), b = smem_u32(sB + s * kTcSmemB);
#pragma unroll
      for (uint32_t q = 0; q < kTcKB / 32; ++q) {
        const uint64_t da = umma_desc(a + 2 * q * (kTcM * 16), kTcM * 16, 128);
        const uint64_t db = umma_desc(b + 2 * q * (kTcN * 16), kTcN * 16, 128);
        const uint32_t acc = (kb > 0 || q > 0) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&mbar[s]))
                   : "memory");
    }
    if (kb + 1 < kTcNumKB) {
      // buffer s^1 was read by the MMAs of block kb-1: wait for their commit
      if (kb >= 1) mbar_wait(smem_u32(&mbar[s ^ 1]), ((kb - 1) >> 1) & 1);
      load_stage(kb + 1, s ^ 1);
    }
  }
  mbar_wait(smem_u32(&mbar[(kTcNumKB - 1) & 1]), ((kTcNumKB - 1) >> 1) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;");

  ks_epilogue(tmem, warp, m0 + t, nt, bias, body, n, count, ms, ms_stride, small_out);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTcN));
}

size_t ks_tc_smem_bytes() { return kTcSmem; }

// ---------------------------------------------------------------- TMA form
// Same GEMM, operands staged by the Tensor Memory Accelerator: per K block
// (128 bytes) one 2D box of A (128 item rows) and one of B (256 limb rows)
// land in shared memory in the 128-byte-swizzled K-major layout the UMMA
// descriptors read directly (SWIZZLE_128B, 8-row groups 1024 B apart); a
// 4-stage ring of full/empty mbarriers decouples the producer thread (TMA)
// from the MMA-issuing thread, so the tensor cores never wait on a CTA-wide
// barrier. Bit-identical to ks_mma_kernel.
constexpr uint32_t kTmaStages = 4;
constexpr uint32_t kTmaStageBytes = kTcSmemA + kTcSmemB;  // 48 KB

__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int32_t c0,
                                            int32_t c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

__global__ void __launch_bounds__(128, 1)
ks_mma_tma_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                  const uint64_t* __restrict__ bias, const uint64_t* __restrict__ body, uint32_t n,
                  uint32_t count, uint16_t* ms, uint32_t ms_stride, uint64_t* small_out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[kTmaStages], empty[kTmaStages], done;
  __shared__ uint32_t taddr_s;

  const uint32_t t = threadIdx.x, warp = t >> 5;
  const uint32_t m0 = blockIdx.y * kTcM;
  const uint32_t nt = blockIdx.x;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&taddr_s)),
                 "r"(kTcN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    for (uint32_t s = 0; s < kTmaStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[s])));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_b)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = taddr_s;

  if (t == 0) {
    // producer: K block kb into stage kb % S once its previous MMAs committed
    for (uint32_t kb = 0; kb < kTcNumKB; ++kb) {
      const uint32_t s = kb % kTmaStages;
      if (kb >= kTmaStages) mbar_wait(smem_u32(&empty[s]), ((kb / kTmaStages) - 1) & 1);
      const uint32_t a = smem_u32(smem + s * kTmaStageBytes), b = a + kTcSmemA;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                       smem_u32(&full[s])),
                   "r"(kTmaStageBytes)
                   : "memory");
      tma_load_2d(a, &tm_a, (int32_t)(kb * kTcKB), (int32_t)m0, smem_u32(&full[s]));
      tma_load_2d(b, &tm_b, (int32_t)(kb * kTcKB), (int32_t)(nt * kTcN), smem_u32(&full[s]));
    }
  } else if (t == 32) {
    // MMA issuer: 4 x (K = 32) per block, commit frees the stage
    const uint32_t idesc =
        (2u << 4) | (0u << 7) | (0u << 10) | ((kTcN >> 3) << 17) | ((kTcM >> 4) << 24);
    for (uint32_t kb = 0; kb < kTcNumKB; ++kb) {
      const uint32_t s = kb % kTmaStages;
      mbar_wait(smem_u32(&full[s]), (kb / kTmaStages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a = smem_u32(smem + s * kTmaStageBytes), b = a + kTcSmemA;
#pragma unroll
      for (uint32_t q = 0; q < kTcKB / 32; ++q) {
        const uint64_t da = umma_desc_sw128(a + q * 32), db = umma_desc_sw128(b + q * 32);
        const uint32_t acc = (kb > 0 || q > 0) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&empty[s]))
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(&done))
                 : "memory");
  }
  mbar_wait(smem_u32(&done), 0);
  __syncwarp();
  asm volatile("tcgen05.fence::after_thread_sync;");

  ks_epilogue(tmem, warp, m0 + t, nt, bias, body, n, count, ms, ms_stride, small_out);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTcN));
}

size_t ks_tma_smem_bytes() { return kTmaStages * kTmaStageBytes + 1024; }

// Host: 2D tensor maps (K bytes innermost, rows), 128 x rows boxes,
// 128-byte swizzle. cuTensorMapEncodeTiled through the runtime's driver
// entry point (no libcuda link dependency).
bool make_ks_tensor_map(CUtensorMap* map, const uint8_t* base, uint64_t rows, uint32_t box_rows) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    encode = reinterpret_cast<EncodeFn>(fn);
  }
  const cuuint64_t dims[2] = {kKsK, rows};
  const cuuint64_t strides[1] = {kKsK};
  const cuuint32_t box[2] = {kTcKB, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(base), dims, strides,
                box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

uint32_t ks_tc_ntiles(uint32_t n) { return (n + 1 + kTcCols - 1) / kTcCols; }

}  // namespace lvb
