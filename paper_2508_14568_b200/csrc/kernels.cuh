// Kernel argument structs and launch wrappers (host <-> device contract).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "common.cuh"

namespace lvb {

// A linear combination of pool ciphertexts plus a public constant:
//   sum_q coef[q] * pool[slot[q]] + body_const * Delta.
// Covers add/sub/scalar_mul/scalar_add/trivial and the fused prologues
// (key = 3 dh - dv + eq9 + 4, fold z = 2x - 2y - eq + 1, ...).
struct LinDesc {
  uint32_t slot[4];
  int32_t coef[4];
  int32_t nterms;
  int32_t body_const;
};

struct LinOut {
  static constexpr int kMaxOut = 2;
  LinDesc d[kMaxOut];
  uint32_t out_slot[kMaxOut];
  int32_t nout;
};

// Blind-rotation epilogue of one item.
//   mode 0: pool[slot_a] = extract + body_add * Delta
//   mode 1: Leuvenshtein cell (kernel.cpp:159-162), in place on the frontier:
//           dv = pool[slot_a], dh = pool[slot_b] (read first), then
//           pool[slot_a] = step - dh, pool[slot_b] = step - dv, with optional
//           snapshots of the new dv / dh into snap_dv / snap_dh (~0u = none).
struct BrOut {
  uint32_t mode;
  uint32_t slot_a;
  uint32_t slot_b;
  uint32_t snap_dv;
  uint32_t snap_dh;
  int32_t body_add;
};
constexpr uint32_t kNoSlot = 0xFFFFFFFFu;

struct BrArgs {
  const uint16_t* ms;          // [count][ms_stride] modulus-switched small LWE
  uint32_t ms_stride;
  const uint32_t* lut_of_item; // [count] test polynomial index
  const uint64_t* test_polys;  // [luts][N]
  const double2* bskf;         // Fourier BSK, MAC layout
  const double2* twiddles;     // per-stage tables T_s (fft.cuh)
  const double2* twist;        // fine twist table zeta^j, j < 128
  uint32_t n;
  uint64_t* pool;              // pool base
  uint32_t pool_stride;
  const BrOut* outs;           // [count]
  uint64_t* glwe_out = nullptr;  // debug: full accumulator [count][2][N] (noise tests)
  // optional completion counters, one per done_chunk items: each CTA adds 1
  // after its outputs are globally visible (lv_pbs_batch_host downloads a
  // chunk as soon as its counter is full)
  uint32_t* done = nullptr;
  uint32_t done_chunk = 1;
};

struct KsArgs {
  const LinDesc* desc;  // [count]
  const uint64_t* pool;
  uint32_t pool_stride;
  const uint64_t* ksk;  // [kN][ks_level][n+1]
  const uint64_t* ksk_bias;  // [n+1] 4 * sum_j,l ksk[j][l][c]
  uint32_t n;
  uint32_t count;
  uint16_t* ms;         // [count][ms_stride]
  uint32_t ms_stride;
  uint64_t* small_out;  // optional [count][n+1] (parity/debug)
};

struct LinArgs {
  const LinOut* ops;
  uint64_t* pool;
  uint32_t pool_stride;
  uint32_t count;
};

struct EncArgs {
  uint64_t* pool;
  uint32_t pool_stride;
  const uint32_t* slots;
  const int32_t* values;
  const uint8_t* sk_glwe;
  uint64_t seed;
  uint64_t counter0;
  uint32_t noise_log2;
  int trivial;
};

struct PhaseArgs {
  const uint64_t* pool;
  uint32_t pool_stride;
  const uint32_t* slots;
  const uint8_t* sk_glwe;
  uint64_t* phase;
};

__global__ void blind_rotate_kernel(BrArgs a);        // lv_params.exact_mask_product = 0
__global__ void blind_rotate_exact_kernel(BrArgs a);  // lv_params.exact_mask_product = 1
size_t blind_rotate_smem_bytes(uint32_t n, bool exact);
__global__ void blind_rotate_pair_kernel(BrArgs a);
__global__ void blind_rotate_pair_exact_kernel(BrArgs a);  // exact_mask_product keys
size_t blind_rotate_pair_smem_bytes(uint32_t n);
__global__ void keyswitch_kernel(KsArgs a);
__global__ void linear_kernel(LinArgs a);
__global__ void encrypt_kernel(EncArgs a);
__global__ void phase_kernel(PhaseArgs a);
__global__ void keygen_secret_kernel(uint64_t seed, uint32_t n, uint8_t* sk_small, uint8_t* sk_glwe);
__global__ void ksk_bias_kernel(const uint64_t* ksk, uint32_t n, uint64_t* bias);
__global__ void keygen_ksk_kernel(uint64_t seed, uint32_t n, uint32_t noise_log2,
                                  const uint8_t* sk_small, const uint8_t* sk_glwe, uint64_t* ksk);
__global__ void keygen_bsk_kernel(uint64_t seed, uint32_t noise_log2, const uint8_t* sk_small,
                                  const uint8_t* sk_glwe, uint64_t* bsk);
__global__ void bsk_fourier_kernel(const uint64_t* polys, uint32_t nouts, const double4* tw_dd,
                                   const double4* twist_dd, double2* bskf);
__global__ void bsk_fourier_f64_kernel(const uint64_t* polys, uint32_t nouts, const double2* tw,
                                       double2* bskf);
__global__ void bsk_split_kernel(const uint64_t* bsk, uint64_t* split);
__global__ void fft_forward_debug_kernel(const int64_t* poly, const double2* tw,
                                         const double2* twist, double2* spec);
__global__ void fft_backward_debug_kernel(const double2* spec, const double2* tw,
                                          const double2* twist, uint64_t* poly);

__global__ void fp64_peak_kernel(double* out, int iters, double seed);
__global__ void flush_kernel(uint4* buf, size_t n16);

void set_twist_coarse(const double2* host8);
void set_fwd_consts(const double2* host7);

constexpr int kKsItems = 32;

}  // namespace lvb

namespace lvb {
// tensor-core key switch (ks_tc.cu)
__global__ void ks_digits_kernel(const LinDesc* desc, const uint64_t* pool, uint32_t pool_stride,
                                 uint32_t count, uint8_t* digits, uint64_t* body);
__global__ void ksk_limbs_kernel(const uint64_t* ksk, uint32_t n, uint8_t* bt);
__global__ void ks_mma_kernel(const uint8_t* digits, const uint8_t* bt, const uint64_t* bias,
                              const uint64_t* body, uint32_t n, uint32_t count, uint16_t* ms,
                              uint32_t ms_stride, uint64_t* small_out);
size_t ks_tc_smem_bytes();
__global__ void ks_mma_tma_kernel(const __grid_constant__ CUtensorMap tm_a,
                                  const __grid_constant__ CUtensorMap tm_b, const uint64_t* bias,
                                  const uint64_t* body, uint32_t n, uint32_t count, uint16_t* ms,
                                  uint32_t ms_stride, uint64_t* small_out);
size_t ks_tma_smem_bytes();
bool make_ks_tensor_map(CUtensorMap* map, const uint8_t* base, uint64_t rows, uint32_t box_rows);
uint32_t ks_tc_ntiles(uint32_t n);
}  // namespace lvb
