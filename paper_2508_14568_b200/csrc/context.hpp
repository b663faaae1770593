// lv_ctx: one keyset resident on one GPU, its ciphertext pool, LUT table,
// host ledgers and counters. Internal to the library (the C ABI in
// include/leuven_b200.h is the public surface).
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <atomic>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/leuven_b200.h"
#include "kernels.cuh"
#include "ledger.hpp"

namespace lvb {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char* what);
#define LV_CUDA(x) ::lvb::cuda_check((x), #x)

template <typename T>
struct DevBuf {  // grow-only device scratch buffer
  T* p = nullptr;
  size_t cap = 0;
  T* get(size_t n) {
    if (n > cap) {
      if (p) cudaFree(p);
      size_t c = std::max<size_t>(n, cap * 2);
      LV_CUDA(cudaMalloc(&p, c * sizeof(T)));
      cap = c;
    }
    return p;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// Scoped device allocation / event (freed on every exit path, exceptions
// included).
template <typename T>
struct DevTemp {
  T* p = nullptr;
  explicit DevTemp(size_t n) { LV_CUDA(cudaMalloc(&p, n * sizeof(T))); }
  ~DevTemp() {
    if (p) cudaFree(p);
  }
  DevTemp(const DevTemp&) = delete;
  DevTemp& operator=(const DevTemp&) = delete;
};
struct Event {
  cudaEvent_t e = nullptr;
  explicit Event(unsigned flags = cudaEventDefault) { LV_CUDA(cudaEventCreateWithFlags(&e, flags)); }
  ~Event() {
    if (e) cudaEventDestroy(e);
  }
  Event(const Event&) = delete;
  Event& operator=(const Event&) = delete;
};

// Epilogue of one blind-rotation item (see BrOut in kernels.cuh).
struct PbsItem {
  LinDesc in;        // key-switch prologue
  uint32_t lut;
  BrOut out;
};

}  // namespace lvb

struct lv_eqtable {
  uint64_t length = 0;
  std::map<char, std::vector<lv_ct>> rows;  // preprocess.hpp:18-39
};

struct lv_ctx {
  lv_params p{};
  uint64_t seed = 0;
  uint64_t key_id = 0;  // key-set fingerprint: hash of public key material (key_fingerprint), never the seed
  cudaStream_t stream = nullptr;
  cudaStream_t copy_out = nullptr;  // lv_pbs_batch_host: chunk downloads behind the compute
  int device = 0;
  std::recursive_mutex mu;

  // keys
  uint8_t* d_sk_small = nullptr;
  uint8_t* d_sk_glwe = nullptr;
  uint64_t* d_ksk = nullptr;
  uint64_t* d_ksk_bias = nullptr;
  double2* d_bskf = nullptr;
  double2* d_tw = nullptr;
  double2* d_twist = nullptr;

  // LUTs
  std::vector<std::array<int32_t, 16>> luts;
  uint64_t* d_tp = nullptr;
  uint32_t tp_cap = 0;

  // ciphertext pool
  uint64_t* d_pool = nullptr;
  uint32_t pool_cap = 0;
  std::vector<uint32_t> free_slots;
  std::vector<uint8_t> live;
  std::vector<lvb::NoiseLedger> ledgers;
  lvb::NoiseLedger::SourceId next_source = 1;
  uint64_t enc_counter = 0;

  std::atomic<uint64_t> pbs_count{0}, refresh_count{0}, linear_count{0};

  // scratch
  lvb::DevBuf<uint16_t> ms;
  lvb::DevBuf<lvb::LinDesc> desc;
  lvb::DevBuf<uint32_t> lut_item;
  lvb::DevBuf<lvb::BrOut> br_out;
  lvb::DevBuf<lvb::LinOut> lin_ops;
  lvb::DevBuf<uint32_t> u32a, u32b;
  lvb::DevBuf<int32_t> i32a;
  lvb::DevBuf<uint64_t> u64a, u64b;
  // tensor-core key switch: KSK byte limbs (transposed, K-major), digits, bodies
  uint8_t* d_ksk_bt = nullptr;
  CUtensorMap ksk_map;          // TMA view of d_ksk_bt (ks_mma_tma_kernel)
  bool ks_tma = false;
  lvb::DevBuf<uint8_t> ks_digits;
  lvb::DevBuf<uint64_t> ks_body;

  // traversal plans per grid shape, LRU-bounded by total cells (a server
  // scanning many string lengths must not grow it without limit); callers
  // hold shared_ptrs, so eviction never invalidates a running traversal
  std::map<std::string, std::pair<std::shared_ptr<const lvb::PairPlan>, uint64_t>> plan_cache;
  uint64_t plan_cache_cells = 0, plan_cache_tick = 0;
  uint32_t min_lut[2] = {0, 0};
  uint32_t br_pair_max = 0;  // waves up to this size run blind_rotate_pair_kernel
  uint32_t br_slots = 0;     // blind-rotation CTAs resident on the whole GPU at once
  uint32_t identity_lut = 0;
};

namespace lvb {

// Every entry point holds the context mutex and makes the context's device
// current on the calling thread (contexts on several GPUs, calls from any
// host thread).
struct CtxLock {
  std::lock_guard<std::recursive_mutex> lk;
  explicit CtxLock(lv_ctx* c) : lk(c->mu) { LV_CUDA(cudaSetDevice(c->device)); }
};

uint32_t ms_stride(const lv_ctx* c);
std::vector<lv_ct> pool_alloc(lv_ctx* c, size_t count);
void pool_free(lv_ctx* c, const lv_ct* cts, size_t count);
void check_handles(const lv_ctx* c, const lv_ct* cts, size_t count);
uint32_t lut_id(lv_ctx* c, const std::array<int32_t, 16>& e);

// Runs count PBS items (key switch with prologue, blind rotation with
// epilogue) on the context stream. Device pointers of the item arrays are
// uploaded here; pool slots must already exist.
void run_pbs_items(lv_ctx* c, const std::vector<PbsItem>& items);
void launch_pbs_dev(lv_ctx* c, const LinDesc* d_desc, const uint32_t* d_lut, const BrOut* d_out,
                    uint32_t count, cudaEvent_t ks_done = nullptr, uint32_t* done = nullptr,
                    uint32_t done_chunk = 1);
void run_linear(lv_ctx* c, const std::vector<LinOut>& ops);
void launch_linear_dev(lv_ctx* c, const LinOut* d_ops, uint32_t count);

}  // namespace lvb
