// Host runtime: context lifecycle and key generation, the device ciphertext
// pool, the Backend operations (proj/include/leuven/backend.hpp:54-76) and
// the batched PBS driver, exposed through the C ABI in include/leuven_b200.h.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "context.hpp"

namespace lvb {

thread_local std::string g_last_error;

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(LV_ERR_CUDA, std::string("CUDA error ") + cudaGetErrorString(e) + " at " + what);
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return LV_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return LV_ERR_CUDA;
  }
}

uint32_t ms_stride(const lv_ctx* c) { return (c->p.n + 1 + 7) / 8 * 8; }

// ---------------------------------------------------------------- pool
static void pool_grow(lv_ctx* c, size_t need) {
  if (need <= c->pool_cap) return;
  size_t cap = std::max<size_t>(need, (size_t)c->pool_cap * 2);
  cap = std::max<size_t>(cap, 1024);
  uint64_t* np = nullptr;
  LV_CUDA(cudaMalloc(&np, cap * kBigStride * sizeof(uint64_t)));
  if (c->d_pool) {
    LV_CUDA(cudaMemcpyAsync(np, c->d_pool, (size_t)c->pool_cap * kBigStride * sizeof(uint64_t),
                            cudaMemcpyDeviceToDevice, c->stream));
    LV_CUDA(cudaStreamSynchronize(c->stream));
    LV_CUDA(cudaFree(c->d_pool));
  }
  c->d_pool = np;
  for (size_t s = cap; s-- > c->pool_cap;) c->free_slots.push_back((uint32_t)s);
  c->live.resize(cap, 0);
  c->ledgers.resize(cap);
  c->pool_cap = (uint32_t)cap;
}

std::vector<lv_ct> pool_alloc(lv_ctx* c, size_t count) {
  if (c->free_slots.size() < count) pool_grow(c, (size_t)c->pool_cap + count - c->free_slots.size());
  std::vector<lv_ct> out(count);
  for (size_t i = 0; i < count; ++i) {
    out[i] = c->free_slots.back();
    c->free_slots.pop_back();
    c->live[out[i]] = 1;
    c->ledgers[out[i]] = NoiseLedger();
  }
  // ascending slots: batches recycled through the LIFO free list come back
  // as long contiguous runs, so host<->device row copies stay one 2D copy
  std::sort(out.begin(), out.end());
  return out;
}

void pool_free(lv_ctx* c, const lv_ct* cts, size_t count) {
  for (size_t i = 0; i < count; ++i) {
    if (cts[i] < c->pool_cap && c->live[cts[i]]) {
      c->live[cts[i]] = 0;
      c->ledgers[cts[i]] = NoiseLedger();
      c->free_slots.push_back(cts[i]);
    }
  }
}

void check_handles(const lv_ctx* c, const lv_ct* cts, size_t count) {
  for (size_t i = 0; i < count; ++i)
    if (cts[i] >= c->pool_cap || !c->live[cts[i]])
      throw Error(LV_ERR_INVALID_HANDLE, "invalid ciphertext handle " + std::to_string(cts[i]));
}

// ---------------------------------------------------------------- LUTs
// Test polynomial of a Lut16 (lut.hpp:15-24): boxes of N/16 coefficients
// holding entries[m] * Delta, rotated by half a box (X^{-N/32}) so the
// rounding window of message m is centred; the negacyclic wrap of X^N = -1
// yields -entries[x-16] for x in [16,32) exactly as negacyclic_eval does
// (proj/src/lut.cpp:9-16).
static void build_test_poly(const std::array<int32_t, 16>& e, uint64_t* tp) {
  const uint32_t box = kN / 16, half = kN / 32;
  for (uint32_t j = 0; j < kN; ++j) {
    const uint32_t t = j + half;
    tp[j] = t < kN ? (uint64_t)(int64_t)e[t / box] * kDelta
                   : (uint64_t)0 - (uint64_t)(int64_t)e[(t - kN) / box] * kDelta;
  }
}

uint32_t lut_id(lv_ctx* c, const std::array<int32_t, 16>& e) {
  for (int v : e)
    if (v < 0 || v >= 32)
      throw Error(LV_ERR_OUT_OF_RANGE, "lookup entry outside [0,32): " + std::to_string(v));
  for (size_t i = 0; i < c->luts.size(); ++i)
    if (c->luts[i] == e) return (uint32_t)i;
  const uint32_t id = (uint32_t)c->luts.size();
  if (id >= c->tp_cap) {
    const uint32_t cap = std::max<uint32_t>(64, c->tp_cap * 2);
    uint64_t* np = nullptr;
    LV_CUDA(cudaMalloc(&np, (size_t)cap * kN * sizeof(uint64_t)));
    if (c->d_tp) {
      LV_CUDA(cudaMemcpyAsync(np, c->d_tp, (size_t)c->tp_cap * kN * 8, cudaMemcpyDeviceToDevice,
                              c->stream));
      LV_CUDA(cudaStreamSynchronize(c->stream));
      LV_CUDA(cudaFree(c->d_tp));
    }
    c->d_tp = np;
    c->tp_cap = cap;
  }
  std::vector<uint64_t> tp(kN);
  build_test_poly(e, tp.data());
  LV_CUDA(cudaMemcpyAsync(c->d_tp + (size_t)id * kN, tp.data(), kN * 8, cudaMemcpyHostToDevice,
                          c->stream));
  LV_CUDA(cudaStreamSynchronize(c->stream));
  c->luts.push_back(e);
  return id;
}

// ---------------------------------------------------------------- PBS driver
#ifndef LVB_KS_TC
#define LVB_KS_TC 1
#endif

// Key switch + modulus switch of `count` items (prologue descriptors d_desc)
// into d_ms: the tcgen05 i8 GEMM (ks_tc.cu) by default, the CUDA-core
// kernel with -DLVB_KS_TC=0 (kept for A/B measurement; both bit-exact).
static void launch_keyswitch(lv_ctx* c, const LinDesc* d_desc, uint32_t count, uint16_t* d_ms,
                             uint64_t* small_out) {
  const uint32_t stride = ms_stride(c);
  const uint32_t row = c->p.n + 1;
#if LVB_KS_TC
  constexpr uint32_t kChunk = 32768;  // items per GEMM launch (grid.y <= 65535 rows)
  const uint32_t rows_max = (std::min(count, kChunk) + 127) / 128 * 128;
  uint8_t* dig = c->ks_digits.get((size_t)rows_max * kBig * kKsLevel);
  uint64_t* body = c->ks_body.get(rows_max);
  for (uint32_t off = 0; off < count; off += kChunk) {
    const uint32_t cnt = std::min(count - off, kChunk);
    const uint32_t mt = (cnt + 127) / 128;
    ks_digits_kernel<<<dim3((kBig + 1 + 255) / 256, mt * 128), 256, 0, c->stream>>>(
        d_desc + off, c->d_pool, kBigStride, cnt, dig, body);
    CUtensorMap amap;
    if (c->ks_tma && make_ks_tensor_map(&amap, dig, (uint64_t)mt * 128, 128))
      ks_mma_tma_kernel<<<dim3(ks_tc_ntiles(c->p.n), mt), 128, ks_tma_smem_bytes(), c->stream>>>(
          amap, c->ksk_map, c->d_ksk_bias, body, c->p.n, cnt, d_ms + (size_t)off * stride, stride,
          small_out ? small_out + (size_t)off * row : nullptr);
    else
      ks_mma_kernel<<<dim3(ks_tc_ntiles(c->p.n), mt), 128, ks_tc_smem_bytes(), c->stream>>>(
          dig, c->d_ksk_bt, c->d_ksk_bias, body, c->p.n, cnt, d_ms + (size_t)off * stride, stride,
          small_out ? small_out + (size_t)off * row : nullptr);
  }
#else
  KsArgs ka{d_desc, c->d_pool, kBigStride, c->d_ksk, c->d_ksk_bias, c->p.n, count, d_ms, stride,
            small_out};
  for (uint32_t off = 0; off < count; off += 65535u * kKsItems) {
    const uint32_t cnt = std::min<uint32_t>(count - off, 65535u * kKsItems);
    KsArgs k2 = ka;
    k2.desc = d_desc + off;
    k2.count = cnt;
    k2.ms = d_ms + (size_t)off * stride;
    k2.small_out = small_out ? small_out + (size_t)off * row : nullptr;
    dim3 grid((row + 127) / 128, (cnt + kKsItems - 1) / kKsItems);
    keyswitch_kernel<<<grid, 128, 0, c->stream>>>(k2);
  }
#endif
  LV_CUDA(cudaGetLastError());
}

// Waves of at most br_pair_max items (default: one per SM) leave SMs idle in
// the single-CTA form; they run the CTA-pair form instead (2 CTAs per item).
// Keys with exact_mask_product use the exact-mask forms of both.
void launch_blind_rotate(lv_ctx* c, const BrArgs& ba, uint32_t count) {
  if (!count) return;
  if (c->p.exact_mask_product == 1 && count <= c->br_pair_max)
    blind_rotate_pair_exact_kernel<<<2 * count, 128, blind_rotate_pair_smem_bytes(c->p.n),
                                     c->stream>>>(ba);
  else if (c->p.exact_mask_product == 1)
    blind_rotate_exact_kernel<<<count, 128, blind_rotate_smem_bytes(c->p.n, true), c->stream>>>(ba);
  else if (count <= c->br_pair_max)
    blind_rotate_pair_kernel<<<2 * count, 128, blind_rotate_pair_smem_bytes(c->p.n), c->stream>>>(ba);
  else
    blind_rotate_kernel<<<count, 128, blind_rotate_smem_bytes(c->p.n, false), c->stream>>>(ba);
  LV_CUDA(cudaGetLastError());
}

void launch_pbs_dev(lv_ctx* c, const LinDesc* d_desc, const uint32_t* d_lut, const BrOut* d_out,
                    uint32_t count, cudaEvent_t ks_done, uint32_t* done, uint32_t done_chunk) {
  if (!count) return;
  const uint32_t stride = ms_stride(c);
  uint16_t* d_ms = c->ms.get((size_t)count * stride);
  launch_keyswitch(c, d_desc, count, d_ms, nullptr);
  if (ks_done) LV_CUDA(cudaEventRecord(ks_done, c->stream));
  BrArgs ba{d_ms, stride, d_lut, c->d_tp, c->d_bskf, c->d_tw, c->d_twist, c->p.n,
            c->d_pool, kBigStride, d_out};
  ba.done = done;
  ba.done_chunk = done_chunk;
  launch_blind_rotate(c, ba, count);
}

void run_pbs_items(lv_ctx* c, const std::vector<PbsItem>& items) {
  const size_t count = items.size();
  if (!count) return;
  std::vector<LinDesc> d(count);
  std::vector<uint32_t> l(count);
  std::vector<BrOut> o(count);
  for (size_t i = 0; i < count; ++i) {
    d[i] = items[i].in;
    l[i] = items[i].lut;
    o[i] = items[i].out;
  }
  LinDesc* dd = c->desc.get(count);
  uint32_t* dl = c->lut_item.get(count);
  BrOut* dout = c->br_out.get(count);
  LV_CUDA(cudaMemcpyAsync(dd, d.data(), count * sizeof(LinDesc), cudaMemcpyHostToDevice, c->stream));
  LV_CUDA(cudaMemcpyAsync(dl, l.data(), count * 4, cudaMemcpyHostToDevice, c->stream));
  LV_CUDA(cudaMemcpyAsync(dout, o.data(), count * sizeof(BrOut), cudaMemcpyHostToDevice, c->stream));
  launch_pbs_dev(c, dd, dl, dout, (uint32_t)count);
  LV_CUDA(cudaStreamSynchronize(c->stream));
}

void launch_linear_dev(lv_ctx* c, const LinOut* d_ops, uint32_t count) {
  if (!count) return;
  for (uint32_t off = 0; off < count; off += 65535u) {
    const uint32_t cnt = std::min<uint32_t>(count - off, 65535u);
    LinArgs la{d_ops + off, c->d_pool, kBigStride, cnt};
    linear_kernel<<<dim3(2, cnt), 1024, 0, c->stream>>>(la);
  }
  LV_CUDA(cudaGetLastError());
}

void run_linear(lv_ctx* c, const std::vector<LinOut>& ops) {
  if (ops.empty()) return;
  LinOut* d = c->lin_ops.get(ops.size());
  LV_CUDA(cudaMemcpyAsync(d, ops.data(), ops.size() * sizeof(LinOut), cudaMemcpyHostToDevice,
                          c->stream));
  launch_linear_dev(c, d, (uint32_t)ops.size());
  LV_CUDA(cudaStreamSynchronize(c->stream));
}

static LinDesc single(uint32_t slot, int32_t coef = 1, int32_t body = 0) {
  LinDesc d{};
  d.slot[0] = slot;
  d.coef[0] = coef;
  d.nterms = 1;
  d.body_const = body;
  return d;
}

static void check_plaintext(int v) {  // backend.cpp:17-21
  if (v < 0 || v >= 32)
    throw Error(LV_ERR_OUT_OF_RANGE, "plaintext outside [0,32): " + std::to_string(v));
}

static void encrypt_into(lv_ctx* c, const int32_t* values, const std::vector<lv_ct>& slots,
                         bool trivial) {
  const size_t count = slots.size();
  if (!count) return;
  uint32_t* ds = c->u32a.get(count);
  int32_t* dv = c->i32a.get(count);
  LV_CUDA(cudaMemcpyAsync(ds, slots.data(), count * 4, cudaMemcpyHostToDevice, c->stream));
  LV_CUDA(cudaMemcpyAsync(dv, values, count * 4, cudaMemcpyHostToDevice, c->stream));
  EncArgs ea{c->d_pool, kBigStride, ds, dv, c->d_sk_glwe, c->seed, c->enc_counter,
             c->p.glwe_noise_log2, trivial ? 1 : 0};
  encrypt_kernel<<<(uint32_t)count, 256, 0, c->stream>>>(ea);
  LV_CUDA(cudaGetLastError());
  LV_CUDA(cudaStreamSynchronize(c->stream));
  if (!trivial) c->enc_counter += count;
}

static void upload_rows(lv_ctx* c, const uint64_t* host, const std::vector<lv_ct>& slots) {
  // contiguous runs of slots become one 2D copy each
  size_t i = 0;
  while (i < slots.size()) {
    size_t j = i + 1;
    while (j < slots.size() && slots[j] == slots[j - 1] + 1) ++j;
    LV_CUDA(cudaMemcpy2DAsync(c->d_pool + (size_t)slots[i] * kBigStride, kBigStride * 8,
                              host + i * (kBig + 1), (kBig + 1) * 8, (kBig + 1) * 8, j - i,
                              cudaMemcpyHostToDevice, c->stream));
    i = j;
  }
}

static void download_rows_on(lv_ctx* c, cudaStream_t st, const std::vector<lv_ct>& slots,
                             uint64_t* host) {
  size_t i = 0;
  while (i < slots.size()) {
    size_t j = i + 1;
    while (j < slots.size() && slots[j] == slots[j - 1] + 1) ++j;
    LV_CUDA(cudaMemcpy2DAsync(host + i * (kBig + 1), (kBig + 1) * 8,
                              c->d_pool + (size_t)slots[i] * kBigStride, kBigStride * 8,
                              (kBig + 1) * 8, j - i, cudaMemcpyDeviceToHost, st));
    i = j;
  }
}
static void download_rows(lv_ctx* c, const std::vector<lv_ct>& slots, uint64_t* host) {
  download_rows_on(c, c->stream, slots, host);
}

static void need_secret(const lv_ctx* c) {
  if (!c->d_sk_glwe)
    throw Error(LV_ERR_INVALID_PARAMS,
                "evaluation-only context (lv_ctx_create_eval) holds no secret key");
}

static std::vector<uint64_t> phases(lv_ctx* c, const lv_ct* cts, size_t count) {
  need_secret(c);
  std::vector<uint64_t> ph(count);
  if (!count) return ph;
  uint32_t* ds = c->u32a.get(count);
  uint64_t* dp = c->u64a.get(count);
  LV_CUDA(cudaMemcpyAsync(ds, cts, count * 4, cudaMemcpyHostToDevice, c->stream));
  PhaseArgs pa{c->d_pool, kBigStride, ds, c->d_sk_glwe, dp};
  phase_kernel<<<(uint32_t)count, 256, 0, c->stream>>>(pa);
  LV_CUDA(cudaGetLastError());
  LV_CUDA(cudaMemcpyAsync(ph.data(), dp, count * 8, cudaMemcpyDeviceToHost, c->stream));
  LV_CUDA(cudaStreamSynchronize(c->stream));
  return ph;
}

static int32_t decode(uint64_t ph) { return (int32_t)(((ph + (kDelta >> 1)) >> 59) & 31); }

// Budget check of SimBackend::pbs (backend.cpp:62-67).
static void check_budget(lv_ctx* c, const lv_ct* in, size_t count) {
  for (size_t i = 0; i < count; ++i) {
    const int64_t v = c->ledgers[in[i]].variance();
    if ((double)v > c->p.max_variance_budget)
      throw Error(LV_ERR_NOISE_BUDGET, "bootstrap input variance " + std::to_string(v) +
                                           " exceeds budget " +
                                           std::to_string(c->p.max_variance_budget));
  }
}

static void pbs_batch(lv_ctx* c, const lv_ct* in, const uint32_t* luts, size_t count, lv_ct* out) {
  check_handles(c, in, count);
  for (size_t i = 0; i < count; ++i)
    if (luts[i] >= c->luts.size()) throw Error(LV_ERR_INVALID_PARAMS, "unknown lut id");
  check_budget(c, in, count);
  std::vector<lv_ct> dst = pool_alloc(c, count);
  std::vector<PbsItem> items(count);
  for (size_t i = 0; i < count; ++i) {
    items[i].in = single(in[i]);
    items[i].lut = luts[i];
    items[i].out = BrOut{0, dst[i], kNoSlot, kNoSlot, kNoSlot, 0};
  }
  run_pbs_items(c, items);
  for (size_t i = 0; i < count; ++i) {
    c->ledgers[dst[i]] = NoiseLedger::fresh(c->next_source++);
    out[i] = dst[i];
  }
  c->pbs_count += count;
}

static void build_tables(lv_ctx* c) {
  const long double PI = 3.141592653589793238462643383279502884L;
  // Linzer-Feig twiddles (c, t) = (cos, tan) rounded from long double
  // (oracle build_tables): forward level s block b at fwd_base(s) + b (b/2 at
  // the sibling levels) is
  // zeta^e, e = (kM >> (s+1)) (1 - 4 brv_s(b)) mod 2N, zeta = exp(i pi / N);
  // inverse conj(W^k) = exp(2 pi i k / kM) at kM + k, k < kM/2.
  std::vector<double2> tw(kTwEntries), twist(128 + kM);
  for (uint32_t s = 0; s < kLogM; ++s)
    for (uint32_t b = 0; b < (1u << s); ++b) {
      uint32_t r = 0;  // brv_s(b)
      for (uint32_t q = 0; q < s; ++q) r |= ((b >> q) & 1u) << (s - 1 - q);
      const int64_t e = ((int64_t)(kM >> (s + 1)) * (1 - 4 * (int64_t)r)) % (int64_t)(2 * kN);
      const long double ang = PI * (long double)(e < 0 ? e + 2 * kN : e) / (long double)kN;
      if (fwd_sibling_level((int)s) && (b & 1)) continue;  // odd blocks: -i x the even sibling
      tw[fwd_base((int)s) + (fwd_sibling_level((int)s) ? b >> 1 : b)] =
          make_double2((double)cosl(ang), (double)tanl(ang));
    }
  for (uint32_t k = 0; k < kM / 2; ++k) {
    const long double ang = 2.0L * PI * (long double)k / (long double)kM;
    tw[kM + k] = make_double2((double)cosl(ang), (double)tanl(ang));
  }
  set_fwd_consts(tw.data());  // levels 0-2 (entries 0..6) as constant operands
  // twist zeta^j = fine[j & 127] * coarse[j >> 7] (oracle build_tables)
  for (uint32_t j = 0; j < 128; ++j) {
    const long double ang = PI * (long double)j / (long double)kN;
    twist[j] = make_double2((double)cosl(ang), (double)sinl(ang));
  }
  double2 coarse[8];
  for (uint32_t k = 0; k < 8; ++k) {
    const long double ang = PI * (long double)(k * 128) / (long double)kN;
    coarse[k] = make_double2((double)cosl(ang), (double)sinl(ang));
  }
  set_twist_coarse(coarse);
  // [128 + x]: the full twist zeta^x = fine[x & 127] * coarse[x >> 7], formed
  // with the kernels' cmul (fma(a.x, b.x, -(a.y b.y)), fma(a.x, b.y, a.y b.x)),
  // so a loaded factor equals a formed one bit for bit
  for (uint32_t j = 0; j < kM; ++j) {
    const double2 f = twist[j & 127], k = coarse[j >> 7];
    twist[128 + j] = (j >> 7) == 0 ? f
                                   : make_double2(std::fma(f.x, k.x, -(f.y * k.y)),
                                                  std::fma(f.x, k.y, f.y * k.x));
  }
  LV_CUDA(cudaMalloc(&c->d_tw, tw.size() * sizeof(double2)));
  LV_CUDA(cudaMalloc(&c->d_twist, twist.size() * sizeof(double2)));
  LV_CUDA(cudaMemcpy(c->d_tw, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice));
  LV_CUDA(cudaMemcpy(c->d_twist, twist.data(), twist.size() * sizeof(double2), cudaMemcpyHostToDevice));
}

static size_t bsk_words(uint32_t n) { return (size_t)n * kRows * (kK + 1) * kN; }
static size_t ksk_words(uint32_t n) { return (size_t)kBig * kKsLevel * (n + 1); }

// Everything the key switch derives from the KSK (c->d_ksk): the bias row
// and the byte limbs of the tensor-core GEMM, with its TMA tensor map.
static void derive_ksk(lv_ctx* c) {
  const uint32_t n = c->p.n;
  LV_CUDA(cudaMalloc(&c->d_ksk_bias, (size_t)(n + 1) * sizeof(uint64_t)));
  ksk_bias_kernel<<<(n + 1 + 127) / 128, 128, 0, c->stream>>>(c->d_ksk, n, c->d_ksk_bias);
  LV_CUDA(cudaGetLastError());
  const uint32_t rows = ks_tc_ntiles(n) * 32 * 8;  // limb rows, zero-padded past n
  LV_CUDA(cudaMalloc(&c->d_ksk_bt, (size_t)rows * kBig * kKsLevel));
  ksk_limbs_kernel<<<dim3((kBig * kKsLevel + 255) / 256, rows / 8), 256, 0, c->stream>>>(
      c->d_ksk, n, c->d_ksk_bt);
  LV_CUDA(cudaGetLastError());
  c->ks_tma = !std::getenv("LVB_KS_NO_TMA") && make_ks_tensor_map(&c->ksk_map, c->d_ksk_bt, rows, 256);
}

// Standard-domain BSK (device, [i][row][poly][N] u64) generated from the seed.
static void gen_bsk(lv_ctx* c, uint64_t* d_bsk) {
  keygen_bsk_kernel<<<c->p.n * kRows, 256, 0, c->stream>>>(c->seed, c->p.glwe_noise_log2,
                                                            c->d_sk_small, c->d_sk_glwe, d_bsk);
  LV_CUDA(cudaGetLastError());
}

// The resident Fourier BSK (c->d_bskf) from a standard-domain BSK.
static void derive_bsk(lv_ctx* c, const uint64_t* d_bsk) {
  const uint32_t n = c->p.n;
  const bool exact = c->p.exact_mask_product == 1;
  const uint32_t nouts = exact ? 3 : 2;  // spectra per GGSW row: [mask, body] or [H, Lo, body]
  LV_CUDA(cudaMalloc(&c->d_bskf, (size_t)n * 8 * kRows * nouts * 128 * sizeof(double2)));
  // double-double twiddle / twist tables for the BSK transform (oracle
  // build_tables: hi = rn(v), lo = rn(v - hi) from long double)
  std::vector<double4> tw_dd(kM / 2), twist_dd(kM);
  {
    const long double PI = 3.141592653589793238462643383279502884L;
    auto split = [](long double cr, long double ci) {
      const double rh = (double)cr, ih = (double)ci;
      return make_double4(rh, (double)(cr - (long double)rh), ih, (double)(ci - (long double)ih));
    };
    for (uint32_t t = 0; t < kM / 2; ++t) {
      const long double ang = 2.0L * PI * (long double)t / (long double)kM;
      tw_dd[t] = split(cosl(ang), -sinl(ang));
    }
    for (uint32_t j = 0; j < kM; ++j) {
      const long double ang = PI * (long double)j / (long double)kN;
      twist_dd[j] = split(cosl(ang), sinl(ang));
    }
  }
  DevTemp<double4> d_tw_dd(tw_dd.size()), d_twist_dd(twist_dd.size());
  LV_CUDA(cudaMemcpy(d_tw_dd.p, tw_dd.data(), tw_dd.size() * sizeof(double4), cudaMemcpyHostToDevice));
  LV_CUDA(cudaMemcpy(d_twist_dd.p, twist_dd.data(), twist_dd.size() * sizeof(double4),
                     cudaMemcpyHostToDevice));
  DevTemp<uint64_t> d_split(exact ? (size_t)n * kRows * 3 * kN : 0);
  if (exact) {
    bsk_split_kernel<<<n * kRows, 256, 0, c->stream>>>(d_bsk, d_split.p);
    LV_CUDA(cudaGetLastError());
  }
  if (c->p.exact_mask_product == 2)  // the reference's algorithm: plain f64 BSK transform
    bsk_fourier_f64_kernel<<<n * kRows * nouts, 128, 0, c->stream>>>(d_bsk, nouts, c->d_tw, c->d_bskf);
  else
    bsk_fourier_kernel<<<n * kRows * nouts, 512, 0, c->stream>>>(exact ? d_split.p : d_bsk, nouts,
                                                                  d_tw_dd.p, d_twist_dd.p, c->d_bskf);
  LV_CUDA(cudaGetLastError());
  LV_CUDA(cudaStreamSynchronize(c->stream));
}

// Secret keys, KSK and BSK from the seed (a client context).
static void keygen(lv_ctx* c) {
  const uint32_t n = c->p.n;
  LV_CUDA(cudaMalloc(&c->d_sk_small, n));
  LV_CUDA(cudaMalloc(&c->d_sk_glwe, kBig));
  keygen_secret_kernel<<<(std::max(n, kBig) + 255) / 256, 256, 0, c->stream>>>(c->seed, n, c->d_sk_small,
                                                                              c->d_sk_glwe);
  LV_CUDA(cudaGetLastError());
  LV_CUDA(cudaMalloc(&c->d_ksk, ksk_words(n) * sizeof(uint64_t)));
  keygen_ksk_kernel<<<kBig * kKsLevel, 256, 0, c->stream>>>(c->seed, n, c->p.lwe_noise_log2,
                                                            c->d_sk_small, c->d_sk_glwe, c->d_ksk);
  LV_CUDA(cudaGetLastError());
  derive_ksk(c);
  DevTemp<uint64_t> d_bsk(bsk_words(n));
  gen_bsk(c, d_bsk.p);
  derive_bsk(c, d_bsk.p);
}

// Evaluation keys received from a client (a server context: no secret key).
static void load_eval_keys(lv_ctx* c, const uint64_t* bsk, const uint64_t* ksk) {
  const uint32_t n = c->p.n;
  LV_CUDA(cudaMalloc(&c->d_ksk, ksk_words(n) * sizeof(uint64_t)));
  LV_CUDA(cudaMemcpy(c->d_ksk, ksk, ksk_words(n) * sizeof(uint64_t), cudaMemcpyHostToDevice));
  derive_ksk(c);
  DevTemp<uint64_t> d_bsk(bsk_words(n));
  LV_CUDA(cudaMemcpy(d_bsk.p, bsk, bsk_words(n) * sizeof(uint64_t), cudaMemcpyHostToDevice));
  derive_bsk(c, d_bsk.p);
}

std::array<int32_t, 16> eq_lut_entries(int scale) {  // equality.cpp:31-36
  std::array<int32_t, 16> e{};
  e[0] = scale;
  return e;
}

// build_min_lut (kernel.cpp:28-72): key -> 1 + min(-eq, dv, dh) over the 18
// packed keys; entries 0..15 are the table, keys 16/17 must be the forced
// negacyclic images (checked: PackingViolation).
std::array<int32_t, 16> min_lut_entries(bool negated) {
  std::array<int32_t, 18> values{};
  for (int key = 0; key < 18; ++key) {
    const int eq = key >= 9 ? 1 : 0;
    const int r = key % 9;
    const int dv_part = r % 3, dh = r / 3 - 1;
    const int dv = negated ? 1 - dv_part : dv_part - 1;
    values[key] = 1 + std::min({-eq, dv, dh});
  }
  std::array<int32_t, 16> e{};
  for (int i = 0; i < 16; ++i) e[i] = ((values[i] % 32) + 32) % 32;
  for (int k = 16; k < 18; ++k) {
    const int img = (32 - e[k - 16]) % 32;
    if (img != ((values[k] % 32) + 32) % 32) throw Error(LV_ERR_PACKING, "min table packing violated");
  }
  return e;
}

}  // namespace lvb

using namespace lvb;

// ====================================================================== C ABI
extern "C" {

void lv_default_params(lv_params* p) {
  p->n = 880;
  p->N = kN;
  p->k = kK;
  p->pbs_base_log = kPbsBaseLog;
  p->pbs_level = kPbsLevel;
  p->ks_base_log = kKsBaseLog;
  p->ks_level = kKsLevel;
  p->lwe_noise_log2 = 44;
  p->glwe_noise_log2 = 17;
  p->max_variance_budget = 4000.0;
  p->exact_mask_product = 0;
  p->device = -1;
}

const char* lv_last_error(void) { return g_last_error.c_str(); }
int lv_abi_version(void) { return LV_ABI_VERSION; }

int lv_lut_table(int32_t which, int32_t* out16) {
  return guard([&] {
    std::array<int32_t, 16> e{};
    switch (which) {
      case LV_TABLE_MINLUT_ORIGINAL: e = min_lut_entries(false); break;
      case LV_TABLE_MINLUT_NEGATED: e = min_lut_entries(true); break;
      case LV_TABLE_EQLUT: e = eq_lut_entries(1); break;
      case LV_TABLE_EQLUT9: e = eq_lut_entries(9); break;
      default: throw Error(LV_ERR_INVALID_PARAMS, "unknown table");
    }
    std::copy(e.begin(), e.end(), out16);
  });
}

// Key-set fingerprint from PUBLIC material only: FNV-1a over the
// parameter set and the first 8192 words of the key-switching key (its
// masks and bodies are public; the generating seed is never exported or
// serialised). Client and server contexts of one key set agree on it.
static uint64_t key_fingerprint(lv_ctx* c) {
  constexpr size_t kWords = 8192;
  std::vector<uint64_t> h(std::min<size_t>(kWords, ksk_words(c->p.n)));
  LV_CUDA(cudaMemcpy(h.data(), c->d_ksk, h.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  uint64_t f = 0xcbf29ce484222325ull;
  auto mix = [&](uint64_t v) {
    for (int b = 0; b < 8; ++b) {
      f ^= (v >> (8 * b)) & 0xff;
      f *= 0x100000001b3ull;
    }
  };
  mix(c->p.n);
  mix(c->p.N);
  mix(c->p.k);
  mix(c->p.exact_mask_product);
  for (uint64_t v : h) mix(v);
  return f;
}

// Carveout preferences (percent of the maximum shared memory; -1 = driver
// default), measured in profiles/r02_lf_variants.txt.
constexpr int kPairCarveoutPct = -1;
constexpr int kBrCarveoutPct = -1;

static int create_ctx(const lv_params* params, uint64_t seed, const uint64_t* bsk,
                      const uint64_t* ksk, uint64_t key_id, lv_ctx** out) {
  return guard([&] {
    lv_params p;
    if (params)
      p = *params;
    else
      lv_default_params(&p);
    if (p.N != kN || p.k != kK || p.pbs_base_log != kPbsBaseLog || p.pbs_level != kPbsLevel ||
        p.ks_base_log != kKsBaseLog || p.ks_level != kKsLevel)
      throw Error(LV_ERR_INVALID_PARAMS, "parameter set does not match the compiled kernels");
    if (p.n < 1 || p.n > kMaxLweN) throw Error(LV_ERR_INVALID_PARAMS, "n out of range");
    if (p.lwe_noise_log2 < 1 || p.lwe_noise_log2 > 62 || p.glwe_noise_log2 < 1 ||
        p.glwe_noise_log2 > 62)
      throw Error(LV_ERR_INVALID_PARAMS, "noise bounds out of range (TUniform 2^1 .. 2^62)");
    if (p.exact_mask_product > 2)
      throw Error(LV_ERR_INVALID_PARAMS, "exact_mask_product must be 0, 1 or 2");
    if (p.max_variance_budget < 1.0)  // backend.hpp:85-88
      throw Error(LV_ERR_INVALID_PARAMS, "noise budget must be at least 1");
    int ndev = 0;
    LV_CUDA(cudaGetDeviceCount(&ndev));
    if (ndev < 1) throw Error(LV_ERR_CUDA, "no CUDA device");
    if (p.device >= ndev) throw Error(LV_ERR_INVALID_PARAMS, "device index out of range");
    if (p.device >= 0) LV_CUDA(cudaSetDevice(p.device));
    lv_ctx* c = new lv_ctx();
    try {
      c->p = p;
      c->seed = seed;
      LV_CUDA(cudaGetDevice(&c->device));
      LV_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      LV_CUDA(cudaStreamCreateWithFlags(&c->copy_out, cudaStreamNonBlocking));
      // Function attributes are process-wide, not per context: allow the
      // dynamic shared memory of the largest supported n, so a context with
      // a smaller n cannot shrink the limit under another context's launches
      // (occupancy still follows each launch's actual request).
      LV_CUDA(cudaFuncSetAttribute(blind_rotate_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)blind_rotate_smem_bytes(kMaxLweN, false)));
      LV_CUDA(cudaFuncSetAttribute(blind_rotate_exact_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)blind_rotate_smem_bytes(kMaxLweN, true)));
      LV_CUDA(cudaFuncSetAttribute(ks_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)ks_tc_smem_bytes()));
      LV_CUDA(cudaFuncSetAttribute(ks_mma_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)ks_tma_smem_bytes()));
      LV_CUDA(cudaFuncSetAttribute(blind_rotate_pair_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)blind_rotate_pair_smem_bytes(kMaxLweN)));
      LV_CUDA(cudaFuncSetAttribute(blind_rotate_pair_exact_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)blind_rotate_pair_smem_bytes(kMaxLweN)));
      // Shared-memory carveout preference (percent of the maximum): the rest
      // of the 256 KB array is L1, which must keep the FFT twiddle tables
      // (~19 KB touched) resident. -1 leaves the choice to the driver.
      auto carveout = [](const char* env, int dflt) {
        const char* e = std::getenv(env);
        return e ? std::atoi(e) : dflt;
      };
      const int pair_pct = carveout("LVB_PAIR_CARVEOUT", kPairCarveoutPct);
      if (pair_pct >= 0) {
        LV_CUDA(cudaFuncSetAttribute(blind_rotate_pair_kernel,
                                     cudaFuncAttributePreferredSharedMemoryCarveout, pair_pct));
        LV_CUDA(cudaFuncSetAttribute(blind_rotate_pair_exact_kernel,
                                     cudaFuncAttributePreferredSharedMemoryCarveout, pair_pct));
      }
      const int br_pct = carveout("LVB_BR_CARVEOUT", kBrCarveoutPct);
      if (br_pct >= 0)
        LV_CUDA(cudaFuncSetAttribute(blind_rotate_kernel,
                                     cudaFuncAttributePreferredSharedMemoryCarveout, br_pct));
      {
        int sms = 148;
        LV_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
        c->br_pair_max = (uint32_t)sms;
        if (const char* e = std::getenv("LVB_BR_PAIR_MAX"))
          c->br_pair_max = (uint32_t)std::strtoul(e, nullptr, 10);
        int per_sm = 1;
        if (p.exact_mask_product == 1)
          LV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
              &per_sm, blind_rotate_exact_kernel, 128, blind_rotate_smem_bytes(p.n, true)));
        else
          LV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
              &per_sm, blind_rotate_kernel, 128, blind_rotate_smem_bytes(p.n, false)));
        c->br_slots = (uint32_t)(sms * std::max(per_sm, 1));
      }
      build_tables(c);
      if (bsk)
        load_eval_keys(c, bsk, ksk);
      else
        keygen(c);
      c->key_id = key_fingerprint(c);
      // a server context checks the client's announced fingerprint
      if (bsk && key_id != 0 && key_id != c->key_id)
        throw Error(LV_ERR_INVALID_PARAMS, "evaluation keys do not match the announced key id");
      c->min_lut[0] = lut_id(c, min_lut_entries(false));
      c->min_lut[1] = lut_id(c, min_lut_entries(true));
      std::array<int32_t, 16> id{};
      for (int i = 0; i < 16; ++i) id[i] = i;
      c->identity_lut = lut_id(c, id);
      pool_grow(c, 1024);
    } catch (...) {
      lv_ctx_destroy(c);
      throw;
    }
    *out = c;
  });
}

int lv_ctx_create(const lv_params* params, uint64_t seed, lv_ctx** out) {
  return create_ctx(params, seed, nullptr, nullptr, 0, out);
}

int lv_ctx_create_eval(const lv_params* params, const uint64_t* bsk, const uint64_t* ksk,
                       uint64_t key_id, lv_ctx** out) {
  if (!bsk || !ksk)
    return guard([] { throw Error(LV_ERR_INVALID_PARAMS, "evaluation keys missing"); });
  return create_ctx(params, 0, bsk, ksk, key_id, out);
}

int lv_keys_size(const lv_params* params, uint64_t* bsk_count, uint64_t* ksk_count) {
  return guard([&] {
    if (params->n < 1 || params->n > kMaxLweN) throw Error(LV_ERR_INVALID_PARAMS, "n out of range");
    *bsk_count = bsk_words(params->n);
    *ksk_count = ksk_words(params->n);
  });
}

int lv_keys_export(lv_ctx* c, uint64_t* bsk, uint64_t* ksk, uint64_t* key_id) {
  return guard([&] {
    CtxLock lk(c);
    need_secret(c);
    const uint32_t n = c->p.n;
    if (ksk) LV_CUDA(cudaMemcpy(ksk, c->d_ksk, ksk_words(n) * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    if (bsk) {  // regenerated from the seed: the context keeps only the Fourier form
      DevTemp<uint64_t> d_bsk(bsk_words(n));
      gen_bsk(c, d_bsk.p);
      LV_CUDA(cudaMemcpyAsync(bsk, d_bsk.p, bsk_words(n) * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                              c->stream));
      LV_CUDA(cudaStreamSynchronize(c->stream));
    }
    if (key_id) *key_id = c->key_id;
  });
}

int lv_ctx_key_id(lv_ctx* c, uint64_t* key_id) {
  return guard([&] { *key_id = c->key_id; });
}

void lv_ctx_destroy(lv_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (void* p : {(void*)c->d_sk_small, (void*)c->d_sk_glwe, (void*)c->d_ksk, (void*)c->d_ksk_bias, (void*)c->d_bskf,
                  (void*)c->d_tw, (void*)c->d_twist, (void*)c->d_tp, (void*)c->d_pool})
    if (p) cudaFree(p);
  c->ms.release();
  c->desc.release();
  c->lut_item.release();
  c->br_out.release();
  c->lin_ops.release();
  c->u32a.release();
  c->u32b.release();
  c->i32a.release();
  c->ks_digits.release();
  c->ks_body.release();
  if (c->d_ksk_bt) cudaFree(c->d_ksk_bt);
  c->u64a.release();
  c->u64b.release();
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->copy_out) cudaStreamDestroy(c->copy_out);
  delete c;
}

int lv_get_params(lv_ctx* c, lv_params* out) {
  return guard([&] { *out = c->p; });
}

int lv_encrypt(lv_ctx* c, const int32_t* values, size_t count, lv_ct* out) {
  return guard([&] {
    CtxLock lk(c);
    need_secret(c);
    for (size_t i = 0; i < count; ++i) check_plaintext(values[i]);
    std::vector<lv_ct> s = pool_alloc(c, count);
    encrypt_into(c, values, s, false);
    for (size_t i = 0; i < count; ++i) {
      c->ledgers[s[i]] = NoiseLedger::fresh(c->next_source++);
      out[i] = s[i];
    }
  });
}

int lv_trivial(lv_ctx* c, const int32_t* values, size_t count, lv_ct* out) {
  return guard([&] {
    CtxLock lk(c);
    for (size_t i = 0; i < count; ++i) check_plaintext(values[i]);
    std::vector<lv_ct> s = pool_alloc(c, count);
    encrypt_into(c, values, s, true);
    for (size_t i = 0; i < count; ++i) out[i] = s[i];
  });
}

int lv_decrypt(lv_ctx* c, const lv_ct* cts, size_t count, int32_t* out) {
  return guard([&] {
    CtxLock lk(c);
    check_handles(c, cts, count);
    std::vector<uint64_t> ph = phases(c, cts, count);
    for (size_t i = 0; i < count; ++i) out[i] = decode(ph[i]);
  });
}

int lv_phase(lv_ctx* c, const lv_ct* cts, size_t count, uint64_t* out) {
  return guard([&] {
    CtxLock lk(c);
    check_handles(c, cts, count);
    std::vector<uint64_t> ph = phases(c, cts, count);
    std::memcpy(out, ph.data(), count * 8);
  });
}

static int linear2(lv_ctx* c, const lv_ct* a, const lv_ct* b, size_t count, lv_ct* out, int sign) {
  return guard([&] {
    CtxLock lk(c);
    check_handles(c, a, count);
    check_handles(c, b, count);
    std::vector<lv_ct> dst = pool_alloc(c, count);
    std::vector<LinOut> ops(count);
    for (size_t i = 0; i < count; ++i) {
      LinOut o{};
      o.nout = 1;
      o.out_slot[0] = dst[i];
      o.d[0].slot[0] = a[i];
      o.d[0].coef[0] = 1;
      o.d[0].slot[1] = b[i];
      o.d[0].coef[1] = sign;
      o.d[0].nterms = 2;
      ops[i] = o;
    }
    run_linear(c, ops);
    for (size_t i = 0; i < count; ++i) {
      NoiseLedger l = c->ledgers[a[i]];
      l.add_scaled(c->ledgers[b[i]], sign);
      c->ledgers[dst[i]] = std::move(l);
      out[i] = dst[i];
    }
    c->linear_count += count;
  });
}

int lv_add(lv_ctx* c, const lv_ct* a, const lv_ct* b, size_t count, lv_ct* out) {
  return linear2(c, a, b, count, out, 1);
}
int lv_sub(lv_ctx* c, const lv_ct* a, const lv_ct* b, size_t count, lv_ct* out) {
  return linear2(c, a, b, count, out, -1);
}

static int scalar_op(lv_ctx* c, const lv_ct* a, const int32_t* k, size_t count, lv_ct* out, bool mul) {
  return guard([&] {
    CtxLock lk(c);
    check_handles(c, a, count);
    std::vector<lv_ct> dst = pool_alloc(c, count);
    std::vector<LinOut> ops(count);
    for (size_t i = 0; i < count; ++i) {
      LinOut o{};
      o.nout = 1;
      o.out_slot[0] = dst[i];
      o.d[0] = single(a[i], mul ? k[i] : 1, mul ? 0 : k[i]);
      ops[i] = o;
    }
    run_linear(c, ops);
    for (size_t i = 0; i < count; ++i) {
      NoiseLedger l = c->ledgers[a[i]];
      if (mul) l.scale(k[i]);
      c->ledgers[dst[i]] = std::move(l);
      out[i] = dst[i];
    }
    c->linear_count += count;
  });
}

int lv_scalar_mul(lv_ctx* c, const lv_ct* a, const int32_t* k, size_t count, lv_ct* out) {
  return scalar_op(c, a, k, count, out, true);
}
int lv_scalar_add(lv_ctx* c, const lv_ct* a, const int32_t* k, size_t count, lv_ct* out) {
  return scalar_op(c, a, k, count, out, false);
}

int lv_lut_upload(lv_ctx* c, const int32_t entries[16], uint32_t* id) {
  return guard([&] {
    CtxLock lk(c);
    std::array<int32_t, 16> e{};
    std::memcpy(e.data(), entries, sizeof(e));
    *id = lut_id(c, e);
  });
}

int lv_pbs_batch(lv_ctx* c, const lv_ct* in, const uint32_t* luts, size_t count, lv_ct* out) {
  return guard([&] {
    CtxLock lk(c);
    pbs_batch(c, in, luts, count, out);
  });
}

int lv_refresh_batch(lv_ctx* c, const lv_ct* in, size_t count, lv_ct* out) {
  return guard([&] {
    CtxLock lk(c);
    check_handles(c, in, count);
    if (c->d_sk_glwe) {  // backend.cpp:72-80; a server (no secret key) cannot check
      std::vector<uint64_t> ph = phases(c, in, count);
      for (size_t i = 0; i < count; ++i) {
        const int32_t v = decode(ph[i]);
        if (v >= 16)
          throw Error(LV_ERR_VALUE_OUTSIDE_LUT_HALF,
                      "refresh needs a value in [0,16), got " + std::to_string(v));
      }
    }
    std::vector<uint32_t> luts(count, c->identity_lut);
    pbs_batch(c, in, luts.data(), count, out);
    c->refresh_count += count;
  });
}

int lv_predict_variance(lv_ctx* c, const lv_ct* cts, const int32_t* coeffs, size_t count,
                        int64_t* out) {
  return guard([&] {
    CtxLock lk(c);
    check_handles(c, cts, count);
    NoiseLedger comb;
    for (size_t i = 0; i < count; ++i) comb.add_scaled(c->ledgers[cts[i]], coeffs[i]);
    *out = comb.variance();
  });
}

int lv_ledger_variance(lv_ctx* c, const lv_ct* cts, size_t count, int64_t* out) {
  return guard([&] {
    CtxLock lk(c);
    check_handles(c, cts, count);
    for (size_t i = 0; i < count; ++i) out[i] = c->ledgers[cts[i]].variance();
  });
}

int lv_get_stats(lv_ctx* c, lv_stats* out) {
  return guard([&] {
    out->pbs_count = c->pbs_count.load();
    out->refresh_count = c->refresh_count.load();
    out->linear_op_count = c->linear_count.load();
  });
}

int lv_release(lv_ctx* c, const lv_ct* cts, size_t count) {
  return guard([&] {
    CtxLock lk(c);
    pool_free(c, cts, count);
  });
}

int lv_export(lv_ctx* c, const lv_ct* cts, size_t count, uint64_t* host) {
  return guard([&] {
    CtxLock lk(c);
    check_handles(c, cts, count);
    download_rows(c, std::vector<lv_ct>(cts, cts + count), host);
    LV_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int lv_import(lv_ctx* c, const uint64_t* host, size_t count, lv_ct* out) {
  return guard([&] {
    CtxLock lk(c);
    std::vector<lv_ct> s = pool_alloc(c, count);
    upload_rows(c, host, s);
    LV_CUDA(cudaStreamSynchronize(c->stream));
    for (size_t i = 0; i < count; ++i) {
      c->ledgers[s[i]] = NoiseLedger::fresh(c->next_source++);
      out[i] = s[i];
    }
  });
}

// cuStreamWaitValue32 through the runtime's driver entry point (no libcuda
// link dependency); null when the driver does not offer stream memory ops.
using WaitValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static WaitValueFn wait_value_fn() {
  static WaitValueFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (WaitValueFn) nullptr;
    return reinterpret_cast<WaitValueFn>(f);
  }();
  return fn;
}

// Host batch: upload, one key switch + one blind rotation launch (one long
// launch keeps the kernel in its steady state: chunked launches measured
// slower), and downloads that start while the launch is still running —
// the blind rotation counts finished CTAs per chunk of br_slots items
// (BrArgs::done) and the copy stream waits on each chunk's counter
// (cuStreamWaitValue32) before copying its rows back.
int lv_pbs_batch_host(lv_ctx* c, const uint64_t* in, const uint32_t* luts, size_t count,
                      uint64_t* out) {
  return guard([&] {
    CtxLock lk(c);
    for (size_t i = 0; i < count; ++i)
      if (luts[i] >= c->luts.size()) throw Error(LV_ERR_INVALID_PARAMS, "unknown lut id");
    if (!count) return;
    std::vector<lv_ct> s = pool_alloc(c, count);
    upload_rows(c, in, s);
    std::vector<LinDesc> d(count);
    std::vector<BrOut> o(count);
    for (size_t i = 0; i < count; ++i) {
      d[i] = single(s[i]);
      o[i] = BrOut{0, s[i], kNoSlot, kNoSlot, kNoSlot, 0};  // in place: KS reads first
    }
    LinDesc* dd = c->desc.get(count);
    uint32_t* dl = c->lut_item.get(count);
    BrOut* dout = c->br_out.get(count);
    LV_CUDA(cudaMemcpyAsync(dd, d.data(), count * sizeof(LinDesc), cudaMemcpyHostToDevice, c->stream));
    LV_CUDA(cudaMemcpyAsync(dl, luts, count * 4, cudaMemcpyHostToDevice, c->stream));
    LV_CUDA(cudaMemcpyAsync(dout, o.data(), count * sizeof(BrOut), cudaMemcpyHostToDevice, c->stream));
    const WaitValueFn wait = wait_value_fn();
    const size_t chunk = std::max<size_t>(c->br_slots, 1);
    const bool overlap = wait && count > c->br_pair_max && count >= 2 * chunk &&
                         std::getenv("LVB_HOST_NO_OVERLAP") == nullptr;
    if (!overlap) {
      launch_pbs_dev(c, dd, dl, dout, (uint32_t)count);
      download_rows(c, s, out);
      LV_CUDA(cudaStreamSynchronize(c->stream));
    } else {
      const size_t nchunks = (count + chunk - 1) / chunk;
      uint32_t* done = c->u32b.get(nchunks);
      LV_CUDA(cudaMemsetAsync(done, 0, nchunks * 4, c->stream));
      Event zeroed(cudaEventDisableTiming);
      LV_CUDA(cudaEventRecord(zeroed.e, c->stream));
      // the copy stream must not see the previous call's counters
      LV_CUDA(cudaStreamWaitEvent(c->copy_out, zeroed.e, 0));
      launch_pbs_dev(c, dd, dl, dout, (uint32_t)count, nullptr, done, (uint32_t)chunk);
      for (size_t k = 0; k < nchunks; ++k) {
        const size_t off = k * chunk, m = std::min(chunk, count - off);
        if (wait(reinterpret_cast<CUstream>(c->copy_out),
                 reinterpret_cast<CUdeviceptr>(done + k), (cuuint32_t)m,
                 CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
          throw Error(LV_ERR_CUDA, "cuStreamWaitValue32 failed");
        std::vector<lv_ct> sk(s.begin() + off, s.begin() + off + m);
        download_rows_on(c, c->copy_out, sk, out + off * (kBig + 1));
      }
      LV_CUDA(cudaStreamSynchronize(c->copy_out));
      LV_CUDA(cudaStreamSynchronize(c->stream));
    }
    pool_free(c, s.data(), count);
    c->pbs_count += count;
  });
}

// ------------------------------------------------------------- debug / parity
int lv_debug_keys(lv_ctx* c, uint8_t* sk_small, uint8_t* sk_glwe, uint64_t* ksk, double* bskf_nat) {
  return guard([&] {
    CtxLock lk(c);
    if (sk_small || sk_glwe) need_secret(c);
    const uint32_t n = c->p.n;
    if (sk_small) LV_CUDA(cudaMemcpy(sk_small, c->d_sk_small, n, cudaMemcpyDeviceToHost));
    if (sk_glwe) LV_CUDA(cudaMemcpy(sk_glwe, c->d_sk_glwe, kBig, cudaMemcpyDeviceToHost));
    if (ksk)
      LV_CUDA(cudaMemcpy(ksk, c->d_ksk, (size_t)kBig * kKsLevel * (n + 1) * 8, cudaMemcpyDeviceToHost));
    if (bskf_nat && c->p.exact_mask_product == 1)
      throw Error(LV_ERR_INVALID_PARAMS, "debug_keys: exact_mask_product keys use the split layout");
    if (bskf_nat) {
      std::vector<double2> raw((size_t)n * 32 * 128);
      LV_CUDA(cudaMemcpy(raw.data(), c->d_bskf, raw.size() * sizeof(double2), cudaMemcpyDeviceToHost));
      // device [i][q*4 + r*2 + o][t] -> oracle [(i*rows + r)*(k+1) + o][f = spec_pos(t, q)] (re, im)
      for (size_t i = 0; i < n; ++i)
        for (uint32_t q = 0; q < 8; ++q)
          for (uint32_t r = 0; r < 2; ++r)
            for (uint32_t o = 0; o < 2; ++o)
              for (uint32_t t = 0; t < 128; ++t) {
                const double2 v = raw[i * 4096 + (q * 4 + r * 2 + o) * 128 + t];
                const size_t base = ((i * kRows + r) * (kK + 1) + o) * 2 * kM + 2 * spec_pos(t, q);
                bskf_nat[base] = v.x * 1024.0;  // undo the exact 2^-10 pre-scaling
                bskf_nat[base + 1] = v.y * 1024.0;
              }
    }
  });
}

int lv_debug_keyswitch(lv_ctx* c, const uint64_t* in, size_t count, uint64_t* out_small) {
  return guard([&] {
    CtxLock lk(c);
    std::vector<lv_ct> s = pool_alloc(c, count);
    upload_rows(c, in, s);
    std::vector<LinDesc> d(count);
    for (size_t i = 0; i < count; ++i) d[i] = single(s[i]);
    LinDesc* dd = c->desc.get(count);
    LV_CUDA(cudaMemcpyAsync(dd, d.data(), count * sizeof(LinDesc), cudaMemcpyHostToDevice, c->stream));
    const uint32_t row = c->p.n + 1, stride = ms_stride(c);
    uint64_t* dsmall = c->u64b.get(count * row);
    uint16_t* dms = c->ms.get(count * stride);
    launch_keyswitch(c, dd, (uint32_t)count, dms, dsmall);
    LV_CUDA(cudaMemcpyAsync(out_small, dsmall, count * row * 8, cudaMemcpyDeviceToHost, c->stream));
    LV_CUDA(cudaStreamSynchronize(c->stream));
    pool_free(c, s.data(), count);
  });
}

int lv_debug_blind_rotate(lv_ctx* c, const uint32_t* ms, const uint32_t* luts, size_t count,
                          uint64_t* out, uint64_t* glwe_out) {
  return guard([&] {
    CtxLock lk(c);
    const uint32_t row = c->p.n + 1, stride = ms_stride(c);
    std::vector<uint16_t> h((size_t)count * stride, 0);
    for (size_t i = 0; i < count; ++i)
      for (uint32_t j = 0; j < row; ++j) h[i * stride + j] = (uint16_t)ms[i * row + j];
    std::vector<lv_ct> s = pool_alloc(c, count);
    std::vector<BrOut> o(count);
    for (size_t i = 0; i < count; ++i) o[i] = BrOut{0, s[i], kNoSlot, kNoSlot, kNoSlot, 0};
    uint16_t* dms = c->ms.get(count * stride);
    uint32_t* dl = c->lut_item.get(count);
    BrOut* dout = c->br_out.get(count);
    LV_CUDA(cudaMemcpyAsync(dms, h.data(), h.size() * 2, cudaMemcpyHostToDevice, c->stream));
    LV_CUDA(cudaMemcpyAsync(dl, luts, count * 4, cudaMemcpyHostToDevice, c->stream));
    LV_CUDA(cudaMemcpyAsync(dout, o.data(), count * sizeof(BrOut), cudaMemcpyHostToDevice, c->stream));
    BrArgs ba{dms, stride, dl, c->d_tp, c->d_bskf, c->d_tw, c->d_twist, c->p.n,
              c->d_pool, kBigStride, dout};
    uint64_t* dglwe = nullptr;
    if (glwe_out) {
      LV_CUDA(cudaMalloc(&dglwe, count * 2 * kN * sizeof(uint64_t)));
      ba.glwe_out = dglwe;
    }
    launch_blind_rotate(c, ba, (uint32_t)count);
    download_rows(c, s, out);
    if (dglwe)
      LV_CUDA(cudaMemcpyAsync(glwe_out, dglwe, count * 2 * kN * 8, cudaMemcpyDeviceToHost, c->stream));
    LV_CUDA(cudaStreamSynchronize(c->stream));
    if (dglwe) cudaFree(dglwe);
    pool_free(c, s.data(), count);
  });
}

int lv_debug_fft(lv_ctx* c, const int64_t* poly, double* spec, uint64_t* roundtrip) {
  return guard([&] {
    CtxLock lk(c);
    int64_t* dpoly = nullptr;
    double2* dspec = nullptr;
    uint64_t* drt = nullptr;
    LV_CUDA(cudaMalloc(&dpoly, kN * 8));
    LV_CUDA(cudaMalloc(&dspec, kM * 16));
    LV_CUDA(cudaMalloc(&drt, kN * 8));
    LV_CUDA(cudaMemcpy(dpoly, poly, kN * 8, cudaMemcpyHostToDevice));
    fft_forward_debug_kernel<<<1, 128, 0, c->stream>>>(dpoly, c->d_tw, c->d_twist, dspec);
    fft_backward_debug_kernel<<<1, 128, 0, c->stream>>>(dspec, c->d_tw, c->d_twist, drt);
    LV_CUDA(cudaGetLastError());
    LV_CUDA(cudaStreamSynchronize(c->stream));
    LV_CUDA(cudaMemcpy(spec, dspec, kM * 16, cudaMemcpyDeviceToHost));
    LV_CUDA(cudaMemcpy(roundtrip, drt, kN * 8, cudaMemcpyDeviceToHost));
    cudaFree(dpoly);
    cudaFree(dspec);
    cudaFree(drt);
  });
}

int lv_bench_fp64_peak(float* tflops) {
  return guard([&] {
    DevTemp<double> d(1);
    int sms = 0, dev = 0;
    LV_CUDA(cudaGetDevice(&dev));
    LV_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int blocks = sms * 8, threads = 256, iters = 8192;
    Event e0, e1;
    float best = 0;
    for (int rep = 0; rep < 4; ++rep) {
      LV_CUDA(cudaEventRecord(e0.e));
      fp64_peak_kernel<<<blocks, threads>>>(d.p, iters, 1.0 + rep);
      LV_CUDA(cudaEventRecord(e1.e));
      LV_CUDA(cudaEventSynchronize(e1.e));
      float ms = 0;
      LV_CUDA(cudaEventElapsedTime(&ms, e0.e, e1.e));
      const double flops = 2.0 * 8 * (double)iters * blocks * threads;
      best = std::max(best, (float)(flops / (ms * 1e-3) / 1e12));
    }
    *tflops = best;
  });
}

int lv_bench_pbs(lv_ctx* c, const lv_ct* in, const uint32_t* luts, size_t count, int iters,
                 uint64_t flush_bytes, float* br_ms, float* ks_ms, float* step_ms) {
  return guard([&] {
    CtxLock lk(c);
    check_handles(c, in, count);
    std::vector<lv_ct> dst = pool_alloc(c, count);
    std::vector<LinDesc> d(count);
    std::vector<BrOut> o(count);
    for (size_t i = 0; i < count; ++i) {
      d[i] = single(in[i]);
      o[i] = BrOut{0, dst[i], kNoSlot, kNoSlot, kNoSlot, 0};
    }
    LinDesc* dd = c->desc.get(count);
    uint32_t* dl = c->lut_item.get(count);
    BrOut* dout = c->br_out.get(count);
    LV_CUDA(cudaMemcpyAsync(dd, d.data(), count * sizeof(LinDesc), cudaMemcpyHostToDevice, c->stream));
    LV_CUDA(cudaMemcpyAsync(dl, luts, count * 4, cudaMemcpyHostToDevice, c->stream));
    LV_CUDA(cudaMemcpyAsync(dout, o.data(), count * sizeof(BrOut), cudaMemcpyHostToDevice, c->stream));
    Event e0, e1, e2;
    DevTemp<uint4> flush(flush_bytes / 16);
    for (int it = 0; it < iters; ++it) {
      if (flush_bytes) flush_kernel<<<1184, 256, 0, c->stream>>>(flush.p, flush_bytes / 16);
      LV_CUDA(cudaEventRecord(e0.e, c->stream));
      launch_pbs_dev(c, dd, dl, dout, (uint32_t)count, e1.e);
      LV_CUDA(cudaEventRecord(e2.e, c->stream));
      LV_CUDA(cudaEventSynchronize(e2.e));
      float a = 0, b = 0, s = 0;
      LV_CUDA(cudaEventElapsedTime(&a, e0.e, e1.e));
      LV_CUDA(cudaEventElapsedTime(&b, e1.e, e2.e));
      LV_CUDA(cudaEventElapsedTime(&s, e0.e, e2.e));
      if (ks_ms) ks_ms[it] = a;
      if (br_ms) br_ms[it] = b;
      if (step_ms) step_ms[it] = s;
    }
    pool_free(c, dst.data(), count);
    c->pbs_count += (uint64_t)count * iters;
  });
}

}  // extern "C"
