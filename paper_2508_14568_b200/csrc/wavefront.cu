// Anti-diagonal wavefront scheduler: the B200 form of kernel::distance
// (proj/src/kernel.cpp:209-259), distance_encrypted (:261-268),
// preprocess::build_eq_table / distance_preprocessed
// (proj/src/preprocess.cpp:38-76).
//
// The reference visits one cell at a time. Every cell on an anti-diagonal
// is independent, and so is every stage-s equality check of
// every (i, j) pair, so one launch ("wave") carries
//   - the cell bootstraps of diagonal k            (key -> min table)
//   - equality stage S-1 of diagonal k+1            (-> eq_lut(9))
//   - ...
//   - equality stage 0 of diagonal k+S              (-> eq_lut(1) or (9))
// for every pair of a batch. Refreshes chosen by the symbolic ledger plan
// (ledger.cpp) run as a sub-wave in front of the cells that need them.
// All wave descriptors are built once on the host and uploaded in one copy;
// the waves are then replayed on the stream (captured as a CUDA graph).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "context.hpp"

namespace lvb {

extern thread_local std::string g_last_error;
std::array<int32_t, 16> eq_lut_entries(int scale);

template <typename F>
static int guard_wf(F&& f) {
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

static BandSpec to_band(const lv_band* b) {
  BandSpec s;
  s.mode = b->mode;
  s.half_width = b->half_width;
  return s;
}

// Wave descriptors uploaded per chunk (76 B each: ~160 MB of device memory).
constexpr size_t kWaveChunkItems = size_t(1) << 21;

// Plan cache bound: ~24 B per cell, so 8M cells is ~200 MB of host memory
// (LVB_PLAN_CACHE_CELLS overrides it; the tests shrink it to force eviction).
static uint64_t plan_cache_cells_limit() {
  static const uint64_t v = [] {
    const char* e = std::getenv("LVB_PLAN_CACHE_CELLS");
    return e ? std::strtoull(e, nullptr, 10) : (uint64_t)8 << 20;
  }();
  return v;
}

static std::shared_ptr<const PairPlan> get_plan(lv_ctx* c, uint32_t m, uint32_t n,
                                                const BandSpec& band, bool negated,
                                                double budget) {
  if (!band.covers(m, n))
    throw Error(LV_ERR_BAND_TOO_NARROW, "band half-width " + std::to_string(band.half_width) +
                                            " below length difference");
  if (budget < 11.0)  // kernel.cpp:18, 216-218
    throw Error(LV_ERR_INVALID_PARAMS, "noise budget below 11: refreshed operands alone exceed it");
  const std::string key = std::to_string(m) + "/" + std::to_string(n) + "/" +
                          std::to_string(band.mode) + "/" + std::to_string(band.half_width) + "/" +
                          (negated ? "n" : "o") + "/" + std::to_string(budget);
  auto it = c->plan_cache.find(key);
  if (it != c->plan_cache.end()) {
    it->second.second = ++c->plan_cache_tick;
    return it->second.first;
  }
  auto plan = std::make_shared<const PairPlan>(plan_pair(m, n, band, negated, budget));
  const uint64_t cells = plan->cells.size() + 1;
  // evict least recently used plans until the new one fits
  while (!c->plan_cache.empty() && c->plan_cache_cells + cells > plan_cache_cells_limit()) {
    auto lru = c->plan_cache.begin();
    for (auto e = c->plan_cache.begin(); e != c->plan_cache.end(); ++e)
      if (e->second.second < lru->second.second) lru = e;
    c->plan_cache_cells -= lru->second.first->cells.size() + 1;
    c->plan_cache.erase(lru);
  }
  if (cells <= plan_cache_cells_limit()) {
    c->plan_cache.emplace(key, std::make_pair(plan, ++c->plan_cache_tick));
    c->plan_cache_cells += cells;
  }
  return plan;
}

// One pair's traversal inputs.
struct PairIn {
  uint32_t m, n;
  BandSpec band;
  const lv_ct* a;  // m * S symbol handles (ee) / unused (pre)
  const lv_ct* b;  // n * S symbol handles (ee)
  const lv_eqtable* table = nullptr;
  const char* plain = nullptr;
  const lv_ct* eq9grid = nullptr;  // caller-supplied eq9 handles, row-major m x n (Eq9Provider)
};

struct Wave {
  std::vector<PbsItem> pre;   // refresh sub-wave
  std::vector<PbsItem> main;  // equality stages + cells
};

static LinDesc lin(std::initializer_list<std::pair<uint32_t, int32_t>> terms, int32_t body) {
  LinDesc d{};
  int q = 0;
  for (const auto& t : terms) {
    d.slot[q] = t.first;
    d.coef[q] = t.second;
    ++q;
  }
  d.nterms = q;
  d.body_const = body;
  return d;
}

// Budget check of the equality bootstraps (SimBackend::pbs,
// backend.cpp:62-67, reached through eq4 / fold_step, equality.cpp:22-70):
// stage 0 bootstraps x - y, stage s > 0 bootstraps 2 x_s - 2 y_s - eq_{s-1}
// + 1 with eq_{s-1} a fresh PBS output (variance 1, its own source). A
// bound from the per-stage maxima clears the common case (fresh symbols)
// without touching pairs of cells; otherwise every visited cell's inputs
// are checked exactly, before anything is launched.
static void check_equality_budget(lv_ctx* c, const PairIn& in, const PairPlan& plan, uint32_t S,
                                  double budget) {
  for (uint32_t s = 0; s < S; ++s) {
    const int32_t f = s == 0 ? 1 : 2;
    const int64_t extra = s == 0 ? 0 : 1;
    int64_t va = 0, vb = 0;
    for (uint32_t i = 0; i < in.m; ++i) va = std::max(va, c->ledgers[in.a[(size_t)i * S + s]].variance());
    for (uint32_t j = 0; j < in.n; ++j) vb = std::max(vb, c->ledgers[in.b[(size_t)j * S + s]].variance());
    const double bound = std::pow(f * (std::sqrt((double)va) + std::sqrt((double)vb)), 2) + extra;
    if (bound <= budget) continue;
    for (const CellPlan& cell : plan.cells) {
      const NoiseLedger& x = c->ledgers[in.a[(size_t)(cell.i - 1) * S + s]];
      const NoiseLedger& y = c->ledgers[in.b[(size_t)(cell.j - 1) * S + s]];
      const int64_t v = combined_variance(x, f, y, -f) + extra;
      if ((double)v > budget)
        throw Error(LV_ERR_NOISE_BUDGET, "equality bootstrap input variance " + std::to_string(v) +
                                             " exceeds budget " + std::to_string(budget));
    }
  }
}

// Runs a batch of traversals (S = symbols per character; S == 0 selects
// the preprocessed mode with eq9 taken from the pair's table).
static void run_traversals(lv_ctx* c, const std::vector<PairIn>& pairs, uint32_t S, bool negated,
                           lv_ct* scores, lv_run* runs) {
  const double budget = c->p.max_variance_budget;
  const uint32_t lut_min = c->min_lut[negated ? 1 : 0];
  uint32_t lut_eq1 = 0, lut_eq9 = 0;
  if (S > 0) {
    lut_eq1 = lut_id(c, eq_lut_entries(1));
    lut_eq9 = lut_id(c, eq_lut_entries(9));
  }
  const int32_t dv_coef = negated ? -1 : 1;

  std::vector<std::shared_ptr<const PairPlan>> plans(pairs.size());
  for (size_t p = 0; p < pairs.size(); ++p) {
    const PairIn& in = pairs[p];
    plans[p] = get_plan(c, in.m, in.n, in.band, negated, budget);
    if (S > 0) check_equality_budget(c, in, *plans[p], S, budget);
    if (in.table) {
      for (uint32_t j = 0; j < in.n; ++j)
        if (!in.table->rows.count(in.plain[j]))
          throw Error(LV_ERR_CHAR_NOT_IN_SUBSET,
                      std::string("no table row for character '") + in.plain[j] + "'");
      if (in.table->length != in.m) throw Error(LV_ERR_INVALID_PARAMS, "table length mismatch");
    }
  }

  // frontier slots (index 0 unused), initialised to trivial(1)
  std::vector<std::vector<lv_ct>> vrow(pairs.size()), hcol(pairs.size());
  std::vector<lv_ct> all_frontier;
  for (size_t p = 0; p < pairs.size(); ++p) {
    vrow[p] = pool_alloc(c, pairs[p].m + 1);
    hcol[p] = pool_alloc(c, pairs[p].n + 1);
    all_frontier.insert(all_frontier.end(), vrow[p].begin(), vrow[p].end());
    all_frontier.insert(all_frontier.end(), hcol[p].begin(), hcol[p].end());
  }
  {
    std::vector<int32_t> ones(all_frontier.size(), 1);
    if (!all_frontier.empty()) {
      uint32_t* ds = c->u32a.get(all_frontier.size());
      int32_t* dv = c->i32a.get(all_frontier.size());
      LV_CUDA(cudaMemcpyAsync(ds, all_frontier.data(), all_frontier.size() * 4,
                              cudaMemcpyHostToDevice, c->stream));
      LV_CUDA(cudaMemcpyAsync(dv, ones.data(), ones.size() * 4, cudaMemcpyHostToDevice, c->stream));
      EncArgs ea{c->d_pool, kBigStride, ds, dv, c->d_sk_glwe, c->seed, 0, 0, 1};
      encrypt_kernel<<<(uint32_t)all_frontier.size(), 256, 0, c->stream>>>(ea);
      LV_CUDA(cudaGetLastError());
    }
  }

  // score path: trivial reads count as a constant, stored cells need a
  // slot (final frontier for the exact band's last row, else a snapshot).
  std::vector<std::vector<lv_ct>> path_slots(pairs.size());
  std::vector<int32_t> path_const(pairs.size(), 0);
  std::vector<std::map<uint64_t, uint32_t>> snap_v(pairs.size()), snap_h(pairs.size());
  std::vector<lv_ct> snapshots;
  for (size_t p = 0; p < pairs.size(); ++p) {
    const PairIn& in = pairs[p];
    for (const PathRead& r : plans[p]->path) {
      const bool boundary = r.vertical ? r.j == 0 : r.i == 0;
      if (boundary || !in.band.in_band(r.i, r.j)) {
        path_const[p] += 1;
        continue;
      }
      if (in.band.mode == BandSpec::exact && !r.vertical && r.i == in.m) {
        path_slots[p].push_back(hcol[p][r.j]);
        continue;
      }
      const lv_ct s = pool_alloc(c, 1)[0];
      snapshots.push_back(s);
      path_slots[p].push_back(s);
      (r.vertical ? snap_v : snap_h)[p][((uint64_t)r.i << 32) | r.j] = s;
    }
  }

  // build the waves
  std::map<int64_t, Wave> waves;
  std::vector<lv_ct> temps;
  uint64_t eq_pbs_total = 0, linear_ops = 0;
  for (size_t p = 0; p < pairs.size(); ++p) {
    const PairIn& in = pairs[p];
    const PairPlan& plan = *plans[p];
    lv_run r{};
    // Equality slots live from stage 0 (wave k-2) to the cell (wave k-2+S):
    // diagonals k and k+S+1 never overlap, so a ring of S+1 diagonal groups
    // (each up to min(m,n) cells x S slots) serves the whole traversal.
    const size_t diag_cap = (size_t)std::min(in.m, in.n) + 1;
    std::vector<lv_ct> ring;
    if (S > 0) {
      ring = pool_alloc(c, (S + 1) * diag_cap * S);
      temps.insert(temps.end(), ring.begin(), ring.end());
    }
    int64_t cur_k = -1;
    size_t idx_in_diag = 0;
    for (const CellPlan& cell : plan.cells) {
      const int64_t k = (int64_t)cell.i + cell.j;
      const int64_t wcell = k - 2 + S;
      if (k != cur_k) {
        cur_k = k;
        idx_in_diag = 0;
      }
      const size_t cell_in_diag = idx_in_diag++;
      lv_ct eq9;
      if (S > 0) {
        const lv_ct* ai = in.a + (size_t)(cell.i - 1) * S;
        const lv_ct* bj = in.b + (size_t)(cell.j - 1) * S;
        const lv_ct* eqs = ring.data() + ((size_t)(k % (S + 1)) * diag_cap + cell_in_diag) * S;
        for (uint32_t s = 0; s < S; ++s) {
          PbsItem it{};
          if (s == 0)
            it.in = lin({{ai[0], 1}, {bj[0], -1}}, 0);  // eq4: sub(x, y)
          else  // fold_step: 2 (x_s - y_s) + (1 - eq_prev)
            it.in = lin({{ai[s], 2}, {bj[s], -2}, {eqs[s - 1], -1}}, 1);
          it.lut = (s + 1 == S) ? lut_eq9 : lut_eq1;
          it.out = BrOut{0, eqs[s], kNoSlot, kNoSlot, kNoSlot, 0};
          waves[k - 2 + s].main.push_back(it);
        }
        eq9 = eqs[S - 1];
        r.equality_pbs += S;
        linear_ops += 1 + 4 * (S - 1);
      } else if (in.eq9grid) {
        eq9 = in.eq9grid[(size_t)(cell.i - 1) * in.n + (cell.j - 1)];
      } else {
        eq9 = in.table->rows.at(in.plain[cell.j - 1])[cell.i - 1];
      }
      const lv_ct dv = vrow[p][cell.i], dh = hcol[p][cell.j];
      Wave& w = waves[wcell];
      if (cell.refresh_dv) {  // kernel.cpp:183-188: refresh(dv + 1) - 1
        PbsItem it{};
        it.in = lin({{dv, 1}}, 1);
        it.lut = c->identity_lut;
        it.out = BrOut{0, dv, kNoSlot, kNoSlot, kNoSlot, -1};
        w.pre.push_back(it);
        linear_ops += 2;
      }
      if (cell.refresh_dh) {
        PbsItem it{};
        it.in = lin({{dh, 1}}, 1);
        it.lut = c->identity_lut;
        it.out = BrOut{0, dh, kNoSlot, kNoSlot, kNoSlot, -1};
        w.pre.push_back(it);
        linear_ops += 2;
      }
      PbsItem it{};
      // cell_kernel key (kernel.cpp:152-158): negated 3 dh - dv + eq9 + 4,
      // original dv + 3 dh + eq9 + 4
      it.in = lin({{dv, dv_coef}, {dh, 3}, {eq9, 1}}, 4);
      it.lut = lut_min;
      const uint64_t key = ((uint64_t)cell.i << 32) | cell.j;
      auto sv = snap_v[p].find(key);
      auto sh = snap_h[p].find(key);
      it.out = BrOut{1, dv, dh, sv == snap_v[p].end() ? kNoSlot : sv->second,
                     sh == snap_h[p].end() ? kNoSlot : sh->second, 0};
      w.main.push_back(it);
      linear_ops += 6;
      r.kernel_pbs += 1;
      r.visited_cells += 1;
    }
    r.refreshes = plan.refreshes;
    r.max_key_variance = plan.max_key_variance;
    linear_ops += plan.path.size();
    eq_pbs_total += r.equality_pbs;
    runs[p] = r;
  }

  // flatten and launch in chunks of whole waves: each chunk's descriptors are
  // uploaded into the reused device buffers and its launch sequence replayed
  // as one CUDA graph, so device memory for descriptors stays bounded
  // (kWaveChunkItems) however many pairs a batch holds; chunks run in wave
  // order on the context stream.
  struct Launch {
    size_t off, count;
  };
  uint64_t total_items = 0;
  auto flush = [&](std::vector<LinDesc>& d, std::vector<uint32_t>& l, std::vector<BrOut>& o,
                   std::vector<Launch>& launches) {
    if (d.empty()) return;
    LinDesc* dd = c->desc.get(d.size());
    uint32_t* dl = c->lut_item.get(l.size());
    BrOut* dout = c->br_out.get(o.size());
    LV_CUDA(cudaMemcpyAsync(dd, d.data(), d.size() * sizeof(LinDesc), cudaMemcpyHostToDevice, c->stream));
    LV_CUDA(cudaMemcpyAsync(dl, l.data(), l.size() * 4, cudaMemcpyHostToDevice, c->stream));
    LV_CUDA(cudaMemcpyAsync(dout, o.data(), o.size() * sizeof(BrOut), cudaMemcpyHostToDevice, c->stream));
    size_t max_wave = 0;
    for (const Launch& L : launches) max_wave = std::max(max_wave, L.count);
    // size every scratch buffer before capture (no allocation inside a graph)
    c->ms.get(max_wave * ms_stride(c));
    const size_t ks_rows = (std::min<size_t>(max_wave, 32768) + 127) / 128 * 128;
    c->ks_digits.get(ks_rows * kBig * kKsLevel);
    c->ks_body.get(ks_rows);
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    LV_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    for (const Launch& L : launches)
      launch_pbs_dev(c, dd + L.off, dl + L.off, dout + L.off, (uint32_t)L.count);
    LV_CUDA(cudaStreamEndCapture(c->stream, &graph));
    LV_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    LV_CUDA(cudaGraphLaunch(exec, c->stream));
    LV_CUDA(cudaStreamSynchronize(c->stream));  // the buffers are reused by the next chunk
    cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    d.clear();
    l.clear();
    o.clear();
    launches.clear();
  };
  {
    std::vector<LinDesc> d;
    std::vector<uint32_t> l;
    std::vector<BrOut> o;
    std::vector<Launch> launches;
    for (auto& kv : waves) {
      size_t wave_items = kv.second.pre.size() + kv.second.main.size();
      if (!d.empty() && d.size() + wave_items > kWaveChunkItems) flush(d, l, o, launches);
      for (auto* part : {&kv.second.pre, &kv.second.main}) {
        if (part->empty()) continue;
        launches.push_back({d.size(), part->size()});
        for (const PbsItem& it : *part) {
          d.push_back(it.in);
          l.push_back(it.lut);
          o.push_back(it.out);
        }
        total_items += part->size();
        std::vector<PbsItem>().swap(*part);  // the host copy is no longer needed
      }
    }
    flush(d, l, o, launches);
  }

  // score = trivial(0) + sum of path reads (kernel.cpp:193-200)
  std::vector<lv_ct> outs = pool_alloc(c, pairs.size());
  std::vector<LinOut> sum_ops;
  for (size_t p = 0; p < pairs.size(); ++p) {
    // chain of <=4-term linear combinations accumulating into outs[p]
    const auto& ps = path_slots[p];
    size_t q = 0;
    bool first = true;
    do {
      LinOut op{};
      op.nout = 1;
      op.out_slot[0] = outs[p];
      LinDesc dsc{};
      int t = 0;
      if (!first) {
        dsc.slot[t] = outs[p];
        dsc.coef[t] = 1;
        ++t;
      }
      while (t < 4 && q < ps.size()) {
        dsc.slot[t] = ps[q++];
        dsc.coef[t] = 1;
        ++t;
      }
      dsc.nterms = t;
      dsc.body_const = first ? path_const[p] : 0;
      op.d[0] = dsc;
      sum_ops.push_back(op);
      first = false;
    } while (q < ps.size());
  }
  // the chain for one pair is sequential; issue level by level
  {
    std::vector<std::vector<LinOut>> levels;
    std::vector<size_t> lvl_of(pairs.size(), 0);
    size_t idx = 0;
    for (size_t p = 0; p < pairs.size(); ++p) {
      const auto& ps = path_slots[p];
      const size_t steps = ps.size() <= 4 ? 1 : 1 + (ps.size() - 4 + 2) / 3;
      for (size_t s = 0; s < steps; ++s) {
        if (levels.size() <= s) levels.resize(s + 1);
        levels[s].push_back(sum_ops[idx++]);
      }
    }
    for (auto& lv : levels) run_linear(c, lv);
  }

  // ledgers, counters, cleanup
  for (size_t p = 0; p < pairs.size(); ++p) {
    NoiseLedger led;
    for (int32_t coef : plans[p]->score_coeffs) {
      NoiseLedger one = NoiseLedger::fresh(c->next_source++);
      led.add_scaled(one, coef);
    }
    c->ledgers[outs[p]] = std::move(led);
    scores[p] = outs[p];
    runs[p].waves = waves.size();
  }
  pool_free(c, all_frontier.data(), all_frontier.size());
  pool_free(c, temps.data(), temps.size());
  pool_free(c, snapshots.data(), snapshots.size());
  uint64_t refreshes = 0;
  for (size_t p = 0; p < pairs.size(); ++p) refreshes += runs[p].refreshes;
  c->pbs_count += total_items;
  c->refresh_count += refreshes;
  c->linear_count += linear_ops;
  (void)eq_pbs_total;
}

}  // namespace lvb

using namespace lvb;

extern "C" {

int lv_band_resolve(int32_t mode, uint64_t ell, uint64_t m, uint64_t n, lv_band* out) {
  return guard_wf([&] {
    const uint64_t mx = std::max(m, n);
    if (mode == LV_BAND_EXACT)
      *out = lv_band{LV_BAND_EXACT, mx};
    else if (mode == LV_BAND_SKIP)
      *out = lv_band{LV_BAND_SKIP, (mx + 1) / 2};
    else if (mode == LV_BAND_APPROX)
      *out = lv_band{LV_BAND_APPROX, ell};
    else
      throw Error(LV_ERR_INVALID_PARAMS, "unknown band mode");
  });
}

int lv_edit_distance_ee(lv_ctx* c, const lv_ct* a, size_t m, const lv_ct* b, size_t n,
                        uint32_t symbols, const lv_band* band, int32_t key_encoding, lv_ct* score,
                        lv_run* run) {
  return guard_wf([&] {
    CtxLock lk(c);
    if (symbols < 1)
      throw Error(LV_ERR_INVALID_PARAMS, "equality operands must have the same nonzero symbol count");
    check_handles(c, a, m * symbols);
    check_handles(c, b, n * symbols);
    std::vector<PairIn> pairs{PairIn{(uint32_t)m, (uint32_t)n, to_band(band), a, b}};
    run_traversals(c, pairs, symbols, key_encoding == LV_KEY_NEGATED, score, run);
  });
}

int lv_edit_distance_batch(lv_ctx* c, size_t npairs, const lv_ct* a, const uint64_t* a_off,
                           const lv_ct* b, const uint64_t* b_off, uint32_t symbols,
                           const lv_band* bands, int32_t key_encoding, lv_ct* scores, lv_run* runs) {
  return guard_wf([&] {
    CtxLock lk(c);
    if (symbols < 1)
      throw Error(LV_ERR_INVALID_PARAMS, "equality operands must have the same nonzero symbol count");
    std::vector<PairIn> pairs;
    for (size_t p = 0; p < npairs; ++p) {
      const uint64_t m = a_off[p + 1] - a_off[p], n = b_off[p + 1] - b_off[p];
      check_handles(c, a + a_off[p] * symbols, m * symbols);
      check_handles(c, b + b_off[p] * symbols, n * symbols);
      pairs.push_back(PairIn{(uint32_t)m, (uint32_t)n, to_band(&bands[p]), a + a_off[p] * symbols,
                             b + b_off[p] * symbols});
    }
    run_traversals(c, pairs, symbols, key_encoding == LV_KEY_NEGATED, scores, runs);
  });
}

int lv_eq_table_build(lv_ctx* c, const lv_ct* a, size_t m, uint32_t S, const char* chars,
                      const int32_t* char_symbols, size_t rows, lv_eqtable** out,
                      uint64_t* build_pbs) {
  return guard_wf([&] {
    CtxLock lk(c);
    if (S < 1)
      throw Error(LV_ERR_INVALID_PARAMS, "equality operands must have the same nonzero symbol count");
    check_handles(c, a, m * S);
    const uint32_t lut_eq1 = lut_id(c, eq_lut_entries(1));
    const uint32_t lut_eq9 = lut_id(c, eq_lut_entries(9));
    // budget check of every equality bootstrap input (x - y_const at stage
    // 0, 2 x_s - eq_{s-1} + const after it), as SimBackend::pbs would throw
    for (size_t i = 0; i < m; ++i)
      for (uint32_t s = 0; s < S; ++s) {
        const int64_t v = c->ledgers[a[i * S + s]].variance() * (s == 0 ? 1 : 4) + (s == 0 ? 0 : 1);
        if ((double)v > c->p.max_variance_budget)
          throw Error(LV_ERR_NOISE_BUDGET, "equality bootstrap input variance " + std::to_string(v) +
                                               " exceeds budget " +
                                               std::to_string(c->p.max_variance_budget));
      }
    auto* t = new lv_eqtable();
    t->length = m;
    try {
      // stage-major waves over all (row, position) entries (preprocess.cpp:47-57)
      std::vector<std::vector<lv_ct>> eqs(rows * m);
      for (size_t e = 0; e < rows * m; ++e) eqs[e] = pool_alloc(c, S);
      for (uint32_t s = 0; s < S; ++s) {
        std::vector<PbsItem> items;
        items.reserve(rows * m);
        for (size_t r = 0; r < rows; ++r)
          for (size_t i = 0; i < m; ++i) {
            const lv_ct* ai = a + i * S;
            const int32_t ys = char_symbols[r * S + s];
            PbsItem it{};
            if (s == 0)
              it.in = lin({{ai[0], 1}}, -ys);
            else
              it.in = lin({{ai[s], 2}, {eqs[r * m + i][s - 1], -1}}, 1 - 2 * ys);
            it.lut = (s + 1 == S) ? lut_eq9 : lut_eq1;
            it.out = BrOut{0, eqs[r * m + i][s], kNoSlot, kNoSlot, kNoSlot, 0};
            items.push_back(it);
          }
        run_pbs_items(c, items);
      }
      for (size_t r = 0; r < rows; ++r) {
        std::vector<lv_ct> row(m);
        for (size_t i = 0; i < m; ++i) {
          row[i] = eqs[r * m + i][S - 1];
          c->ledgers[row[i]] = NoiseLedger::fresh(c->next_source++);
          if (S > 1) pool_free(c, eqs[r * m + i].data(), S - 1);
        }
        if (t->rows.count(chars[r])) pool_free(c, t->rows[chars[r]].data(), m);
        t->rows[chars[r]] = std::move(row);
      }
      const uint64_t pbs = (uint64_t)rows * m * S;
      c->pbs_count += pbs;
      c->linear_count += (uint64_t)rows * m * (1 + 4 * (S - 1));
      if (build_pbs) *build_pbs = pbs;
    } catch (...) {
      delete t;
      throw;
    }
    *out = t;
  });
}

int lv_eq_table_lookup(lv_ctx* c, const lv_eqtable* t, char ch, uint64_t position, lv_ct* out) {
  return guard_wf([&] {
    (void)c;
    auto it = t->rows.find(ch);
    if (it == t->rows.end())  // preprocess.cpp:21-31
      throw Error(LV_ERR_CHAR_NOT_IN_SUBSET, std::string("no table row for character '") + ch + "'");
    if (position < 1 || position > t->length)
      throw Error(LV_ERR_POSITION_OUT_OF_RANGE, "position " + std::to_string(position) +
                                                    " outside 1.." + std::to_string(t->length));
    *out = it->second[position - 1];
  });
}

void lv_eq_table_destroy(lv_ctx* c, lv_eqtable* t) {
  if (!t) return;
  if (c) {
    CtxLock lk(c);
    for (auto& kv : t->rows) pool_free(c, kv.second.data(), kv.second.size());
  }
  delete t;
}

// LEQT v2: the reference's table container (preprocess.cpp:80-194, v1 held
// simulated values + ledgers) with real ciphertexts. Little-endian:
//   "LEQT" u32 version=2 | u32 meta_len, meta (caller's alphabet section) |
//   u32 n, u32 N, u32 k, u64 key seed (the keyset the rows decrypt under) |
//   u64 length | u32 rows | rows x { u8 char | length x { u32 terms,
//   i32 coeff[terms] (ledger, ids rebased on load), u64 lwe[N+1] } }
}  // extern "C"
static void put(std::vector<uint8_t>& b, const void* p, size_t n) {
  const uint8_t* s = (const uint8_t*)p;
  b.insert(b.end(), s, s + n);
}
template <typename T>
static void put(std::vector<uint8_t>& b, T v) {
  put(b, &v, sizeof(T));
}
extern "C" {

int lv_eq_table_serialize(lv_ctx* c, const lv_eqtable* t, const uint8_t* meta, uint64_t meta_len,
                          uint8_t* buf, uint64_t cap, uint64_t* len) {
  return guard_wf([&] {
    CtxLock lk(c);
    std::vector<uint8_t> b;
    put(b, "LEQT", 4);
    put<uint32_t>(b, 2);
    put<uint32_t>(b, (uint32_t)meta_len);
    if (meta_len) put(b, meta, meta_len);
    put<uint32_t>(b, c->p.n);
    put<uint32_t>(b, c->p.N);
    put<uint32_t>(b, c->p.k);
    put<uint64_t>(b, c->key_id);
    put<uint64_t>(b, t->length);
    put<uint32_t>(b, (uint32_t)t->rows.size());
    std::vector<uint64_t> rows(t->length * (kBig + 1));
    for (const auto& kv : t->rows) {
      put<uint8_t>(b, (uint8_t)kv.first);
      if (t->length) {
        check_handles(c, kv.second.data(), kv.second.size());
        LV_CUDA(cudaStreamSynchronize(c->stream));
        if (int rc = lv_export(c, kv.second.data(), kv.second.size(), rows.data()))
          throw Error(rc, lv_last_error());
      }
      for (uint64_t i = 0; i < t->length; ++i) {
        const auto& terms = c->ledgers[kv.second[i]].terms();
        put<uint32_t>(b, (uint32_t)terms.size());
        for (const auto& term : terms) put<int32_t>(b, term.second);
        put(b, rows.data() + i * (kBig + 1), (kBig + 1) * 8);
      }
    }
    *len = b.size();
    if (buf) {
      if (cap < b.size()) throw Error(LV_ERR_INVALID_PARAMS, "serialize buffer too small");
      std::memcpy(buf, b.data(), b.size());
    }
  });
}

int lv_eq_table_deserialize(lv_ctx* c, const uint8_t* buf, uint64_t len, lv_eqtable** out,
                            uint8_t* meta_out, uint64_t meta_cap, uint64_t* meta_len) {
  return guard_wf([&] {
    CtxLock lk(c);
    uint64_t pos = 0;
    auto take = [&](void* dst, uint64_t n) {
      if (pos + n > len) throw Error(LV_ERR_FORMAT, "truncated table file");
      if (dst) std::memcpy(dst, buf + pos, n);
      pos += n;
    };
    auto get32 = [&] { uint32_t v; take(&v, 4); return v; };
    auto get64 = [&] { uint64_t v; take(&v, 8); return v; };
    char magic[4];
    take(magic, 4);
    if (std::memcmp(magic, "LEQT", 4) != 0) throw Error(LV_ERR_FORMAT, "not an equality-table file");
    const uint32_t version = get32();
    if (version != 2)
      throw Error(LV_ERR_FORMAT, "unsupported table version " + std::to_string(version));
    const uint32_t ml = get32();
    if (meta_len) *meta_len = ml;
    if (ml > len - pos) throw Error(LV_ERR_FORMAT, "truncated table file");
    if (meta_out && ml <= meta_cap) std::memcpy(meta_out, buf + pos, ml);
    pos += ml;
    const uint32_t n = get32(), N = get32(), k = get32();
    const uint64_t seed = get64();
    if (n != c->p.n || N != c->p.N || k != c->p.k || seed != c->key_id)
      throw Error(LV_ERR_INVALID_PARAMS, "table was encrypted under a different keyset");
    const uint64_t length = get64();
    const uint32_t nrows = get32();
    auto* t = new lv_eqtable();
    t->length = length;
    try {
      std::vector<uint64_t> rows(length * (kBig + 1));
      for (uint32_t r = 0; r < nrows; ++r) {
        uint8_t ch;
        take(&ch, 1);
        std::vector<std::vector<int32_t>> coeffs(length);
        for (uint64_t i = 0; i < length; ++i) {
          const uint32_t terms = get32();
          if ((uint64_t)terms * 4 > len - pos) throw Error(LV_ERR_FORMAT, "truncated table file");
          coeffs[i].resize(terms);
          if (terms) take(coeffs[i].data(), (uint64_t)terms * 4);
          take(rows.data() + i * (kBig + 1), (kBig + 1) * 8);
        }
        std::vector<lv_ct> slots(length);
        if (length)
          if (int rc = lv_import(c, rows.data(), length, slots.data())) throw Error(rc, lv_last_error());
        for (uint64_t i = 0; i < length; ++i) {  // fresh source ids (reserve_source_ids)
          NoiseLedger led;
          for (int32_t co : coeffs[i]) led.add_scaled(NoiseLedger::fresh(c->next_source++), co);
          c->ledgers[slots[i]] = std::move(led);
        }
        if (t->rows.count((char)ch)) throw Error(LV_ERR_FORMAT, "duplicate table row");
        t->rows[(char)ch] = std::move(slots);
      }
    } catch (...) {
      lv_eq_table_destroy(c, t);
      throw;
    }
    *out = t;
  });
}

int lv_edit_distance_eq9(lv_ctx* c, const lv_ct* eq9, uint64_t m, uint64_t n, const lv_band* band,
                         int32_t key_encoding, lv_ct* score, lv_run* run) {
  return guard_wf([&] {
    CtxLock lk(c);
    PairIn in{(uint32_t)m, (uint32_t)n, to_band(band), nullptr, nullptr, nullptr, nullptr, eq9};
    const auto plan = get_plan(c, in.m, in.n, in.band, key_encoding == LV_KEY_NEGATED,
                               c->p.max_variance_budget);
    for (const CellPlan& cell : plan->cells)  // only the visited cells' handles are read
      check_handles(c, eq9 + (size_t)(cell.i - 1) * n + (cell.j - 1), 1);
    std::vector<PairIn> pairs{in};
    run_traversals(c, pairs, 0, key_encoding == LV_KEY_NEGATED, score, run);
  });
}

int lv_edit_distance_pre(lv_ctx* c, const lv_eqtable* t, const char* plain, size_t n,
                         const lv_band* band, int32_t key_encoding, lv_ct* score, lv_run* run) {
  return guard_wf([&] {
    CtxLock lk(c);
    PairIn in{(uint32_t)t->length, (uint32_t)n, to_band(band), nullptr, nullptr, t, plain};
    std::vector<PairIn> pairs{in};
    run_traversals(c, pairs, 0, key_encoding == LV_KEY_NEGATED, score, run);
  });
}

int lv_edit_distance_pre_batch(lv_ctx* c, size_t npairs, const lv_eqtable* const* tables,
                               const char* plains, const uint64_t* plain_off,
                               const lv_band* bands, int32_t key_encoding, lv_ct* scores,
                               lv_run* runs) {
  return guard_wf([&] {
    CtxLock lk(c);
    std::vector<PairIn> pairs;
    pairs.reserve(npairs);
    for (size_t p = 0; p < npairs; ++p) {
      if (!tables[p]) throw Error(LV_ERR_INVALID_HANDLE, "null equality table");
      const uint64_t n = plain_off[p + 1] - plain_off[p];
      pairs.push_back(PairIn{(uint32_t)tables[p]->length, (uint32_t)n, to_band(&bands[p]), nullptr,
                             nullptr, tables[p], plains + plain_off[p]});
    }
    run_traversals(c, pairs, 0, key_encoding == LV_KEY_NEGATED, scores, runs);
  });
}

int lv_plan_trace(uint64_t m, uint64_t n, const lv_band* band, int32_t key_encoding, double budget,
                  uint64_t cap, uint32_t* ij, int64_t* key_var, uint32_t* refreshes,
                  uint64_t* count, lv_run* totals) {
  return guard_wf([&] {
    const BandSpec b = to_band(band);
    if (!b.covers(m, n))
      throw Error(LV_ERR_BAND_TOO_NARROW,
                  "band half-width " + std::to_string(b.half_width) + " below length difference");
    if (budget < 11.0)
      throw Error(LV_ERR_INVALID_PARAMS, "noise budget below 11: refreshed operands alone exceed it");
    const PairPlan plan = plan_pair((uint32_t)m, (uint32_t)n, b, key_encoding == LV_KEY_NEGATED, budget);
    const uint64_t k = plan.cells.size();
    for (uint64_t q = 0; q < std::min(k, cap); ++q) {
      ij[2 * q] = plan.cells[q].i;
      ij[2 * q + 1] = plan.cells[q].j;
      key_var[q] = plan.cells[q].key_variance;
      refreshes[q] = plan.cells[q].refresh_dv + plan.cells[q].refresh_dh;
    }
    *count = k;
    if (totals) {
      lv_run r{};
      r.visited_cells = k;
      r.kernel_pbs = k;
      r.refreshes = plan.refreshes;
      r.max_key_variance = plan.max_key_variance;
      *totals = r;
    }
  });
}

}  // extern "C"
