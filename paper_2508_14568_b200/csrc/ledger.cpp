#include "ledger.hpp"

#include <algorithm>

namespace lvb {

void NoiseLedger::add_scaled(const NoiseLedger& other, int32_t factor) {
  if (factor == 0 || other.terms_.empty()) return;
  std::vector<Term> merged;
  merged.reserve(terms_.size() + other.terms_.size());
  size_t a = 0, b = 0;
  while (a < terms_.size() || b < other.terms_.size()) {
    if (b == other.terms_.size() || (a < terms_.size() && terms_[a].first < other.terms_[b].first)) {
      merged.push_back(terms_[a++]);
    } else if (a == terms_.size() || other.terms_[b].first < terms_[a].first) {
      merged.emplace_back(other.terms_[b].first, other.terms_[b].second * factor);
      ++b;
    } else {
      const int32_t c = terms_[a].second + other.terms_[b].second * factor;
      if (c != 0) merged.emplace_back(terms_[a].first, c);
      ++a;
      ++b;
    }
  }
  terms_ = std::move(merged);
}

void NoiseLedger::scale(int32_t factor) {
  if (factor == 0) {
    terms_.clear();
    return;
  }
  if (factor == 1) return;
  for (auto& t : terms_) t.second *= factor;
}

int64_t combined_variance(const NoiseLedger& x, int32_t a, const NoiseLedger& y, int32_t b) {
  const auto& X = x.terms();
  const auto& Y = y.terms();
  size_t p = 0, q = 0;
  int64_t s = 0;
  while (p < X.size() || q < Y.size()) {
    int64_t c;
    if (q == Y.size() || (p < X.size() && X[p].first < Y[q].first)) {
      c = (int64_t)X[p++].second * a;
    } else if (p == X.size() || Y[q].first < X[p].first) {
      c = (int64_t)Y[q++].second * b;
    } else {
      c = (int64_t)X[p++].second * a + (int64_t)Y[q++].second * b;
    }
    s += c * c;
  }
  return s;
}

std::vector<PathRead> score_path(const BandSpec& band, uint32_t m, uint32_t n) {
  std::vector<PathRead> path;
  path.reserve(m + n);
  if (band.mode == BandSpec::exact) {  // last_row_path, kernel.cpp:100-106
    for (uint32_t i = 1; i <= m; ++i) path.push_back({true, i, 0});
    for (uint32_t j = 1; j <= n; ++j) path.push_back({false, m, j});
    return path;
  }
  if (m >= n) {  // staircase_path, kernel.cpp:79-98
    const uint32_t d = m - n;
    for (uint32_t i = 1; i <= d; ++i) path.push_back({true, i, 0});
    for (uint32_t k = 1; k <= n; ++k) {
      path.push_back({false, d + k - 1, k});
      path.push_back({true, d + k, k});
    }
  } else {
    const uint32_t d = n - m;
    for (uint32_t j = 1; j <= d; ++j) path.push_back({false, 0, j});
    for (uint32_t k = 1; k <= m; ++k) {
      path.push_back({true, k, d + k - 1});
      path.push_back({false, k, d + k});
    }
  }
  return path;
}

PairPlan plan_pair(uint32_t m, uint32_t n, const BandSpec& band, bool negated, double budget) {
  PairPlan plan;
  plan.m = m;
  plan.n = n;
  plan.band = band;
  const int32_t dv_coeff = negated ? -1 : 1;
  NoiseLedger::SourceId next = 1;
  // frontier ledgers; boundary / out-of-band reads are trivial(1): empty ledger.
  std::vector<NoiseLedger> v_row(m + 1), h_col(n + 1);
  std::vector<uint32_t> v_col(m + 1, 0), h_row(n + 1, 0);  // coordinate tag of the frontier
  plan.path = score_path(band, m, n);
  // kept ledgers for the score path cells
  std::vector<NoiseLedger> path_led(plan.path.size());
  std::vector<std::vector<std::pair<uint32_t, size_t>>> want_v(m + 1), want_h(m + 1);
  for (size_t p = 0; p < plan.path.size(); ++p) {
    const PathRead& r = plan.path[p];
    (r.vertical ? want_v : want_h)[r.i].push_back({r.j, p});
  }
  const NoiseLedger empty;
  for (uint64_t k = 2; k <= (uint64_t)m + n; ++k) {
    const uint64_t i_lo = k > n ? k - n : 1;
    const uint64_t i_hi = std::min<uint64_t>(m, k - 1);
    for (uint64_t i = i_lo; i <= i_hi; ++i) {
      const uint64_t j = k - i;
      if (!band.in_band(i, j)) continue;
      const bool dv_live = (j - 1) != 0 && band.in_band(i, j - 1);
      const bool dh_live = (i - 1) != 0 && band.in_band(i - 1, j);
      NoiseLedger dv = dv_live ? v_row[i] : empty;
      NoiseLedger dh = dh_live ? h_col[j] : empty;
      CellPlan c{(uint32_t)i, (uint32_t)j, 0, 0, 0};
      // key = dv_coeff*dv + 3*dh + eq9, eq9 a fresh independent source
      int64_t kv = combined_variance(dv, dv_coeff, dh, 3) + 1;
      if ((double)kv > budget) {
        if (dv.variance() > 1) {
          dv = NoiseLedger::fresh(next++);
          c.refresh_dv = 1;
          ++plan.refreshes;
        }
        if (dh.variance() > 1) {
          dh = NoiseLedger::fresh(next++);
          c.refresh_dh = 1;
          ++plan.refreshes;
        }
        kv = combined_variance(dv, dv_coeff, dh, 3) + 1;
      }
      c.key_variance = kv;
      plan.max_key_variance = std::max(plan.max_key_variance, kv);
      const NoiseLedger step = NoiseLedger::fresh(next++);
      NoiseLedger dv_out = step;
      dv_out.add_scaled(dh, -1);
      NoiseLedger dh_out = step;
      dh_out.add_scaled(dv, -1);
      for (const auto& w : want_v[i])
        if (w.first == j) path_led[w.second] = dv_out;
      for (const auto& w : want_h[i])
        if (w.first == j) path_led[w.second] = dh_out;
      v_row[i] = std::move(dv_out);
      v_col[i] = (uint32_t)j;
      h_col[j] = std::move(dh_out);
      h_row[j] = (uint32_t)i;
      plan.cells.push_back(c);
    }
  }
  NoiseLedger score;
  for (const auto& l : path_led) score.add_scaled(l, 1);
  for (const auto& t : score.terms()) plan.score_coeffs.push_back(t.second);
  return plan;
}

}  // namespace lvb
