// Host-side noise bookkeeping and the symbolic traversal plan.
//
// NoiseLedger restates proj/include/leuven/noise.hpp:19-51 and
// proj/src/noise.cpp:7-36 (sparse sorted signed coefficients over noise
// sources, variance = sum of squares, exact cancellation). It never touches
// the GPU: SURVEY §8(a) a11 — the refresh schedule is data-independent, so
// the planner below replays kernel::distance's ledger arithmetic
// (proj/src/kernel.cpp:165-191, 209-259) once per grid shape and the device
// executes the resulting wave schedule.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

namespace lvb {

class NoiseLedger {
 public:
  using SourceId = uint64_t;
  using Term = std::pair<SourceId, int32_t>;

  static NoiseLedger fresh(SourceId id) {
    NoiseLedger l;
    l.terms_.emplace_back(id, 1);
    return l;
  }
  bool empty() const { return terms_.empty(); }
  size_t term_count() const { return terms_.size(); }
  int64_t variance() const {
    int64_t s = 0;
    for (const auto& t : terms_) s += (int64_t)t.second * t.second;
    return s;
  }
  void add_scaled(const NoiseLedger& other, int32_t factor);
  void scale(int32_t factor);
  const std::vector<Term>& terms() const { return terms_; }

 private:
  std::vector<Term> terms_;
};

// Variance of a*x + b*y without materialising the merge.
int64_t combined_variance(const NoiseLedger& x, int32_t a, const NoiseLedger& y, int32_t b);

struct BandSpec {  // kernel.hpp:47-72
  enum Mode { exact = 0, skip = 1, approx = 2 };
  int mode = exact;
  uint64_t half_width = 0;
  bool covers(uint64_t m, uint64_t n) const { return half_width >= (m > n ? m - n : n - m); }
  bool in_band(uint64_t i, uint64_t j) const { return (i > j ? i - j : j - i) <= half_width; }
};

struct PathRead {  // kernel.hpp:75-81
  bool vertical;
  uint32_t i, j;
};

// staircase_path / last_row_path, kernel.cpp:79-106
std::vector<PathRead> score_path(const BandSpec& band, uint32_t m, uint32_t n);

struct CellPlan {
  uint32_t i, j;
  uint8_t refresh_dv, refresh_dh;
  int64_t key_variance;
};

struct PairPlan {
  uint32_t m = 0, n = 0;
  BandSpec band;
  std::vector<CellPlan> cells;  // reference visiting order (diagonal, then i)
  uint64_t refreshes = 0;
  int64_t max_key_variance = 0;
  std::vector<PathRead> path;
  std::vector<int32_t> score_coeffs;  // score ledger coefficients (fresh ids at run time)
};

// Replays the ledger arithmetic of kernel::distance for one grid shape.
// Throws via the caller-supplied error path (returns false + message) when
// the band is too narrow or the budget is below 11 (kernel.cpp:18, 211-218).
PairPlan plan_pair(uint32_t m, uint32_t n, const BandSpec& band, bool negated, double budget);

}  // namespace lvb
