// Host-side planning for the mask builder: the scalar radial-prior formulas
// of stage (a) evaluated per ordered frame pair, with the exact integer /
// double arithmetic of the reference so that every decision (window, split,
// tier, k) is bit-identical:
//   group_index / base_span / decay_length   radial.cpp:10-28
//   window_width                             radial.cpp:30-39
//   split_factor / frame_retained            radial.cpp:41-54
//   CandidateSet::pair_count                 radial.cpp:56-62
//   distance_tier / retention / threshold    selection.cpp:34-59
// These are O(N_f^2) scalars that size and parameterise the device work
// (launch planning); all per-token and per-pair work runs on the GPU.
#pragma once

#include <cmath>
#include <cstdint>
#include <limits>
#include <stdexcept>
#include <vector>

#include "dynrad.h"

namespace rp {
namespace plan {

inline int group_index(int64_t t) {
  if (t < 1) throw std::invalid_argument("group_index: t must be >= 1");
  int b = 0;
  for (uint64_t x = static_cast<uint64_t>(t); x; x >>= 1) ++b;
  return b;
}

inline int64_t base_span(int64_t n) {
  if (n < 1) throw std::invalid_argument("base_span: tokens_per_frame must be >= 1");
  int64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

inline double decay_length(int64_t t, double factor, int64_t base) {
  return factor * static_cast<double>(base) /
         static_cast<double>(int64_t{1} << group_index(t));
}

inline int64_t window_width(int i, int j, const rp_config& c, const rp_grid& g) {
  const int64_t t = std::llabs(static_cast<long long>(i) - j);
  if (t <= 1) return g.tokens_per_frame;
  const double len = decay_length(t, c.decay_factor, base_span(g.tokens_per_frame));
  const int64_t r = std::llround(len);
  return r > g.block_size ? r : g.block_size;
}

inline int64_t split_factor(int64_t t, const rp_config& c, const rp_grid& g) {
  if (t < 1) throw std::invalid_argument("split_factor: t must be >= 1");
  const double len = decay_length(t, c.long_range_factor, base_span(g.tokens_per_frame));
  const double raw = static_cast<double>(g.block_size) / (len + c.split_epsilon);
  const int64_t f = static_cast<int64_t>(raw);
  return f > 1 ? f : 1;
}

inline bool frame_retained(int64_t t, const rp_config& c, const rp_grid& g) {
  if (t <= 1) return true;
  return t % split_factor(t, c, g) == 0;
}

inline int64_t band_pairs(int64_t n, int64_t w) {
  if (w >= n - 1) return n * n;
  const int64_t m = n - 1 - w;
  return n * n - m * (m + 1);
}

inline int distance_tier(int i, int j, const rp_config& c, const rp_grid& g) {
  const int64_t t = std::llabs(static_cast<long long>(i) - j);
  if (t <= 1) return 0;
  const double len = decay_length(t, c.decay_factor, base_span(g.tokens_per_frame));
  return len >= static_cast<double>(g.block_size) ? 1 : 2;
}

// Smallest count c in [0, B] with double(c)/B >= theta (thresholds are
// evaluated exactly as the reference's double comparisons, mask.cpp:115-122);
// B + 1 if none.
inline int count_threshold(double theta, int B) {
  for (int c = 0; c <= B; ++c)
    if (static_cast<double>(c) / B >= theta) return c;
  return B + 1;
}

// One job = one ordered frame pair (i != j) that survives the split rule
// (or every pair when disable_split), mask.cpp:185-192.
enum JobKind : int32_t {
  kFullBand = 0,  // ratio >= 1 or tau = -inf: closed-form column counts
  kSample = 1,    // static ratio < 1: partial Fisher-Yates
  kScore = 2,     // dynamic finite tau: proxy scores + z threshold
  kEmpty = 3      // pruned pair kept by disable_split with no candidates
};

struct Job {
  int32_t i, j;
  int32_t kind;
  int32_t tier;
  int64_t width;
  int64_t n;      // candidate pairs (0 if not retained)
  int64_t k;      // static: draws; otherwise 0
  double param;   // ratio or tau
  uint64_t stream_seed;
};

inline void validate(const rp_config& c) {
  if (!(c.decay_factor > 0.0))
    throw std::invalid_argument("config: decay_factor must be positive");
  if (!(c.long_range_factor > 0.0))
    throw std::invalid_argument("config: long_range_factor must be positive");
  if (!(c.mask_threshold > 0.0 && c.mask_threshold <= 1.0))
    throw std::invalid_argument("config: mask_threshold must be in (0, 1]");
  if (!(c.col_threshold > 0.0 && c.col_threshold <= 1.0))
    throw std::invalid_argument("config: col_threshold must be in (0, 1]");
  if (c.fallback_k < 1) throw std::invalid_argument("config: fallback_k must be >= 1");
  if (c.mode == RP_STATIC_RATIO) {
    if (!(c.near_param > 0.0 && c.near_param <= 1.0) ||
        !(c.far_param > 0.0 && c.far_param <= 1.0))
      throw std::invalid_argument("config: static retention ratios must be in (0, 1]");
  } else {
    if (!std::isfinite(c.near_param) || !std::isfinite(c.far_param))
      throw std::invalid_argument("config: dynamic thresholds must be finite");
  }
}

}  // namespace plan
}  // namespace rp
