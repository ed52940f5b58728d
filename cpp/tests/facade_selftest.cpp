// TEST INFRASTRUCTURE — unit tests of the C++ facade (no reference needed).
//
//   facade_selftest            host-side checks; GPU checks when a device is
//                              present, else every GPU entry point must throw
//                              (no CPU fallback)
//   facade_selftest mask ARGS  prints the hex of build_mask's BlockMask for
//                              pytest to compare with the oracle:
//     nf nt bs mode gamma lambda theta_m theta_c near far fallback_k seed
//     [feat_seed heads dim]   (dynamic mode: random_batch features)
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN_DEFERRED
#include "doctest.h"

#include <cuda_runtime_api.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>

#include "radialplan/attention.hpp"
#include "radialplan/mask.hpp"
#include "radialplan/profiler.hpp"
#include "radialplan/radial.hpp"
#include "radialplan/selection.hpp"

using namespace radialplan;

static bool have_gpu() {
  int n = 0;
  return cudaGetDeviceCount(&n) == cudaSuccess && n > 0;
}

TEST_CASE("grid geometry and errors") {
  const GridSpec g = make_grid(21, 3600, 128);
  CHECK(g.total_tokens == 75600);
  CHECK(g.padded_tokens == 75648);
  CHECK(g.blocks_per_dim == 591);
  CHECK(frame_of(75647, g) == 20);
  CHECK(block_of(75647, g) == 590);
  CHECK_THROWS_AS(make_grid(2, 4, 12), std::invalid_argument);
  CHECK_THROWS_AS(block_of(75648, g), std::out_of_range);
}

TEST_CASE("radial scalars (SPEC.md:121-159 examples)") {
  const GridSpec g = make_grid(21, 3600, 128);
  RadialParams p;
  p.decay_factor = 2.0;
  CHECK(base_span(3600) == 4096);
  CHECK(window_width(0, 2, p, g) == 2048);
  CHECK(window_width(0, 4, p, g) == 1024);
  CHECK(window_width(0, 16, p, g) == 256);
  CHECK(window_width(3, 3, p, g) == 3600);
  p.long_range_factor = 0.3;
  int kept = 0;
  for (int t = 2; t < 21; ++t) kept += frame_retained(t, p, g);
  CHECK(kept == 15);  // Wan Low keeps 15/19 distances
  const CandidateSet cs = candidate_set(0, 2, p, g);
  CHECK(cs.pair_count() == 3600LL * 3600 - 1551LL * 1552);
  const auto off = cs.row_offsets();
  CHECK(off.back() == cs.pair_count());
  const auto uv = cs.pair_at(cs.pair_count() - 1);
  CHECK((uv.first == 3599 && uv.second == 3599));
}

TEST_CASE("config validation messages") {
  SparsityConfig c;
  c.mask_threshold = 0.0;
  try {
    c.validate();
    CHECK(false);
  } catch (const std::invalid_argument& e) {
    CHECK(std::string(e.what()) == "config: mask_threshold must be in (0, 1]");
  }
  SparsityConfig d;
  d.mode = Mode::DynamicThreshold;
  d.near_param = 1.0 / 0.0;
  CHECK_THROWS_AS(d.validate(), std::invalid_argument);
}

TEST_CASE("aggregate_block (SPEC.md:319)") {
  std::vector<std::pair<int, int>> kept;
  for (int r = 0; r < 4; ++r) {
    kept.emplace_back(r, 0);
    kept.emplace_back(r, 1);
  }
  CHECK(aggregate_block(kept, 0.5, 0.5, 4));
  CHECK_FALSE(aggregate_block(kept, 0.5, 0.6, 4));
  CHECK_THROWS_AS(aggregate_block({{4, 0}}, 0.5, 0.5, 4), std::out_of_range);
}

TEST_CASE("mask files (mask.cpp:291-376 formats)") {
  BlockMask m(11);
  m.set(0, 0);
  m.set(3, 10);
  m.set(10, 4);
  const std::string base = "/tmp/facade_selftest_mask";
  write_mask(m, mask_format_for_path(base + ".bin"), base + ".bin");
  CHECK(read_mask(base + ".bin") == m);
  write_mask(m, MaskFormat::Csv, base + ".csv");
  std::ifstream csv(base + ".csv");
  std::string all((std::istreambuf_iterator<char>(csv)), std::istreambuf_iterator<char>());
  CHECK(all == "0,0\n3,10\n10,4\n");
  CHECK_THROWS_AS(mask_format_for_path("m.txt"), std::invalid_argument);
  CHECK_THROWS_AS(read_mask(base + ".csv"), std::runtime_error);
}

TEST_CASE("GPU operators or a loud failure") {
  const GridSpec g = make_grid(4, 64, 16);
  SparsityConfig c;
  c.near_param = c.far_param = 0.3;
  CHECK_THROWS_AS(masked_attention(random_batch(64, 1, 8, 5, true), TokenMask(64), 0.0),
                  std::invalid_argument);  // attention.cpp:109-110, before any device work
  if (!have_gpu()) {
    CHECK_THROWS_AS(build_mask(g, c, 7), std::runtime_error);
    CHECK_THROWS_AS(sparsity(BlockMask(4)), std::runtime_error);
    return;
  }
  const BlockMask m = build_mask(g, c, 7);
  CHECK(m.dim == g.blocks_per_dim);
  const double sp = sparsity(m);
  CHECK(sp == doctest::Approx(1.0 - static_cast<double>(m.active_count()) / (16.0 * 16.0)));
  const TokenMask t = expand_mask(m, g);
  for (std::int64_t r = 0; r < g.padded_tokens; r += 7)
    for (std::int64_t col = 0; col < g.padded_tokens; col += 5)
      CHECK(t.get(r, col) == m.get(r / 16, col / 16));
  // normalize_scores KAT: {0, 2} -> {-1, +1}
  ScoreStats st;
  const auto z = normalize_scores({0.0f, 2.0f}, &st);
  CHECK(st.mean == 1.0);
  CHECK(st.stddev == 1.0);
  CHECK(z[0] == doctest::Approx(-1.0));
  CHECK(z[1] == doctest::Approx(1.0));
  // static_select KAT: k = 13 of |P| = 52 at rho = .25
  RadialParams p;
  const GridSpec g2 = make_grid(2, 8, 4);
  CandidateSet cs = candidate_set(0, 1, p, g2);
  cs.width = 3;  // |u - v| <= 3 over 8 tokens: 8*8 - 4*5 = 44 pairs
  CHECK(cs.pair_count() == 44);
  CHECK(static_select(cs, 0.25, 9).size() == 11u);
  // masked_attention_exact: single-key rows reproduce V
  const FeatureBatch b = random_batch(64, 1, 8, 5, true);
  BlockMask diag(4);
  for (int x = 0; x < 4; ++x) diag.set(x, x);
  const GridSpec g3 = make_grid(1, 64, 16);
  const auto o = masked_attention_exact(b, expand_mask(diag, g3));
  CHECK(o.size() == 1u);
  CHECK(o[0].rows() == 64);
  // soft mask: at eps -> 0 it approaches the exact variant
  const auto os = masked_attention(b, expand_mask(diag, g3), 1e-12);
  float worst = 0.f;
  for (Eigen::Index r = 0; r < 64; ++r)
    for (Eigen::Index e = 0; e < 8; ++e) worst = std::max(worst, std::abs(os[0](r, e) - o[0](r, e)));
  CHECK(worst < 1e-5f);
}

// facade_selftest objective nf nt bs dim mode gamma lambda tm tc near far fk seed
// prints loss mse sparsity (%.17g) without and with a host DenseProxyCache;
// features f[t][d] = ((t*131 + d*71) % 97 - 48) / 32 (exact in any language).
static int print_objective(int argc, char** argv) {
  if (argc < 15) return 2;
  ProxyBatch b;
  b.grid = make_grid(std::atoi(argv[2]), std::atoi(argv[3]), std::atoi(argv[4]));
  b.feature_dim = std::atoi(argv[5]);
  b.seed = std::strtoull(argv[14], nullptr, 10);
  b.features = Eigen::MatrixXf(b.grid.total_tokens, b.feature_dim);
  for (std::int64_t t = 0; t < b.grid.total_tokens; ++t)
    for (int d = 0; d < b.feature_dim; ++d)
      b.features(t, d) = static_cast<float>((t * 131 + d * 71) % 97 - 48) / 32.0f;
  SparsityConfig c;
  c.mode = std::atoi(argv[6]) ? Mode::DynamicThreshold : Mode::StaticRatio;
  c.radial.decay_factor = std::atof(argv[7]);
  c.radial.long_range_factor = std::atof(argv[8]);
  c.mask_threshold = std::atof(argv[9]);
  c.col_threshold = std::atof(argv[10]);
  c.near_param = std::atof(argv[11]);
  c.far_param = std::atof(argv[12]);
  c.fallback_k = std::atoi(argv[13]);
  const TrialRecord a = objective(c, b, 10.0, 0.8);
  const DenseProxyCache cache = build_proxy_cache(b);
  const TrialRecord r = objective(c, b, 10.0, 0.8, &cache);
  std::printf("%.17g %.17g %.17g\n%.17g %.17g %.17g\n%.17g\n", a.loss, a.mse,
              a.achieved_sparsity, r.loss, r.mse, r.achieved_sparsity, cache.reference_sq_norm);
  return 0;
}

static int print_mask(int argc, char** argv) {
  if (argc < 14) {
    std::fprintf(stderr, "usage: mask nf nt bs mode gamma lambda tm tc near far fk seed "
                         "[feat_seed heads dim]\n");
    return 2;
  }
  const GridSpec g = make_grid(std::atoi(argv[2]), std::atoi(argv[3]), std::atoi(argv[4]));
  SparsityConfig c;
  c.mode = std::atoi(argv[5]) ? Mode::DynamicThreshold : Mode::StaticRatio;
  c.radial.decay_factor = std::atof(argv[6]);
  c.radial.long_range_factor = std::atof(argv[7]);
  c.mask_threshold = std::atof(argv[8]);
  c.col_threshold = std::atof(argv[9]);
  c.near_param = std::atof(argv[10]);
  c.far_param = std::atof(argv[11]);
  c.fallback_k = std::atoi(argv[12]);
  const std::uint64_t seed = std::strtoull(argv[13], nullptr, 10);
  FeatureBatch f;
  BuildOptions o;
  if (argc >= 17) {
    f = random_batch(g.total_tokens, std::atoi(argv[15]), std::atoi(argv[16]),
                     std::strtoull(argv[14], nullptr, 10), false);
    o.features = &f;
  }
  BuildTimings t;
  o.timings = &t;
  const BlockMask m = build_mask(g, c, seed, o);
  for (std::uint8_t byte : m.bits) std::printf("%02x", byte);
  std::printf("\n");
  std::fprintf(stderr, "retained %lld scored %lld\n", static_cast<long long>(t.retained_frame_pairs),
               static_cast<long long>(t.scored_pairs));
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && std::strcmp(argv[1], "mask") == 0) return print_mask(argc, argv);
  if (argc > 1 && std::strcmp(argv[1], "objective") == 0) return print_objective(argc, argv);
  return doctest::run_all();
}
