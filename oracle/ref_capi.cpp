// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A thin extern "C" wrapper around the reference's OWN radialplan sources,
// compiled in place from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libradialplan_ref.so.  Python tests (ctypes) use it to run the
// unmodified reference implementation on the same inputs as the CUDA path,
// and bench.py's reference arm times it as the CPU baseline.
//
// Layout convention at this boundary: feature tensors are [tokens, heads,
// head_dim] row-major float32 (the product's [S, H, d] layout); they are
// scattered into the reference's per-head column-major Eigen::MatrixXf
// (attention.hpp:18-27) before the call.
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "oracle.hpp"
#include "radialplan/attention.hpp"
#include "radialplan/mask.hpp"
#include "radialplan/profiler.hpp"
#include "radialplan/proxy.hpp"
#include "radialplan/radial.hpp"
#include "radialplan/selection.hpp"

using namespace radialplan;

extern "C" {

struct ref_cfg {
  int mode;  // 0 static, 1 dynamic
  double decay_factor, long_range_factor, split_epsilon;
  double mask_threshold, col_threshold, near_param, far_param;
  int fallback_k;
};

}  // extern "C"

namespace {

thread_local std::string g_err;

// Error codes mirror include/dynrad.h's rp_status: 1 invalid_argument,
// 2 out_of_range, 3 domain_error, 4 runtime_error, 5 other.
template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 2;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

SparsityConfig to_cfg(const ref_cfg* c) {
  SparsityConfig s;
  s.mode = c->mode == 0 ? Mode::StaticRatio : Mode::DynamicThreshold;
  s.radial.decay_factor = c->decay_factor;
  s.radial.long_range_factor = c->long_range_factor;
  s.radial.split_epsilon = c->split_epsilon;
  s.mask_threshold = c->mask_threshold;
  s.col_threshold = c->col_threshold;
  s.near_param = c->near_param;
  s.far_param = c->far_param;
  s.fallback_k = c->fallback_k;
  return s;
}

std::vector<Eigen::MatrixXf> unpack(const float* x, std::int64_t tokens,
                                    int heads, int d) {
  std::vector<Eigen::MatrixXf> out;
  for (int h = 0; h < heads; ++h) {
    Eigen::MatrixXf m(tokens, d);
    for (std::int64_t t = 0; t < tokens; ++t)
      for (int k = 0; k < d; ++k)
        m(t, k) = x[(t * heads + h) * d + k];
    out.push_back(std::move(m));
  }
  return out;
}

FeatureBatch make_batch(const float* q, const float* k, const float* v,
                        std::int64_t tokens, int heads, int d) {
  FeatureBatch b;
  b.tokens = tokens;
  b.heads = heads;
  b.head_dim = d;
  b.queries = unpack(q, tokens, heads, d);
  b.keys = unpack(k, tokens, heads, d);
  if (v) b.values = unpack(v, tokens, heads, d);
  return b;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_make_grid(int nf, int nt, int bs, std::int64_t* out4) {
  return guarded([&] {
    GridSpec g = make_grid(nf, nt, bs);
    out4[0] = g.total_tokens;
    out4[1] = g.padded_tokens;
    out4[2] = g.blocks_per_dim;
    out4[3] = (g.blocks_per_dim + 7) / 8;
  });
}

// radialplan::build_mask (mask.hpp:88).  q/k: [tokens, heads, d] or NULL.
// out_bits: blocks * row_bytes bytes.  timings: 5 doubles (candidates_s,
// selection_s, aggregation_s, retained_frame_pairs, scored_pairs) or NULL.
int ref_build_mask(int nf, int nt, int bs, const ref_cfg* cfg,
                   std::uint64_t seed, int disable_split, const float* q,
                   const float* k, std::int64_t tokens, int heads, int d,
                   std::uint8_t* out_bits, double* timings) {
  return guarded([&] {
    GridSpec g = make_grid(nf, nt, bs);
    SparsityConfig c = to_cfg(cfg);
    BuildTimings bt;
    BuildOptions opt;
    opt.disable_split = disable_split != 0;
    opt.timings = &bt;
    FeatureBatch fb;
    if (q && k) {
      fb = make_batch(q, k, nullptr, tokens, heads, d);
      opt.features = &fb;
    }
    BlockMask m = build_mask(g, c, seed, opt);
    std::memcpy(out_bits, m.bits.data(), m.bits.size());
    if (timings) {
      timings[0] = bt.candidates_s;
      timings[1] = bt.selection_s;
      timings[2] = bt.aggregation_s;
      timings[3] = static_cast<double>(bt.retained_frame_pairs);
      timings[4] = static_cast<double>(bt.scored_pairs);
    }
  });
}

// The reference's own brute-force transcription (tests/oracle.cpp:166).
// out_dense: blocks*blocks bytes, one per block.
int ref_oracle_build(int nf, int nt, int bs, const ref_cfg* cfg,
                     std::uint64_t seed, int disable_split, const float* q,
                     const float* k, std::int64_t tokens, int heads, int d,
                     std::uint8_t* out_dense) {
  return guarded([&] {
    oracle::Grid g = oracle::grid(nf, nt, bs);
    SparsityConfig c = to_cfg(cfg);
    FeatureBatch fb;
    const FeatureBatch* fp = nullptr;
    if (q && k) {
      fb = make_batch(q, k, nullptr, tokens, heads, d);
      fp = &fb;
    }
    oracle::DenseMask m = oracle::build(g, c, fp, seed, disable_split != 0);
    std::memcpy(out_dense, m.a.data(), m.a.size());
  });
}

// masked_attention / masked_attention_exact (attention.hpp:37-44) on the
// token expansion of a block mask.  out: [padded_tokens, heads, d].
int ref_masked_attention(int nf, int nt, int bs, const std::uint8_t* bits,
                         const float* q, const float* k, const float* v,
                         std::int64_t tokens, int heads, int d, int exact,
                         double eps, float* out) {
  return guarded([&] {
    GridSpec g = make_grid(nf, nt, bs);
    BlockMask bm(g.blocks_per_dim);
    std::memcpy(bm.bits.data(), bits, bm.bits.size());
    TokenMask tm = expand_mask(bm, g);
    FeatureBatch fb = make_batch(q, k, v, tokens, heads, d);
    std::vector<Eigen::MatrixXf> o =
        exact ? masked_attention_exact(fb, tm) : masked_attention(fb, tm, eps);
    const std::int64_t n = g.padded_tokens;
    for (int h = 0; h < heads; ++h)
      for (std::int64_t t = 0; t < n; ++t)
        for (int c = 0; c < d; ++c) out[(t * heads + h) * d + c] = o[h](t, c);
  });
}

// expand_mask (mask.hpp:57, mask.cpp:52-66): the TokenMask bytes.
int ref_expand_mask(int nf, int nt, int bs, const std::uint8_t* bits, std::uint8_t* out) {
  return guarded([&] {
    GridSpec g = make_grid(nf, nt, bs);
    BlockMask bm(g.blocks_per_dim);
    std::memcpy(bm.bits.data(), bits, bm.bits.size());
    TokenMask tm = expand_mask(bm, g);
    std::memcpy(out, tm.bits.data(), tm.bits.size());
  });
}

// random_batch (attention.hpp:62): [tokens, heads, d] each; v may be NULL.
int ref_random_batch(std::int64_t tokens, int heads, int d, std::uint64_t seed,
                     float* q, float* k, float* v) {
  return guarded([&] {
    FeatureBatch b = random_batch(tokens, heads, d, seed, v != nullptr);
    for (int h = 0; h < heads; ++h)
      for (std::int64_t t = 0; t < tokens; ++t)
        for (int c = 0; c < d; ++c) {
          const std::int64_t o = (t * heads + h) * d + c;
          q[o] = b.queries[h](t, c);
          k[o] = b.keys[h](t, c);
          if (v) v[o] = b.values[h](t, c);
        }
  });
}

// Stage (a) scalar helpers (radial.hpp:23-76, selection.hpp:33-48).
// out: [width, retained, pair_count, tier, split_factor]
int ref_frame_pair(int nf, int nt, int bs, const ref_cfg* cfg, int i, int j,
                   std::int64_t* out5) {
  return guarded([&] {
    GridSpec g = make_grid(nf, nt, bs);
    SparsityConfig c = to_cfg(cfg);
    CandidateSet cs = candidate_set(i, j, c.radial, g);
    out5[0] = cs.width;
    out5[1] = cs.retained ? 1 : 0;
    out5[2] = cs.pair_count();
    out5[3] = distance_tier(i, j, c.radial, g);
    const std::int64_t t = cs.distance;
    out5[4] = t >= 1 ? split_factor(t, c.radial, g) : 1;
  });
}

// static_select (selection.cpp:61-91): out_uv receives 2*k int64 (u, v)
// in shuffle order; *k_out the count.  cap = capacity in pairs.
int ref_static_select(int nf, int nt, int bs, const ref_cfg* cfg, int i, int j,
                      double ratio, std::uint64_t seed, std::int64_t* out_uv,
                      std::int64_t cap, std::int64_t* k_out) {
  return guarded([&] {
    GridSpec g = make_grid(nf, nt, bs);
    SparsityConfig c = to_cfg(cfg);
    CandidateSet cs = candidate_set(i, j, c.radial, g);
    auto sel = static_select(cs, ratio, seed);
    *k_out = static_cast<std::int64_t>(sel.size());
    if (static_cast<std::int64_t>(sel.size()) > cap)
      throw std::out_of_range("ref_static_select: capacity");
    for (std::size_t x = 0; x < sel.size(); ++x) {
      out_uv[2 * x] = sel[x].first;
      out_uv[2 * x + 1] = sel[x].second;
    }
  });
}

// proxy_scores + normalize_scores (selection.cpp:93-148) for one frame pair.
// scores: pair_count floats; z: pair_count doubles (may be NULL);
// stats2: {mean, stddev}.
int ref_proxy_scores(int nf, int nt, int bs, const ref_cfg* cfg, int i, int j,
                     const float* q, const float* k, std::int64_t tokens,
                     int heads, int d, float* scores, double* z,
                     double* stats2) {
  return guarded([&] {
    GridSpec g = make_grid(nf, nt, bs);
    SparsityConfig c = to_cfg(cfg);
    CandidateSet cs = candidate_set(i, j, c.radial, g);
    FeatureBatch fb = make_batch(q, k, nullptr, tokens, heads, d);
    auto s = proxy_scores(fb, i, j, cs, nt);
    std::memcpy(scores, s.data(), s.size() * sizeof(float));
    ScoreStats st;
    auto zz = normalize_scores(s, &st);
    if (z) std::memcpy(z, zz.data(), zz.size() * sizeof(double));
    if (stats2) {
      stats2[0] = st.mean;
      stats2[1] = st.stddev;
    }
  });
}

// dynamic_select (selection.cpp:150-185) on given z values.
int ref_dynamic_select(int nf, int nt, int bs, const ref_cfg* cfg, int i, int j,
                       const double* z, std::int64_t n, double tau, int fallback_k,
                       std::int64_t* out_uv, std::int64_t cap, std::int64_t* k_out) {
  return guarded([&] {
    GridSpec g = make_grid(nf, nt, bs);
    SparsityConfig c = to_cfg(cfg);
    CandidateSet cs = candidate_set(i, j, c.radial, g);
    std::vector<double> zz(z, z + n);
    auto sel = dynamic_select(cs, zz, tau, fallback_k);
    *k_out = static_cast<std::int64_t>(sel.size());
    if (static_cast<std::int64_t>(sel.size()) > cap)
      throw std::out_of_range("ref_dynamic_select: capacity");
    for (std::size_t x = 0; x < sel.size(); ++x) {
      out_uv[2 * x] = sel[x].first;
      out_uv[2 * x + 1] = sel[x].second;
    }
  });
}

// write_mask / read_mask (mask.cpp:291-376): the reference's own mask files.
// fmt: 0 binary (DRBM), 1 CSV, 2 PGM.
int ref_write_mask(const std::uint8_t* bits, std::int64_t dim, int fmt, const char* path) {
  return guarded([&] {
    BlockMask m(dim);
    std::memcpy(m.bits.data(), bits, m.bits.size());
    write_mask(m, fmt == 0 ? MaskFormat::Binary : fmt == 1 ? MaskFormat::Csv : MaskFormat::Pgm,
               path);
  });
}

// *dim_out receives S_b; bits must hold cap bytes.
int ref_read_mask(const char* path, std::uint8_t* bits, std::int64_t cap, std::int64_t* dim_out) {
  return guarded([&] {
    BlockMask m = read_mask(path);
    *dim_out = m.dim;
    if (static_cast<std::int64_t>(m.bits.size()) > cap)
      throw std::out_of_range("ref_read_mask: capacity");
    std::memcpy(bits, m.bits.data(), m.bits.size());
  });
}

// ---- the profiler's per-trial objective (profiler.cpp:49-148) --

// simulate (proxy.hpp:36-39): drift_rate < 0 selects a regime preset
// (regime = -drift_rate - 1: 0 Low, 1 Mid, 2 High).  features out:
// [total_tokens, feature_dim] row-major.
int ref_simulate(int nf, int nt, int bs, double drift_rate, int feature_dim,
                 double spatial_scale, std::uint64_t seed, float* features) {
  return guarded([&] {
    const GridSpec g = make_grid(nf, nt, bs);
    const ProxyBatch b =
        drift_rate < 0 ? simulate(static_cast<Regime>(static_cast<int>(-drift_rate) - 1), g,
                                  feature_dim, spatial_scale, seed)
                       : simulate(drift_rate, g, feature_dim, spatial_scale, seed);
    for (std::int64_t t = 0; t < g.total_tokens; ++t)
      for (int d = 0; d < feature_dim; ++d) features[t * feature_dim + d] = b.features(t, d);
  });
}

namespace {
ProxyBatch proxy_batch(int nf, int nt, int bs, const float* features, int feature_dim,
                       std::uint64_t seed) {
  ProxyBatch b;
  b.grid = make_grid(nf, nt, bs);
  b.feature_dim = feature_dim;
  b.seed = seed;
  b.features.resize(b.grid.total_tokens, feature_dim);
  for (std::int64_t t = 0; t < b.grid.total_tokens; ++t)
    for (int d = 0; d < feature_dim; ++d) b.features(t, d) = features[t * feature_dim + d];
  return b;
}
}  // namespace

// build_proxy_cache: weights [n, n] row-major (or NULL), row_sums [n],
// reference_sq_norm [1].
int ref_proxy_cache(int nf, int nt, int bs, const float* features, int feature_dim,
                    float* weights, double* row_sums, double* sq_norm) {
  return guarded([&] {
    const ProxyBatch b = proxy_batch(nf, nt, bs, features, feature_dim, 0);
    const DenseProxyCache c = build_proxy_cache(b);
    const std::int64_t n = b.grid.total_tokens;
    if (weights)
      for (std::int64_t r = 0; r < n; ++r)
        for (std::int64_t col = 0; col < n; ++col) weights[r * n + col] = c.weights(r, col);
    for (std::int64_t r = 0; r < n; ++r) row_sums[r] = c.row_sums[static_cast<std::size_t>(r)];
    *sq_norm = c.reference_sq_norm;
  });
}

// objective (with its own cache): out3 = {loss, mse, achieved_sparsity}.
int ref_objective(int nf, int nt, int bs, const ref_cfg* cfg, const float* features,
                  int feature_dim, std::uint64_t batch_seed, double penalty_weight,
                  double sparsity_target, double* out3) {
  return guarded([&] {
    const ProxyBatch b = proxy_batch(nf, nt, bs, features, feature_dim, batch_seed);
    const TrialRecord r = objective(to_cfg(cfg), b, penalty_weight, sparsity_target, nullptr);
    out3[0] = r.loss;
    out3[1] = r.mse;
    out3[2] = r.achieved_sparsity;
  });
}

}  // extern "C"
