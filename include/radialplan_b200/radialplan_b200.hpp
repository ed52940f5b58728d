// radialplan_b200.hpp — C++ façade of the B200-native DynamicRad hot path.
//
// Drop-in for the reference's C++ operator API (arxiv/paper_2604_20470,
// proj/include/radialplan/*.hpp): the same namespace `radialplan`, the same
// type names and fields, the same free-function signatures and the same
// exception types and messages.  A reference caller switches by putting
// include/radialplan_b200 on its include path instead of the reference's
// include/ (the thin radialplan/{grid,radial,selection,mask,attention,rng}.hpp
// forwarders there all land here) and linking libradialplan_b200.so instead
// of libradialplan.a.
//
// Every data-path operation is executed by the CUDA kernels of libdynrad.so
// through the C ABI (include/dynrad.h); there is no CPU fallback — without a
// CUDA device those calls throw std::runtime_error("cuda: ...").  Scalar
// helpers of stage (a) (window widths, split factors, tiers, ...) are O(1)
// host formulas evaluated by the same library code that plans the kernels.
//
// Beyond the reference signatures, namespace radialplan::b200 adds the
// device-resident API a B200 caller uses per layer: a cached Plan, bf16 /
// f32 device tensor views, block-sparse row lists and the tcgen05 sparse
// attention forward on device pointers.
#pragma once

#include <Eigen/Dense>

#include <cmath>
#include <cstdint>
#include <functional>
#include <numbers>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "dynrad.h"

namespace radialplan {

// ======================================================= rng (rng.hpp) ====
// The pinned splitmix64 contract (reference rng.hpp:19-91); also compiled
// into the kernels (csrc/common.cuh), so host and device agree bit for bit.
inline constexpr std::uint64_t kSplitMixGamma = 0x9E3779B97F4A7C15ull;

inline std::uint64_t mix64(std::uint64_t z) {
  z += kSplitMixGamma;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
inline std::uint64_t mix64(std::uint64_t a, std::uint64_t b) { return mix64(mix64(a) ^ b); }
inline std::uint64_t mix64(std::uint64_t a, std::uint64_t b, std::uint64_t c) {
  return mix64(mix64(a, b) ^ c);
}
inline std::uint64_t mix64(std::uint64_t a, std::uint64_t b, std::uint64_t c,
                           std::uint64_t d) {
  return mix64(mix64(a, b, c) ^ d);
}

class SplitMix64 {
 public:
  explicit SplitMix64(std::uint64_t seed) : s_(seed) {}
  // call c (0-based) of the stream equals mix64(seed + c * gamma)
  std::uint64_t next() { return mix64((s_ += kSplitMixGamma) - kSplitMixGamma); }
  std::uint64_t bounded(std::uint64_t n) { return next() % n; }
  double u01_open() { return static_cast<double>((next() >> 11) + 1) * 0x1.0p-53; }
  double u01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double gaussian() {
    const double a = u01_open();
    const double b = u01();
    return std::sqrt(-2.0 * std::log(a)) * std::cos(2.0 * std::numbers::pi * b);
  }

 private:
  std::uint64_t s_;
};

inline double gaussian_at(std::uint64_t key) {
  const double a =
      static_cast<double>((mix64(key ^ 0x8D5CF3D2A3B1E601ull) >> 11) + 1) * 0x1.0p-53;
  const double b = static_cast<double>(mix64(key ^ 0xC2B2AE3D27D4EB4Full) >> 11) * 0x1.0p-53;
  return std::sqrt(-2.0 * std::log(a)) * std::cos(2.0 * std::numbers::pi * b);
}

// ===================================================== grid (grid.hpp) ====
struct GridSpec {
  int n_frames = 0;
  int tokens_per_frame = 0;
  int block_size = 0;
  std::int64_t total_tokens = 0;    // S  = n_frames * tokens_per_frame
  std::int64_t padded_tokens = 0;   // S' = S rounded up to block_size
  std::int64_t blocks_per_dim = 0;  // S_b = S' / block_size
};

// Validated by rp_make_grid (same messages as the reference).
GridSpec make_grid(int n_frames, int tokens_per_frame, int block_size);

inline std::int64_t block_of(std::int64_t token, const GridSpec& g) {
  if (token < 0 || token >= g.padded_tokens)
    throw std::out_of_range("block_of: token outside padded range");
  return token / g.block_size;
}
// Padding tokens belong to the last frame.
inline int frame_of(std::int64_t token, const GridSpec& g) {
  if (token < 0 || token >= g.padded_tokens)
    throw std::out_of_range("frame_of: token outside padded range");
  return token >= g.total_tokens ? g.n_frames - 1
                                 : static_cast<int>(token / g.tokens_per_frame);
}

// ================================================= radial (radial.hpp) ====
struct RadialParams {
  double decay_factor = 1.0;       // gamma: window decay length scale
  double long_range_factor = 1.0;  // lambda: split decay length scale
  double split_epsilon = 1e-6;     // guards the split divisor
};

int group_index(std::int64_t t);
std::int64_t base_span(std::int64_t tokens_per_frame);
double decay_length(std::int64_t t, double factor, std::int64_t base);
std::int64_t window_width(int frame_i, int frame_j, const RadialParams& p, const GridSpec& g);
std::int64_t split_factor(std::int64_t t, const RadialParams& p, const GridSpec& g);
bool frame_retained(std::int64_t t, const RadialParams& p, const GridSpec& g);

// The lazy band |u - v| <= width over local in-frame indices of one ordered
// frame pair; canonical row-major order.
struct CandidateSet {
  int frame_i = 0;
  int frame_j = 0;
  std::int64_t distance = 0;
  std::int64_t tokens_per_frame = 0;
  std::int64_t width = 0;
  bool retained = false;

  std::int64_t pair_count() const;
  std::int64_t v_lo(std::int64_t u) const;
  std::int64_t v_hi(std::int64_t u) const;
  std::pair<std::int64_t, std::int64_t> pair_at(std::int64_t index) const;
  std::vector<std::int64_t> row_offsets() const;
  bool contains(std::int64_t u, std::int64_t v) const;
  void visit(const std::function<void(std::int64_t, std::int64_t)>& fn) const;
};

CandidateSet candidate_set(int frame_i, int frame_j, const RadialParams& p, const GridSpec& g);
double mean_candidates_per_query(const GridSpec& g, const RadialParams& p, bool ignore_split);

// ============================================ features (attention.hpp) ====
// Per-head column-major float matrices [tokens x head_dim], as the reference
// carries them; the façade packs them into the kernels' [S, H, d] layout.
struct FeatureBatch {
  std::int64_t tokens = 0;
  int heads = 0;
  int head_dim = 0;
  std::vector<Eigen::MatrixXf> queries;
  std::vector<Eigen::MatrixXf> keys;
  std::vector<Eigen::MatrixXf> values;
  void validate(bool need_values) const;
};

// Counter-based synthetic batch: value(t, d) of role r (1 Q, 2 K, 3 V) and
// head h is gaussian_at(mix64(mix64(seed, r, h), t, d)).
FeatureBatch random_batch(std::int64_t tokens, int heads, int head_dim, std::uint64_t seed,
                          bool with_values = true);

// ============================================= selection (selection.hpp) ==
enum class Mode { StaticRatio, DynamicThreshold };

struct SparsityConfig {
  Mode mode = Mode::StaticRatio;
  RadialParams radial;
  double mask_threshold = 0.75;  // theta_m
  double col_threshold = 0.20;   // theta_c
  double near_param = 0.25;      // rho1 (static) or tau1 (dynamic)
  double far_param = 0.55;       // rho2 or tau2
  int fallback_k = 1;
  void validate() const;
};

int distance_tier(int frame_i, int frame_j, const RadialParams& p, const GridSpec& g);
double retention_ratio(int frame_i, int frame_j, const SparsityConfig& c, const GridSpec& g);
double score_threshold(int frame_i, int frame_j, const SparsityConfig& c, const GridSpec& g);

inline std::uint64_t pair_seed(std::uint64_t seed, int frame_i, int frame_j) {
  return mix64(seed, static_cast<std::uint64_t>(frame_i), static_cast<std::uint64_t>(frame_j));
}

// Per-frame-pair selection operators (the building blocks build_mask runs
// fused on the GPU), each executed by its own CUDA kernel here.
std::vector<std::pair<std::int64_t, std::int64_t>> static_select(const CandidateSet& cands,
                                                                 double ratio,
                                                                 std::uint64_t seed);
std::vector<float> proxy_scores(const FeatureBatch& features, int frame_i, int frame_j,
                                const CandidateSet& cands, std::int64_t tokens_per_frame);

struct ScoreStats {
  double mean = 0.0;
  double stddev = 0.0;  // population
};
std::vector<double> normalize_scores(const std::vector<float>& scores,
                                     ScoreStats* stats = nullptr);
std::vector<std::pair<std::int64_t, std::int64_t>> dynamic_select(
    const CandidateSet& cands, const std::vector<double>& normalized, double threshold,
    int fallback_k = 1);

// ======================================================= mask (mask.hpp) ==
// Bit-packed S_b x S_b block mask: row-major, LSB-first, ceil(S_b/8) bytes
// per row — byte-identical to the reference and to the device mask.
struct BlockMask {
  std::int64_t dim = 0;
  std::int64_t row_bytes = 0;
  std::vector<std::uint8_t> bits;

  BlockMask() = default;
  explicit BlockMask(std::int64_t blocks_per_dim);
  bool get(std::int64_t row, std::int64_t col) const {
    return (bits[row * row_bytes + col / 8] >> (col % 8)) & 1u;
  }
  void set(std::int64_t row, std::int64_t col) {
    bits[row * row_bytes + col / 8] |= static_cast<std::uint8_t>(1u << (col % 8));
  }
  void merge(const BlockMask& other);
  std::int64_t active_count() const;
  bool operator==(const BlockMask&) const = default;
};

struct TokenMask {
  std::int64_t dim = 0;
  std::int64_t row_bytes = 0;
  std::vector<std::uint8_t> bits;

  TokenMask() = default;
  explicit TokenMask(std::int64_t tokens);
  bool get(std::int64_t row, std::int64_t col) const {
    return (bits[row * row_bytes + col / 8] >> (col % 8)) & 1u;
  }
  void set(std::int64_t row, std::int64_t col) {
    bits[row * row_bytes + col / 8] |= static_cast<std::uint8_t>(1u << (col % 8));
  }
};

double sparsity(const BlockMask& mask);
TokenMask expand_mask(const BlockMask& mask, const GridSpec& g);
bool aggregate_block(const std::vector<std::pair<int, int>>& kept_in_tile, double col_threshold,
                     double mask_threshold, int block_size);

struct BuildTimings {
  double candidates_s = 0.0;
  double selection_s = 0.0;
  double aggregation_s = 0.0;
  std::int64_t retained_frame_pairs = 0;
  std::int64_t scored_pairs = 0;
};

struct BuildOptions {
  bool disable_split = false;
  BuildTimings* timings = nullptr;
  const FeatureBatch* features = nullptr;  // dynamic mode
};

// Mask files (mask.hpp:93-101): DRBM binary, CSV of active (row, col), PGM
// image -- host-side file I/O, byte-compatible with the reference's.
enum class MaskFormat { Binary, Csv, Pgm };
MaskFormat mask_format_for_path(const std::string& path);
void write_mask(const BlockMask& mask, MaskFormat format, const std::string& path);
BlockMask read_mask(const std::string& path);

// Algorithm 1 on the GPU (stages a-c), returned as a host mask.
BlockMask build_mask(const GridSpec& g, const SparsityConfig& c, std::uint64_t seed,
                     const BuildOptions& opt = {});

// ==================================================== attention (exact) ===
// masked_attention_exact on the GPU (fp32 logits, fp64 softmax: within 1e-5
// of the reference).  The TokenMask must be block-structured (as produced by
// expand_mask); its block size is recovered on the device.  Returns per-head
// [S' x head_dim] matrices (padding rows included).  Throws
// std::domain_error when a row has no active key.
std::vector<Eigen::MatrixXf> masked_attention_exact(const FeatureBatch& batch,
                                                    const TokenMask& mask);

// masked_attention (attention.hpp:32-39, attention.cpp:59-81, 107-113): soft
// mask, logits + log(mask + epsilon) (log1p(eps) on active blocks, log(eps)
// elsewhere), on the GPU with the same precision as masked_attention_exact.
// Throws std::invalid_argument unless epsilon > 0.
std::vector<Eigen::MatrixXf> masked_attention(const FeatureBatch& batch, const TokenMask& mask,
                                              double epsilon = 1e-10);

// ====================== profiler objective (profiler.hpp / proxy.hpp subset) ==
// SURVEY 8f3.  Only the per-trial objective and its dense cache are on the
// B200 path; the simulator, TPE search and LUT I/O stay out of scope.
// proxy.hpp:26-33
struct ProxyBatch {
  GridSpec grid;
  int feature_dim = 0;
  double spatial_scale = 0.0;
  double drift_rate = 0.0;
  std::uint64_t seed = 0;
  Eigen::MatrixXf features;  // total_tokens x feature_dim
};

// proxy.hpp:69: the features split into fused heads (q = k).
FeatureBatch scoring_features(const ProxyBatch& batch, int fused_heads = 1);

// profiler.hpp:43-49.
struct TrialRecord {
  int trial_index = 0;
  SparsityConfig config;
  double loss = 0.0;
  double mse = 0.0;
  double achieved_sparsity = 0.0;
};

// profiler.hpp:53-58.
struct DenseProxyCache {
  Eigen::MatrixXf weights;  // exp(logits - row max)
  std::vector<double> row_sums;
  double reference_sq_norm = 0.0;
};

// build_proxy_cache (profiler.cpp:49-78) on the GPU; returns the reference's
// host layout (S x S weights).
DenseProxyCache build_proxy_cache(const ProxyBatch& batch);

// objective (profiler.hpp:68-76, profiler.cpp:80-148) on the GPU.  With a
// cache, its weights are uploaded and reduced to block statistics; without,
// the statistics are built on the device from the features.
TrialRecord objective(const SparsityConfig& c, const ProxyBatch& batch, double penalty_weight,
                      double sparsity_target, const DenseProxyCache* cache = nullptr);

// ======================================= B200 device API (beyond the ref) ==
namespace b200 {

// Throws the reference exception type matching an rp_status.
void check(rp_status st);

// A [tokens, heads, head_dim] device view (element strides).
struct DeviceTensor {
  void* data = nullptr;
  rp_dtype dtype = RP_BF16;
  std::int64_t tokens = 0;
  int heads = 0;
  int head_dim = 0;
  std::int64_t token_stride = 0;
  std::int64_t head_stride = 0;
  static DeviceTensor contiguous(void* data, rp_dtype dt, std::int64_t tokens, int heads,
                                 int head_dim) {
    return {data, dt, tokens, heads, head_dim, static_cast<std::int64_t>(heads) * head_dim,
            head_dim};
  }
  rp_tensor c() const {
    return {data, static_cast<int>(dtype), tokens, heads, head_dim, token_stride, head_stride};
  }
};

rp_grid to_c(const GridSpec& g);
rp_config to_c(const SparsityConfig& c);

// Cached per (grid, config, seed, options): static masks are built once.
class Plan {
 public:
  Plan(const GridSpec& g, const SparsityConfig& c, std::uint64_t seed, bool disable_split = false,
       int score_engine = 0);
  ~Plan();
  Plan(const Plan&) = delete;
  Plan& operator=(const Plan&) = delete;
  // mask_bits_dev: S_b * ceil(S_b/8) device bytes; q/k: scoring features
  // (first n_score_heads heads), dynamic mode only.
  void build_mask(std::uint8_t* mask_bits_dev, const DeviceTensor* q, const DeviceTensor* k,
                  int n_score_heads, rp_build_stats* stats, rp_stream stream) const;
  const GridSpec& grid() const { return g_; }

 private:
  GridSpec g_;
  rp_plan p_ = nullptr;
};

// Bit-packed device mask -> row lists (row_ptr[S_b+1], col_idx[cap],
// row_order[S_b] LPT order); nnz written to nnz_dev.
void mask_to_csr(const GridSpec& g, const std::uint8_t* mask_bits_dev, std::int32_t* row_ptr,
                 std::int32_t* col_idx, std::int64_t cap, std::int32_t* row_order,
                 std::int64_t* nnz_dev, rp_stream stream);

// Block-sparse attention forward (bf16: tcgen05 kernel; f32: exact path).
void sparse_attention(const GridSpec& g, const DeviceTensor& q, const DeviceTensor& k,
                      const DeviceTensor& v, DeviceTensor& o, const std::int32_t* row_ptr,
                      const std::int32_t* col_idx, const std::int32_t* row_order,
                      float softmax_scale, rp_stream stream);

// Device-resident proxy cache for a search loop: built once per batch
// (block statistics, S x ceil(S/B) x 16 bytes), reused by every trial.
class ProxyCache {
 public:
  explicit ProxyCache(const ProxyBatch& batch);
  ~ProxyCache();
  ProxyCache(const ProxyCache&) = delete;
  ProxyCache& operator=(const ProxyCache&) = delete;
  TrialRecord objective(const SparsityConfig& c, double penalty_weight,
                        double sparsity_target) const;

 private:
  GridSpec g_;
  std::uint64_t seed_ = 0;
  int dim_ = 0;
  float* features_ = nullptr;  // device [S, dim]
  rp_proxy_cache* cache_ = nullptr;
};

}  // namespace b200
}  // namespace radialplan
