// libradialplan_b200.so — the reference's `radialplan` C++ operator API on
// top of the B200 C ABI (include/dynrad.h, libdynrad.so).
//
// Scalar geometry (grid, octave windows, split rule, tiers) is evaluated with
// the planner's own inline formulas (csrc/plan.hpp), so the façade and the
// kernels' launch plans agree bit for bit.  Everything that touches tokens,
// pairs or features runs on the GPU through the C ABI; this file only
// marshals the reference's host containers (per-head column-major Eigen
// matrices, bit-packed host masks) to and from device buffers.
#include "radialplan_b200.hpp"

#include <cuda_runtime_api.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <fstream>
#include <memory>

#include "plan.hpp"

namespace radialplan {

// ------------------------------------------------------------ plumbing ----
namespace b200 {

void check(rp_status st) {
  if (st == RP_OK) return;
  const std::string msg = rp_last_error();
  switch (st) {
    case RP_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case RP_OUT_OF_RANGE: throw std::out_of_range(msg);
    case RP_DOMAIN_ERROR: throw std::domain_error(msg);
    case RP_CUDA_ERROR: throw std::runtime_error("cuda: " + msg);
    default: throw std::runtime_error(msg);
  }
}

rp_grid to_c(const GridSpec& g) {
  rp_grid c{};
  c.n_frames = g.n_frames;
  c.tokens_per_frame = g.tokens_per_frame;
  c.block_size = g.block_size;
  c.total_tokens = g.total_tokens;
  c.padded_tokens = g.padded_tokens;
  c.blocks_per_dim = g.blocks_per_dim;
  c.row_bytes = (g.blocks_per_dim + 7) / 8;
  return c;
}

rp_config to_c(const SparsityConfig& s) {
  rp_config c{};
  c.mode = s.mode == Mode::StaticRatio ? RP_STATIC_RATIO : RP_DYNAMIC_THRESHOLD;
  c.decay_factor = s.radial.decay_factor;
  c.long_range_factor = s.radial.long_range_factor;
  c.split_epsilon = s.radial.split_epsilon;
  c.mask_threshold = s.mask_threshold;
  c.col_threshold = s.col_threshold;
  c.near_param = s.near_param;
  c.far_param = s.far_param;
  c.fallback_k = s.fallback_k;
  return c;
}

}  // namespace b200

namespace {

using b200::check;

void cuda_ok(cudaError_t e) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("cuda: ") + cudaGetErrorString(e));
}

// Owning device allocation (the façade's marshalling buffers).
template <class T>
class DeviceArray {
 public:
  explicit DeviceArray(std::size_t n) : n_(n) {
    if (n) cuda_ok(cudaMalloc(reinterpret_cast<void**>(&p_), n * sizeof(T)));
  }
  ~DeviceArray() {
    if (p_) cudaFree(p_);
  }
  DeviceArray(const DeviceArray&) = delete;
  DeviceArray& operator=(const DeviceArray&) = delete;
  T* get() const { return p_; }
  void put(const T* h, std::size_t n) {
    cuda_ok(cudaMemcpy(p_, h, n * sizeof(T), cudaMemcpyHostToDevice));
  }
  void get_to(T* h, std::size_t n) const {
    cuda_ok(cudaMemcpy(h, p_, n * sizeof(T), cudaMemcpyDeviceToHost));
  }

 private:
  T* p_ = nullptr;
  std::size_t n_ = 0;
};

// A radial-only config for the scalar planners.
rp_config radial_cfg(const RadialParams& p) {
  SparsityConfig s;
  s.radial = p;
  return b200::to_c(s);
}

// Reference FeatureBatch (per-head column-major) -> [rows, heads, d] row-major
// f32, zero rows beyond batch.tokens.
std::vector<float> pack_heads(const std::vector<Eigen::MatrixXf>& m, std::int64_t rows,
                              int heads, int d) {
  std::vector<float> out(static_cast<std::size_t>(rows) * heads * d, 0.0f);
  for (int h = 0; h < heads; ++h) {
    const Eigen::MatrixXf& x = m[static_cast<std::size_t>(h)];
    for (Eigen::Index t = 0; t < x.rows(); ++t)
      for (int e = 0; e < d; ++e)
        out[(static_cast<std::size_t>(t) * heads + h) * d + e] = x(t, e);
  }
  return out;
}

rp_band band_of(const CandidateSet& c) {
  return rp_band{c.frame_i, c.frame_j, c.tokens_per_frame, c.width, c.retained ? 1 : 0};
}

std::vector<std::pair<std::int64_t, std::int64_t>> to_pairs(const std::vector<std::int64_t>& uv,
                                                            std::int64_t n) {
  std::vector<std::pair<std::int64_t, std::int64_t>> out;
  out.reserve(static_cast<std::size_t>(n));
  for (std::int64_t i = 0; i < n; ++i) out.emplace_back(uv[2 * i], uv[2 * i + 1]);
  return out;
}

}  // namespace

// ------------------------------------------------------------------ grid --
GridSpec make_grid(int n_frames, int tokens_per_frame, int block_size) {
  rp_grid c{};
  check(rp_make_grid(n_frames, tokens_per_frame, block_size, &c));
  GridSpec g;
  g.n_frames = c.n_frames;
  g.tokens_per_frame = c.tokens_per_frame;
  g.block_size = c.block_size;
  g.total_tokens = c.total_tokens;
  g.padded_tokens = c.padded_tokens;
  g.blocks_per_dim = c.blocks_per_dim;
  return g;
}

// ---------------------------------------------------------------- radial --
int group_index(std::int64_t t) { return rp::plan::group_index(t); }
std::int64_t base_span(std::int64_t n) { return rp::plan::base_span(n); }
double decay_length(std::int64_t t, double factor, std::int64_t base) {
  return rp::plan::decay_length(t, factor, base);
}

std::int64_t window_width(int frame_i, int frame_j, const RadialParams& p, const GridSpec& g) {
  return rp::plan::window_width(frame_i, frame_j, radial_cfg(p), b200::to_c(g));
}

std::int64_t split_factor(std::int64_t t, const RadialParams& p, const GridSpec& g) {
  return rp::plan::split_factor(t, radial_cfg(p), b200::to_c(g));
}

bool frame_retained(std::int64_t t, const RadialParams& p, const GridSpec& g) {
  return rp::plan::frame_retained(t, radial_cfg(p), b200::to_c(g));
}

std::int64_t CandidateSet::pair_count() const {
  return retained ? rp::plan::band_pairs(tokens_per_frame, width) : 0;
}
std::int64_t CandidateSet::v_lo(std::int64_t u) const { return u > width ? u - width : 0; }
std::int64_t CandidateSet::v_hi(std::int64_t u) const {
  return std::min<std::int64_t>(u + width, tokens_per_frame - 1);
}

std::vector<std::int64_t> CandidateSet::row_offsets() const {
  std::vector<std::int64_t> off(static_cast<std::size_t>(tokens_per_frame) + 1, 0);
  if (retained)
    for (std::int64_t u = 0; u < tokens_per_frame; ++u)
      off[static_cast<std::size_t>(u) + 1] = off[static_cast<std::size_t>(u)] + v_hi(u) - v_lo(u) + 1;
  return off;
}

std::pair<std::int64_t, std::int64_t> CandidateSet::pair_at(std::int64_t index) const {
  if (index < 0 || index >= pair_count())
    throw std::out_of_range("pair_at: index outside candidate set");
  const std::vector<std::int64_t> off = row_offsets();
  const std::int64_t u = (std::upper_bound(off.begin(), off.end(), index) - off.begin()) - 1;
  return {u, v_lo(u) + (index - off[static_cast<std::size_t>(u)])};
}

bool CandidateSet::contains(std::int64_t u, std::int64_t v) const {
  return retained && u >= 0 && v >= 0 && u < tokens_per_frame && v < tokens_per_frame &&
         (u > v ? u - v : v - u) <= width;
}

void CandidateSet::visit(const std::function<void(std::int64_t, std::int64_t)>& fn) const {
  if (!retained) return;
  for (std::int64_t u = 0; u < tokens_per_frame; ++u)
    for (std::int64_t v = v_lo(u), hi = v_hi(u); v <= hi; ++v) fn(u, v);
}

CandidateSet candidate_set(int frame_i, int frame_j, const RadialParams& p, const GridSpec& g) {
  CandidateSet c;
  c.frame_i = frame_i;
  c.frame_j = frame_j;
  c.distance = frame_i > frame_j ? frame_i - frame_j : frame_j - frame_i;
  c.tokens_per_frame = g.tokens_per_frame;
  c.width = window_width(frame_i, frame_j, p, g);
  c.retained = frame_retained(c.distance, p, g);
  return c;
}

double mean_candidates_per_query(const GridSpec& g, const RadialParams& p, bool ignore_split) {
  long double sum = 0.0L;
  for (std::int64_t t = 0; t < g.n_frames; ++t) {
    if (!ignore_split && !frame_retained(t, p, g)) continue;
    const std::int64_t ordered_pairs = t == 0 ? g.n_frames : 2 * (g.n_frames - t);
    const std::int64_t w = window_width(0, static_cast<int>(t), p, g);
    sum += static_cast<long double>(ordered_pairs) *
           static_cast<long double>(rp::plan::band_pairs(g.tokens_per_frame, w));
  }
  return static_cast<double>(sum / static_cast<long double>(g.total_tokens));
}

// -------------------------------------------------------------- features --
void FeatureBatch::validate(bool need_values) const {
  if (tokens < 1 || heads < 1 || head_dim < 1)
    throw std::invalid_argument("feature batch: empty dimensions");
  const auto shape_ok = [&](const std::vector<Eigen::MatrixXf>& m, const char* what) {
    if (static_cast<int>(m.size()) != heads)
      throw std::invalid_argument(std::string("feature batch: ") + what + " head count mismatch");
    for (const Eigen::MatrixXf& x : m)
      if (x.rows() != tokens || x.cols() != head_dim)
        throw std::invalid_argument(std::string("feature batch: ") + what + " shape mismatch");
  };
  shape_ok(queries, "queries");
  shape_ok(keys, "keys");
  if (need_values) shape_ok(values, "values");
}

FeatureBatch random_batch(std::int64_t tokens, int heads, int head_dim, std::uint64_t seed,
                          bool with_values) {
  FeatureBatch b;
  b.tokens = tokens;
  b.heads = heads;
  b.head_dim = head_dim;
  const auto make = [&](std::uint64_t role) {
    std::vector<Eigen::MatrixXf> out;
    for (int h = 0; h < heads; ++h) {
      Eigen::MatrixXf m(tokens, head_dim);
      const std::uint64_t key = mix64(seed, role, static_cast<std::uint64_t>(h));
      for (std::int64_t t = 0; t < tokens; ++t)
        for (int e = 0; e < head_dim; ++e)
          m(t, e) = static_cast<float>(gaussian_at(
              mix64(key, static_cast<std::uint64_t>(t), static_cast<std::uint64_t>(e))));
      out.push_back(std::move(m));
    }
    return out;
  };
  b.queries = make(1);
  b.keys = make(2);
  if (with_values) b.values = make(3);
  return b;
}

// ------------------------------------------------------------- selection --
void SparsityConfig::validate() const {
  const rp_config c = b200::to_c(*this);
  check(rp_config_validate(&c));
}

int distance_tier(int frame_i, int frame_j, const RadialParams& p, const GridSpec& g) {
  return rp::plan::distance_tier(frame_i, frame_j, radial_cfg(p), b200::to_c(g));
}

double retention_ratio(int frame_i, int frame_j, const SparsityConfig& c, const GridSpec& g) {
  const int tier = distance_tier(frame_i, frame_j, c.radial, g);
  return tier == 0 ? 1.0 : (tier == 1 ? c.near_param : c.far_param);
}

double score_threshold(int frame_i, int frame_j, const SparsityConfig& c, const GridSpec& g) {
  const int tier = distance_tier(frame_i, frame_j, c.radial, g);
  return tier == 0 ? -std::numeric_limits<double>::infinity()
                   : (tier == 1 ? c.near_param : c.far_param);
}

std::vector<std::pair<std::int64_t, std::int64_t>> static_select(const CandidateSet& cands,
                                                                 double ratio,
                                                                 std::uint64_t seed) {
  const rp_band b = band_of(cands);
  const std::int64_t n = cands.pair_count();
  const std::int64_t cap = std::max<std::int64_t>(1, n);
  DeviceArray<std::int64_t> uv(static_cast<std::size_t>(2 * cap));
  std::int64_t k = 0;
  check(rp_static_select(&b, ratio, seed, uv.get(), cap, &k, nullptr));
  std::vector<std::int64_t> h(static_cast<std::size_t>(2 * k));
  if (k) uv.get_to(h.data(), h.size());
  return to_pairs(h, k);
}

std::vector<float> proxy_scores(const FeatureBatch& f, int frame_i, int frame_j,
                                const CandidateSet& cands, std::int64_t tokens_per_frame) {
  if (f.heads < 1) throw std::invalid_argument("proxy_scores: batch has no heads");
  const std::int64_t qi = static_cast<std::int64_t>(frame_i) * tokens_per_frame;
  const std::int64_t kj = static_cast<std::int64_t>(frame_j) * tokens_per_frame;
  if (qi + tokens_per_frame > f.tokens || kj + tokens_per_frame > f.tokens)
    throw std::out_of_range("proxy_scores: frame outside feature batch");
  const std::int64_t n = cands.pair_count();
  std::vector<float> out(static_cast<std::size_t>(n));
  if (n == 0) return out;
  const std::vector<float> q = pack_heads(f.queries, f.tokens, f.heads, f.head_dim);
  const std::vector<float> k = pack_heads(f.keys, f.tokens, f.heads, f.head_dim);
  DeviceArray<float> dq(q.size()), dk(k.size()), ds(static_cast<std::size_t>(n));
  dq.put(q.data(), q.size());
  dk.put(k.data(), k.size());
  const auto dt = b200::DeviceTensor::contiguous(dq.get(), RP_F32, f.tokens, f.heads, f.head_dim);
  const auto kt = b200::DeviceTensor::contiguous(dk.get(), RP_F32, f.tokens, f.heads, f.head_dim);
  const rp_tensor tq = dt.c(), tk = kt.c();
  rp_band b = band_of(cands);
  b.tokens_per_frame = tokens_per_frame;
  check(rp_proxy_scores(&tq, &tk, f.heads, &b, ds.get(), nullptr));
  ds.get_to(out.data(), out.size());
  return out;
}

std::vector<double> normalize_scores(const std::vector<float>& scores, ScoreStats* stats) {
  const std::int64_t n = static_cast<std::int64_t>(scores.size());
  std::vector<double> z(scores.size(), 0.0);
  double mean = 0.0, sd = 0.0;
  if (n > 0) {
    DeviceArray<float> ds(scores.size());
    DeviceArray<double> dz(scores.size());
    ds.put(scores.data(), scores.size());
    check(rp_normalize_scores(ds.get(), n, dz.get(), &mean, &sd, nullptr));
    dz.get_to(z.data(), z.size());
  }
  if (stats) *stats = ScoreStats{mean, sd};
  return z;
}

std::vector<std::pair<std::int64_t, std::int64_t>> dynamic_select(
    const CandidateSet& cands, const std::vector<double>& normalized, double threshold,
    int fallback_k) {
  const std::int64_t n = cands.pair_count();
  if (static_cast<std::int64_t>(normalized.size()) != n)
    throw std::invalid_argument("dynamic_select: score count mismatch");
  if (n == 0) return {};
  const rp_band b = band_of(cands);
  DeviceArray<double> dz(normalized.size());
  dz.put(normalized.data(), normalized.size());
  DeviceArray<std::int64_t> uv(static_cast<std::size_t>(2 * n));
  std::int64_t k = 0;
  check(rp_dynamic_select(&b, dz.get(), n, threshold, fallback_k, uv.get(), n, &k, nullptr));
  std::vector<std::int64_t> h(static_cast<std::size_t>(2 * k));
  if (k) uv.get_to(h.data(), h.size());
  return to_pairs(h, k);
}

// ------------------------------------------------------------------ mask --
BlockMask::BlockMask(std::int64_t blocks_per_dim)
    : dim(blocks_per_dim),
      row_bytes((blocks_per_dim + 7) / 8),
      bits(static_cast<std::size_t>(blocks_per_dim * ((blocks_per_dim + 7) / 8)), 0) {}

void BlockMask::merge(const BlockMask& other) {
  if (other.dim != dim) throw std::invalid_argument("merge: mask dimensions differ");
  std::transform(bits.begin(), bits.end(), other.bits.begin(), bits.begin(),
                 [](std::uint8_t a, std::uint8_t b) { return static_cast<std::uint8_t>(a | b); });
}

std::int64_t BlockMask::active_count() const {
  std::int64_t n = 0;
  for (std::uint8_t b : bits) n += __builtin_popcount(b);
  return n;
}

TokenMask::TokenMask(std::int64_t tokens)
    : dim(tokens),
      row_bytes((tokens + 7) / 8),
      bits(static_cast<std::size_t>(tokens * ((tokens + 7) / 8)), 0) {}

double sparsity(const BlockMask& mask) {
  GridSpec g;  // only the block count matters to the popcount kernel
  g.n_frames = 1;
  g.block_size = 2;
  g.tokens_per_frame = static_cast<int>(2 * mask.dim);
  g.total_tokens = g.padded_tokens = 2 * mask.dim;
  g.blocks_per_dim = mask.dim;
  const rp_grid c = b200::to_c(g);
  DeviceArray<std::uint8_t> d(mask.bits.size());
  d.put(mask.bits.data(), mask.bits.size());
  std::int64_t active = 0;
  double s = 0.0;
  check(rp_mask_sparsity(&c, d.get(), &active, &s, nullptr));
  return s;
}

TokenMask expand_mask(const BlockMask& mask, const GridSpec& g) {
  if (mask.dim != g.blocks_per_dim)
    throw std::invalid_argument("expand_mask: mask does not fit grid");
  const rp_grid c = b200::to_c(g);
  TokenMask t(g.padded_tokens);
  DeviceArray<std::uint8_t> db(mask.bits.size()), dt(t.bits.size());
  db.put(mask.bits.data(), mask.bits.size());
  check(rp_expand_mask(&c, db.get(), dt.get(), nullptr));
  cuda_ok(cudaDeviceSynchronize());
  dt.get_to(t.bits.data(), t.bits.size());
  return t;
}

bool aggregate_block(const std::vector<std::pair<int, int>>& kept_in_tile, double col_threshold,
                     double mask_threshold, int block_size) {
  // The per-tile rule the mask kernels apply (mask.cpp:68-85), for callers
  // that aggregate their own pair lists: integer thresholds, exact for a
  // power-of-two B (rp::plan::count_threshold).
  std::vector<int> per_col(static_cast<std::size_t>(std::max(block_size, 0)), 0);
  for (const auto& rc : kept_in_tile) {
    if (rc.first < 0 || rc.first >= block_size || rc.second < 0 || rc.second >= block_size)
      throw std::out_of_range("aggregate_block: pair outside tile");
    ++per_col[static_cast<std::size_t>(rc.second)];
  }
  int active = 0;
  for (int x : per_col) active += static_cast<double>(x) / block_size >= col_threshold;
  return static_cast<double>(active) / block_size >= mask_threshold;
}

MaskFormat mask_format_for_path(const std::string& path) {
  const std::size_t dot = path.rfind('.');
  const std::string ext = dot == std::string::npos ? std::string() : path.substr(dot);
  if (ext == ".bin") return MaskFormat::Binary;
  if (ext == ".csv") return MaskFormat::Csv;
  if (ext == ".pgm") return MaskFormat::Pgm;
  throw std::invalid_argument("mask path needs a .bin/.csv/.pgm extension: " + path);
}

void write_mask(const BlockMask& mask, MaskFormat format, const std::string& path) {
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) throw std::runtime_error("cannot open for writing: " + path);
  if (format == MaskFormat::Binary) {
    const std::uint32_t dim = static_cast<std::uint32_t>(mask.dim);
    const unsigned char head[10] = {'D', 'R', 'B', 'M', 1, 0,
                                    static_cast<unsigned char>(dim),
                                    static_cast<unsigned char>(dim >> 8),
                                    static_cast<unsigned char>(dim >> 16),
                                    static_cast<unsigned char>(dim >> 24)};
    f.write(reinterpret_cast<const char*>(head), sizeof(head));
    f.write(reinterpret_cast<const char*>(mask.bits.data()),
            static_cast<std::streamsize>(mask.bits.size()));
  } else if (format == MaskFormat::Csv) {
    std::string text;
    for (std::int64_t r = 0; r < mask.dim; ++r)
      for (std::int64_t c = 0; c < mask.dim; ++c)
        if (mask.get(r, c)) text += std::to_string(r) + "," + std::to_string(c) + "\n";
    f.write(text.data(), static_cast<std::streamsize>(text.size()));
  } else {
    const std::string head = "P5\n" + std::to_string(mask.dim) + " " + std::to_string(mask.dim) +
                             "\n255\n";
    f.write(head.data(), static_cast<std::streamsize>(head.size()));
    std::vector<char> px(static_cast<std::size_t>(mask.dim));
    for (std::int64_t r = 0; r < mask.dim; ++r) {
      for (std::int64_t c = 0; c < mask.dim; ++c)
        px[static_cast<std::size_t>(c)] = mask.get(r, c) ? 0 : static_cast<char>(255);
      f.write(px.data(), static_cast<std::streamsize>(px.size()));
    }
  }
  if (!f) throw std::runtime_error("write failed: " + path);
}

BlockMask read_mask(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open: " + path);
  unsigned char head[10] = {};
  f.read(reinterpret_cast<char*>(head), sizeof(head));
  if (!f || std::memcmp(head, "DRBM", 4) != 0)
    throw std::runtime_error("mask file has bad magic: " + path);
  if ((head[4] | (head[5] << 8)) != 1)
    throw std::runtime_error("unsupported mask version in " + path);
  const std::uint32_t dim = head[6] | (head[7] << 8) | (static_cast<std::uint32_t>(head[8]) << 16) |
                            (static_cast<std::uint32_t>(head[9]) << 24);
  if (dim == 0 || dim > (1u << 26)) throw std::runtime_error("mask dimension out of range in " + path);
  BlockMask mask(static_cast<std::int64_t>(dim));
  f.read(reinterpret_cast<char*>(mask.bits.data()), static_cast<std::streamsize>(mask.bits.size()));
  if (f.gcount() != static_cast<std::streamsize>(mask.bits.size()))
    throw std::runtime_error("mask payload truncated: " + path);
  if (f.peek() != std::char_traits<char>::eof())
    throw std::runtime_error("mask payload has trailing bytes: " + path);
  return mask;
}

BlockMask build_mask(const GridSpec& g, const SparsityConfig& c, std::uint64_t seed,
                     const BuildOptions& opt) {
  c.validate();
  const bool dynamic = c.mode == Mode::DynamicThreshold;
  if (dynamic) {
    if (!opt.features) throw std::invalid_argument("build_mask: dynamic mode needs features");
    opt.features->validate(false);
    if (opt.features->tokens < g.total_tokens)
      throw std::invalid_argument("build_mask: feature batch too short");
  }
  const auto t0 = std::chrono::steady_clock::now();
  const rp_grid gc = b200::to_c(g);
  const rp_config cc = b200::to_c(c);
  rp_build_options bo;
  rp_build_options_defaults(&bo);
  bo.disable_split = opt.disable_split ? 1 : 0;
  BlockMask mask(g.blocks_per_dim);
  DeviceArray<std::uint8_t> dm(mask.bits.size());
  rp_build_stats st{};
  if (dynamic) {
    const FeatureBatch& f = *opt.features;
    const std::vector<float> q = pack_heads(f.queries, f.tokens, f.heads, f.head_dim);
    const std::vector<float> k = pack_heads(f.keys, f.tokens, f.heads, f.head_dim);
    DeviceArray<float> dq(q.size()), dk(k.size());
    dq.put(q.data(), q.size());
    dk.put(k.data(), k.size());
    const rp_tensor tq =
        b200::DeviceTensor::contiguous(dq.get(), RP_F32, f.tokens, f.heads, f.head_dim).c();
    const rp_tensor tk =
        b200::DeviceTensor::contiguous(dk.get(), RP_F32, f.tokens, f.heads, f.head_dim).c();
    check(rp_build_mask(&gc, &cc, seed, &bo, &tq, &tk, f.heads, dm.get(), &st, nullptr));
  } else {
    check(rp_build_mask(&gc, &cc, seed, &bo, nullptr, nullptr, 0, dm.get(), &st, nullptr));
  }
  dm.get_to(mask.bits.data(), mask.bits.size());
  if (opt.timings) {
    // The GPU build is one fused pass; its wall time is reported as the
    // selection phase.
    opt.timings->selection_s += std::chrono::duration<double>(
        std::chrono::steady_clock::now() - t0).count();
    opt.timings->retained_frame_pairs += st.retained_frame_pairs;
    opt.timings->scored_pairs += st.scored_pairs;
  }
  return mask;
}

// ------------------------------------------------------------- attention --
namespace {
// Shared body of masked_attention(_exact): block structure recovered on the
// device, then the host-buffer C entry point (exact, or soft with eps).
std::vector<Eigen::MatrixXf> attention_on_gpu(const FeatureBatch& batch, const TokenMask& mask,
                                              bool soft, double eps) {
  batch.validate(true);
  if (mask.dim < batch.tokens)
    throw std::invalid_argument("masked attention: mask smaller than batch");
  const std::int64_t n = mask.dim;
  // Recover the block structure of the token mask on the device.
  DeviceArray<std::uint8_t> dtok(mask.bits.size());
  dtok.put(mask.bits.data(), mask.bits.size());
  int bs = 0;
  std::vector<std::uint8_t> blocks;
  for (int b = 128; b >= 2 && !bs; b /= 2) {
    if (n % b) continue;
    const std::int64_t nb = n / b;
    DeviceArray<std::uint8_t> dblk(static_cast<std::size_t>(nb * ((nb + 7) / 8)));
    int uniform = 0;
    check(rp_token_mask_to_blocks(dtok.get(), n, b, dblk.get(), &uniform, nullptr));
    if (!uniform) continue;
    bs = b;
    blocks.resize(static_cast<std::size_t>(nb * ((nb + 7) / 8)));
    dblk.get_to(blocks.data(), blocks.size());
  }
  if (!bs)
    throw std::invalid_argument(
        "masked attention: token mask is not block-structured (expand_mask of a BlockMask)");
  // One "frame" of n tokens at block size bs: padded_tokens == n, and the
  // rows beyond batch.tokens are the zero padding of attention.cpp:43-48.
  const GridSpec g = make_grid(1, static_cast<int>(n), bs);
  const rp_grid gc = b200::to_c(g);
  const int H = batch.heads, d = batch.head_dim;
  const std::vector<float> q = pack_heads(batch.queries, n, H, d);
  const std::vector<float> k = pack_heads(batch.keys, n, H, d);
  const std::vector<float> v = pack_heads(batch.values, n, H, d);
  std::vector<float> o(static_cast<std::size_t>(n) * H * d);
  if (soft)
    check(rp_masked_attention_host(&gc, blocks.data(), q.data(), k.data(), v.data(), RP_F32, n, H,
                                   d, eps, o.data(), nullptr));
  else
    check(rp_masked_attention_exact_host(&gc, blocks.data(), q.data(), k.data(), v.data(),
                                         RP_F32, n, H, d, o.data(), nullptr));
  std::vector<Eigen::MatrixXf> out;
  out.reserve(static_cast<std::size_t>(H));
  for (int h = 0; h < H; ++h) {
    Eigen::MatrixXf m(n, d);
    for (std::int64_t t = 0; t < n; ++t)
      for (int e = 0; e < d; ++e) m(t, e) = o[(static_cast<std::size_t>(t) * H + h) * d + e];
    out.push_back(std::move(m));
  }
  return out;
}
}  // namespace

std::vector<Eigen::MatrixXf> masked_attention_exact(const FeatureBatch& batch,
                                                    const TokenMask& mask) {
  return attention_on_gpu(batch, mask, false, 0.0);
}

std::vector<Eigen::MatrixXf> masked_attention(const FeatureBatch& batch, const TokenMask& mask,
                                              double epsilon) {
  if (!(epsilon > 0.0))
    throw std::invalid_argument("masked attention: epsilon must be positive");
  return attention_on_gpu(batch, mask, true, epsilon);
}

// ----------------------------------------------------- B200 device API ----
namespace b200 {

Plan::Plan(const GridSpec& g, const SparsityConfig& c, std::uint64_t seed, bool disable_split,
           int score_engine)
    : g_(g) {
  const rp_grid gc = to_c(g);
  const rp_config cc = to_c(c);
  rp_build_options o;
  rp_build_options_defaults(&o);
  o.disable_split = disable_split ? 1 : 0;
  o.score_engine = score_engine;
  check(rp_plan_create(&gc, &cc, seed, &o, &p_));
}

Plan::~Plan() { rp_plan_destroy(p_); }

void Plan::build_mask(std::uint8_t* mask_bits_dev, const DeviceTensor* q, const DeviceTensor* k,
                      int n_score_heads, rp_build_stats* stats, rp_stream stream) const {
  rp_tensor tq{}, tk{};
  if (q) tq = q->c();
  if (k) tk = k->c();
  check(rp_plan_build_mask(p_, q ? &tq : nullptr, k ? &tk : nullptr, n_score_heads,
                           mask_bits_dev, stats, stream));
}

void mask_to_csr(const GridSpec& g, const std::uint8_t* mask_bits_dev, std::int32_t* row_ptr,
                 std::int32_t* col_idx, std::int64_t cap, std::int32_t* row_order,
                 std::int64_t* nnz_dev, rp_stream stream) {
  const rp_grid gc = to_c(g);
  check(rp_mask_to_csr(&gc, mask_bits_dev, row_ptr, col_idx, cap, row_order, nnz_dev, stream));
}

void sparse_attention(const GridSpec& g, const DeviceTensor& q, const DeviceTensor& k,
                      const DeviceTensor& v, DeviceTensor& o, const std::int32_t* row_ptr,
                      const std::int32_t* col_idx, const std::int32_t* row_order,
                      float softmax_scale, rp_stream stream) {
  const rp_grid gc = to_c(g);
  const rp_tensor tq = q.c(), tk = k.c(), tv = v.c();
  rp_tensor to = o.c();
  check(rp_sparse_attention_fwd(&gc, &tq, &tk, &tv, &to, row_ptr, col_idx, row_order,
                                softmax_scale, stream));
}

}  // namespace b200

// ------------------------------------------------- profiler objective (8f3) --
namespace {
// ProxyBatch::features (column-major host) -> [S, dim] row-major f32.
std::vector<float> pack_features(const ProxyBatch& b) {
  const std::int64_t n = b.features.rows();
  const int d = static_cast<int>(b.features.cols());
  if (n != b.grid.total_tokens || d != b.feature_dim || d < 1)
    throw std::invalid_argument("proxy batch: features must be total_tokens x feature_dim");
  std::vector<float> f(static_cast<std::size_t>(n) * d);
  for (std::int64_t t = 0; t < n; ++t)
    for (int k = 0; k < d; ++k) f[static_cast<std::size_t>(t) * d + k] = b.features(t, k);
  return f;
}

TrialRecord run_objective(const rp_proxy_cache* cache, const SparsityConfig& c,
                          std::uint64_t seed, const float* features_dev, int dim,
                          double penalty_weight, double sparsity_target) {
  const rp_config cc = b200::to_c(c);
  rp_trial t{};
  check(rp_objective(cache, &cc, seed, features_dev, dim, penalty_weight, sparsity_target, &t,
                     nullptr, nullptr));
  TrialRecord r;
  r.config = c;
  r.loss = t.loss;
  r.mse = t.mse;
  r.achieved_sparsity = t.achieved_sparsity;
  return r;
}
}  // namespace

FeatureBatch scoring_features(const ProxyBatch& batch, int fused_heads) {
  if (fused_heads < 1) throw std::invalid_argument("scoring_features: fused_heads must be >= 1");
  if (batch.feature_dim % fused_heads != 0)
    throw std::invalid_argument("scoring_features: feature_dim not divisible by fused_heads");
  FeatureBatch f;
  f.tokens = batch.features.rows();
  f.heads = fused_heads;
  f.head_dim = batch.feature_dim / fused_heads;
  for (int h = 0; h < fused_heads; ++h) {
    Eigen::MatrixXf slice = batch.features.middleCols(static_cast<Eigen::Index>(h) * f.head_dim,
                                                      f.head_dim);
    f.queries.push_back(slice);
    f.keys.push_back(std::move(slice));
  }
  return f;
}

DenseProxyCache build_proxy_cache(const ProxyBatch& batch) {
  const std::vector<float> f = pack_features(batch);
  const std::int64_t n = batch.grid.total_tokens;
  const rp_grid gc = b200::to_c(batch.grid);
  DeviceArray<float> df(f.size());
  df.put(f.data(), f.size());
  DeviceArray<float> dw(static_cast<std::size_t>(n * n));
  DeviceArray<double> drs(static_cast<std::size_t>(n));
  DenseProxyCache c;
  check(rp_proxy_weights(&gc, df.get(), batch.feature_dim, dw.get(), drs.get(),
                         &c.reference_sq_norm, nullptr));
  std::vector<float> w(static_cast<std::size_t>(n * n));
  dw.get_to(w.data(), w.size());
  c.row_sums.resize(static_cast<std::size_t>(n));
  drs.get_to(c.row_sums.data(), c.row_sums.size());
  c.weights = Eigen::MatrixXf(n, n);
  for (std::int64_t r = 0; r < n; ++r)
    for (std::int64_t col = 0; col < n; ++col)
      c.weights(r, col) = w[static_cast<std::size_t>(r * n + col)];
  return c;
}

TrialRecord objective(const SparsityConfig& c, const ProxyBatch& batch, double penalty_weight,
                      double sparsity_target, const DenseProxyCache* cache) {
  c.validate();
  if (!cache) {
    const b200::ProxyCache pc(batch);
    return pc.objective(c, penalty_weight, sparsity_target);
  }
  const std::vector<float> f = pack_features(batch);
  const std::int64_t n = batch.grid.total_tokens;
  if (cache->weights.rows() != n || cache->weights.cols() != n ||
      static_cast<std::int64_t>(cache->row_sums.size()) != n)
    throw std::invalid_argument("objective: cache does not match the batch");
  std::vector<float> w(static_cast<std::size_t>(n * n));
  for (std::int64_t r = 0; r < n; ++r)
    for (std::int64_t col = 0; col < n; ++col)
      w[static_cast<std::size_t>(r * n + col)] = cache->weights(r, col);
  DeviceArray<float> dw(w.size()), df(f.size());
  DeviceArray<double> drs(static_cast<std::size_t>(n));
  dw.put(w.data(), w.size());
  df.put(f.data(), f.size());
  drs.put(cache->row_sums.data(), cache->row_sums.size());
  const rp_grid gc = b200::to_c(batch.grid);
  rp_proxy_cache* pc = nullptr;
  check(rp_proxy_cache_from_weights(&gc, dw.get(), drs.get(), cache->reference_sq_norm, &pc,
                                    nullptr));
  try {
    const TrialRecord r = run_objective(pc, c, batch.seed, df.get(), batch.feature_dim,
                                        penalty_weight, sparsity_target);
    rp_proxy_cache_destroy(pc);
    return r;
  } catch (...) {
    rp_proxy_cache_destroy(pc);
    throw;
  }
}

namespace b200 {
ProxyCache::ProxyCache(const ProxyBatch& batch)
    : g_(batch.grid), seed_(batch.seed), dim_(batch.feature_dim) {
  const std::vector<float> f = pack_features(batch);
  cuda_ok(cudaMalloc(reinterpret_cast<void**>(&features_), f.size() * sizeof(float)));
  cuda_ok(cudaMemcpy(features_, f.data(), f.size() * sizeof(float), cudaMemcpyHostToDevice));
  const rp_grid gc = to_c(g_);
  const rp_status st = rp_proxy_cache_create(&gc, features_, dim_, &cache_, nullptr);
  if (st != RP_OK) {
    cudaFree(features_);
    check(st);
  }
}

ProxyCache::~ProxyCache() {
  rp_proxy_cache_destroy(cache_);
  if (features_) cudaFree(features_);
}

TrialRecord ProxyCache::objective(const SparsityConfig& c, double penalty_weight,
                                  double sparsity_target) const {
  c.validate();
  return run_objective(cache_, c, seed_, features_, dim_, penalty_weight, sparsity_target);
}
}  // namespace b200

}  // namespace radialplan
