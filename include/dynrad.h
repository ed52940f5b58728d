/* dynrad.h — C ABI of the B200-native DynamicRad sparse-attention hot path.
 *
 * This is the drop-in boundary.  The reference (arxiv/paper_2604_20470,
 * `radialplan`) exposes the path as a C++ library API in namespace
 * radialplan (proj/include/radialplan/ headers); it has no extern "C" layer.
 * Each entry point below names the reference interface it replaces.  The C++
 * facade in include/radialplan_b200/radialplan_b200.hpp re-exposes the reference
 * signatures on top of these calls, and INTEGRATION.md shows the bindings.
 *
 * Conventions
 *  - Device buffers are caller-allocated and stream-ordered; every call that
 *    takes a cudaStream_t only enqueues work unless documented otherwise.
 *  - Errors: an rp_status whose codes map 1:1 onto the reference's exception
 *    types, with the reference's message text available from
 *    rp_last_error() (thread-local).  There is no CPU fallback: without a
 *    CUDA device every compute entry point returns RP_CUDA_ERROR.
 *  - Bit-packed block masks use the reference layout (mask.hpp:13-35):
 *    row-major, LSB-first, row_bytes = ceil(S_b / 8).
 */
#ifndef DYNRAD_H
#define DYNRAD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* rp_stream; /* == cudaStream_t */

typedef enum {
  RP_OK = 0,
  RP_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  RP_OUT_OF_RANGE = 2,     /* std::out_of_range */
  RP_DOMAIN_ERROR = 3,     /* std::domain_error */
  RP_RUNTIME_ERROR = 4,    /* std::runtime_error */
  RP_CUDA_ERROR = 5        /* CUDA failure / no device (no CPU fallback) */
} rp_status;

/* Thread-local message of the last failing call on this thread. */
const char* rp_last_error(void);
/* Library version string. */
const char* rp_version(void);

/* ------------------------------------------------------------------ grid --
 * radialplan::GridSpec / make_grid (grid.hpp:13-42). */
typedef struct {
  int n_frames;
  int tokens_per_frame;
  int block_size;
  int64_t total_tokens;   /* S  = n_frames * tokens_per_frame */
  int64_t padded_tokens;  /* S' = ceil(S / B) * B */
  int64_t blocks_per_dim; /* S_b = S' / B */
  int64_t row_bytes;      /* ceil(S_b / 8) */
} rp_grid;

rp_status rp_make_grid(int n_frames, int tokens_per_frame, int block_size,
                       rp_grid* out);

/* --------------------------------------------------------------- config --
 * radialplan::SparsityConfig + RadialParams (selection.hpp:19-29,
 * radial.hpp:16-20); defaults as in the reference. */
typedef enum { RP_STATIC_RATIO = 0, RP_DYNAMIC_THRESHOLD = 1 } rp_mode;

typedef struct {
  int mode;                 /* rp_mode */
  double decay_factor;      /* gamma */
  double long_range_factor; /* lambda */
  double split_epsilon;
  double mask_threshold; /* theta_m */
  double col_threshold;  /* theta_c */
  double near_param;     /* rho1 or tau1 */
  double far_param;      /* rho2 or tau2 */
  int fallback_k;
} rp_config;

void rp_config_defaults(rp_config* c);
/* SparsityConfig::validate (selection.cpp:11-32). */
rp_status rp_config_validate(const rp_config* c);

/* Per ordered frame pair scalars: window_width, frame_retained, pair_count,
 * distance_tier, split_factor (radial.cpp:30-121, selection.cpp:34-59). */
typedef struct {
  int64_t width;
  int retained;
  int64_t pair_count;
  int tier;
  int64_t split_factor;
  double retention_or_threshold; /* retention_ratio or score_threshold */
} rp_frame_pair;
rp_status rp_frame_pair_info(const rp_grid* g, const rp_config* c, int frame_i,
                             int frame_j, rp_frame_pair* out);

/* ---------------------------------------------------------------- tensors --
 * A [tokens, heads, head_dim] view; strides in elements.  The reference's
 * FeatureBatch holds one column-major matrix per head (attention.hpp:18-27);
 * the facade packs those into this layout. */
typedef enum { RP_F32 = 0, RP_BF16 = 1 } rp_dtype;

typedef struct {
  void* data; /* device pointer */
  int dtype;  /* rp_dtype */
  int64_t tokens;
  int heads;
  int head_dim;
  int64_t token_stride; /* elements between consecutive tokens */
  int64_t head_stride;  /* elements between consecutive heads */
} rp_tensor;

/* random_batch (attention.hpp:62-63, attention.cpp:182-204) on the device:
 * the reference's counter-based synthetic features.  Writes heads
 * [first_head, first_head + heads) of the reference's batch into q / k / v
 * (each may be NULL; [tokens, heads, head_dim] f32 or bf16 -- bf16 is the
 * round-to-nearest-even of the reference's float).  head_dim % 8 == 0. */
rp_status rp_random_batch(int64_t tokens, int heads, int head_dim, uint64_t seed,
                          int first_head, rp_tensor* q, rp_tensor* k, rp_tensor* v,
                          rp_stream stream);

/* ------------------------------------------------------------ mask build --
 * radialplan::build_mask (mask.hpp:88-89, mask.cpp:162-289): stages (a)
 * candidates, (b) proxy scoring, (c) selection + theta_c/theta_m block
 * aggregation, OR-merged into a bit-packed S_b x S_b mask.
 *
 * A plan caches everything that depends only on (grid, config, seed,
 * options): the frame-pair job table, the content-independent base mask
 * (intra-frame rectangles + full bands), and in static mode the whole mask.
 * Static masks are built once (first call) and re-emitted from the cache,
 * matching the paper's precomputed static masks. */
typedef struct rp_plan_s* rp_plan;

typedef struct {
  int disable_split; /* BuildOptions::disable_split (mask.hpp:77-81) */
  /* Dynamic mode scoring engine: 0 = auto, 1 = tensor-core scores with an
   * exact fp64 recheck of every pair within `recheck_delta` of its
   * threshold, 2 = exact fp64 SIMT scores + sequential per-pair statistics
   * (bit-identical to the reference; for small grids and fp32 features). */
  int score_engine;
  double recheck_delta; /* in z units; <= 0 selects the default (1e-5) */
  /* Multi-GPU split of the dynamic scoring (SURVEY 8e option 2): only the
   * scored frame pairs whose ordinal (row-major over (i, j)) is congruent to
   * shard_index mod shard_count are scored; the intra-frame rectangles and
   * full bands are set on every shard, so the bitwise OR of all shards'
   * masks is the unsharded mask.  Ignored in static mode.  Defaults 0 / 1. */
  int shard_index;
  int shard_count;
} rp_build_options;

typedef struct {
  int64_t retained_frame_pairs; /* BuildTimings::retained_frame_pairs */
  int64_t scored_pairs;         /* BuildTimings::scored_pairs */
  int64_t sampled_pairs;        /* static: Fisher-Yates draws */
  int64_t rechecked_pairs;      /* dynamic fast engine: fp64 rechecks */
  int64_t fallback_frame_pairs; /* dynamic: pairs that used fallback_k */
  int64_t active_blocks;        /* popcount of the mask */
} rp_build_stats;

void rp_build_options_defaults(rp_build_options* o);
rp_status rp_plan_create(const rp_grid* g, const rp_config* c, uint64_t seed,
                         const rp_build_options* opt, rp_plan* out);
void rp_plan_destroy(rp_plan p);

/* Build the mask for one layer into mask_bits_dev (S_b * row_bytes bytes,
 * device).  q/k: the scoring features (the first n_score_heads heads of the
 * layer's Q/K are used, H_f in the paper; FeatureBatch::heads in the
 * reference); required in dynamic mode, ignored (may be NULL) in static
 * mode.  stats may be NULL; filling it synchronizes the stream. */
rp_status rp_plan_build_mask(rp_plan p, const rp_tensor* q, const rp_tensor* k,
                             int n_score_heads, uint8_t* mask_bits_dev,
                             rp_build_stats* stats, rp_stream stream);

/* One-shot convenience: plan + build + destroy, synchronous. */
rp_status rp_build_mask(const rp_grid* g, const rp_config* c, uint64_t seed,
                        const rp_build_options* opt, const rp_tensor* q,
                        const rp_tensor* k, int n_score_heads,
                        uint8_t* mask_bits_dev, rp_build_stats* stats,
                        rp_stream stream);

/* ------------------------------------- per-frame-pair selection operators --
 * The building blocks build_mask runs fused, exposed one by one with the
 * reference's semantics (selection.hpp:60-82) for callers that drive the
 * selection themselves.  A band is one ordered frame pair's candidate set
 * (radial.hpp:50-73: |u - v| <= width over local in-frame indices, empty
 * when not retained).  Pair lists are int64 (u, v) pairs in the reference's
 * output order.  These are synchronous (they return counts to the host). */
typedef struct {
  int frame_i;
  int frame_j;
  int64_t tokens_per_frame;
  int64_t width;
  int retained;
} rp_band;

/* static_select (selection.cpp:61-91): partial Fisher-Yates of
 * k = max(1, floor(n * ratio)) flat indices with SplitMix64(pair_seed(seed,
 * i, j)), in slot order.  uv_dev holds cap pairs; *count = k (0 if the band
 * is empty).  RP_INVALID_ARGUMENT for ratio outside (0, 1]. */
rp_status rp_static_select(const rp_band* band, double ratio, uint64_t seed, int64_t* uv_dev,
                           int64_t cap, int64_t* count, rp_stream stream);

/* proxy_scores (selection.cpp:93-123): s(u,v) = float(sum_h dot_h(q_u, k_v)
 * / sqrt(d) / H) over the first n_heads heads, fp64 accumulation in the
 * reference's order (bit-identical); scores_dev holds pair_count floats in
 * canonical row-major band order. */
rp_status rp_proxy_scores(const rp_tensor* q, const rp_tensor* k, int n_heads,
                          const rp_band* band, float* scores_dev, rp_stream stream);

/* normalize_scores (selection.cpp:125-148): sequential population mean /
 * stddev in fp64 (bit-identical) and z = (s - mean) / (stddev + 1e-8).
 * n = 0 gives mean = stddev = 0.  mean/stddev are host outputs (may be
 * NULL). */
rp_status rp_normalize_scores(const float* scores_dev, int64_t n, double* z_dev, double* mean,
                              double* stddev, rp_stream stream);

/* dynamic_select (selection.cpp:150-185): pairs with z >= threshold in flat
 * order; if none, the fallback_k best z (ties to the lower flat index) in
 * ascending flat order.  n must equal the band's pair count. */
rp_status rp_dynamic_select(const rp_band* band, const double* z_dev, int64_t n,
                            double threshold, int fallback_k, int64_t* uv_dev, int64_t cap,
                            int64_t* count, rp_stream stream);

/* Token-level mask (dim x ceil(dim/8) bytes, the reference's TokenMask
 * layout) -> block mask at block_size B (dim % B == 0): the block bit of
 * every B x B block; *uniform = 1 iff every block is constant (the token
 * mask is an expand_mask of the result).  Synchronous. */
rp_status rp_token_mask_to_blocks(const uint8_t* token_bits_dev, int64_t dim, int block_size,
                                  uint8_t* block_bits_dev, int* uniform, rp_stream stream);

/* --------------------------------------------- pooled block selector --
 * the north star's stages (b)/(c) as it words them -- NOT the
 * reference's semantics (the reference scores every token pair of the radial
 * band, selection.cpp:93-185; that is rp_build_mask).  Its oracle is a CPU
 * restatement in the tests; parity against the reference is not defined.
 *   candidates: blocks meeting the radial band |u - v| <= w(i, j) of a
 *     retained frame pair at distance >= 2 (window / split of `c`); blocks
 *     holding pairs at distance <= 1 are always kept (the reference's tier 0);
 *   (b) block means of the first n_score_heads heads of Q and K (HBM-bound),
 *     block scores Qp_r . Kp_c / sqrt(d) / n_score_heads;
 *   (c) per block row: RP_POOLED_TOPK keeps the max(1, floor(param * n)) best
 *     candidates; RP_POOLED_MASS keeps the smallest best-first prefix whose
 *     softmax mass over the row's candidates reaches param; ties go to the
 *     lower column.
 * bf16 features, n_score_heads * head_dim <= 512.  Writes the bit-packed
 * mask (reference layout). */
typedef enum { RP_POOLED_TOPK = 0, RP_POOLED_MASS = 1 } rp_pooled_mode;
rp_status rp_pooled_select(const rp_grid* g, const rp_config* c, const rp_tensor* q,
                           const rp_tensor* k, int n_score_heads, int mode, double param,
                           uint8_t* mask_bits_dev, rp_stream stream);

/* -------------------------------------------------------- mask utilities --
 * Block-sparse row lists (new; the reference stops at the bitmask):
 * row_ptr[S_b+1], col_idx[col_cap] (ascending per row), row_order[S_b]
 * (rows by descending nnz, ties by index; may be NULL), nnz_dev[1] (may be
 * NULL).  Fails with RP_OUT_OF_RANGE (reported asynchronously through
 * nnz > col_cap) if the mask has more active blocks than col_cap. */
rp_status rp_mask_to_csr(const rp_grid* g, const uint8_t* mask_bits_dev,
                         int32_t* row_ptr_dev, int32_t* col_idx_dev,
                         int64_t col_cap, int32_t* row_order_dev,
                         int64_t* nnz_dev, rp_stream stream);

/* expand_mask (mask.cpp:52-66): token-level bits, S' x ceil(S'/8) bytes. */
rp_status rp_expand_mask(const rp_grid* g, const uint8_t* mask_bits_dev,
                         uint8_t* token_bits_dev, rp_stream stream);

/* sparsity (mask.cpp:47-50) and active-block count; synchronous. */
rp_status rp_mask_sparsity(const rp_grid* g, const uint8_t* mask_bits_dev,
                           int64_t* active_blocks, double* sparsity,
                           rp_stream stream);

/* ------------------------------------------------------ sparse attention --
 * masked_attention_exact (attention.hpp:43-44, attention.cpp:50-121): per
 * head, O = softmax(Q K^T * scale restricted to active blocks) V over the
 * padded token axis.  Padding rows of Q/K/V (tokens >= S) are zeros and
 * take part as keys whenever their block is active (attention.cpp:43-48).
 * o: [S', heads, head_dim], same dtype as q.
 *   bf16: tcgen05/TMEM/TMA block-sparse flash forward (requires B = 128 and
 *         head_dim in {64, 128}); fp32 softmax.
 *   f32 : exact-precision path (fp32 logits, fp64 softmax), any B.
 * softmax_scale <= 0 selects 1/sqrt(head_dim).  row_order may be NULL. */
rp_status rp_sparse_attention_fwd(const rp_grid* g, const rp_tensor* q,
                                  const rp_tensor* k, const rp_tensor* v,
                                  rp_tensor* o, const int32_t* row_ptr_dev,
                                  const int32_t* col_idx_dev,
                                  const int32_t* row_order_dev,
                                  float softmax_scale, rp_stream stream);

/* Same, plus the reference's empty-row check (attention.cpp:85-86 throws
 * std::domain_error when a row has no active key): rows without an active
 * block are zero-filled and *err_flag_dev (device int, caller-zeroed; may be
 * NULL) is set to 1.  Stream-ordered: the caller reads the flag after the
 * stream and raises RP_DOMAIN_ERROR / domain_error itself. */
rp_status rp_sparse_attention_fwd_checked(const rp_grid* g, const rp_tensor* q,
                                          const rp_tensor* k, const rp_tensor* v,
                                          rp_tensor* o, const int32_t* row_ptr_dev,
                                          const int32_t* col_idx_dev,
                                          const int32_t* row_order_dev,
                                          float softmax_scale, int* err_flag_dev,
                                          rp_stream stream);

/* Name of the stage-(d) kernel rp_sparse_attention_fwd launches for this
 * grid, dtype (rp_dtype) and head_dim.  bf16: "db" while one head's K + V
 * fit in 64 MiB, "rp" above (DYNRAD_K6 = db | rp forces one per process). */
const char* rp_attention_kernel(const rp_grid* g, int dtype, int head_dim);

/* Host-buffer convenience with the reference's calling convention: host
 * Q/K/V [tokens, heads, d] (pinned or pageable; dtype f32 or bf16), host
 * bit-packed block mask; host output [S', heads, d].  Copies in, builds the
 * row lists, runs the kernel, copies out, synchronizes.  Throws
 * RP_DOMAIN_ERROR when a row has no active block (attention.cpp:85-86). */
rp_status rp_masked_attention_exact_host(const rp_grid* g,
                                         const uint8_t* mask_bits_host,
                                         const void* q_host, const void* k_host,
                                         const void* v_host, int dtype,
                                         int64_t tokens, int heads,
                                         int head_dim, void* o_host,
                                         rp_stream stream);

/* One whole attention layer from host buffers, stages (a)-(d): host Q/K/V
 * [tokens, heads, d] (pinned for full PCIe speed; f32 or bf16) are copied in
 * by head chunks; the plan builds the block mask (rp_plan_build_mask; in
 * dynamic mode from the first n_score_heads heads of Q/K, in static mode
 * from its cache, n_score_heads may be 0), then the row lists, and every
 * chunk's attention runs as soon as its inputs have landed while finished
 * chunks are copied out.  o_host: [S', heads, d]; mask_bits_host_out (may
 * be NULL) receives the bit-packed mask.  Synchronous.  RP_DOMAIN_ERROR
 * when a row has no active block (attention.cpp:85-86; the output is still
 * written, with zeros in that row). */
rp_status rp_sparse_layer_host(rp_plan plan, const rp_grid* g, const void* q_host,
                               const void* k_host, const void* v_host, int dtype,
                               int64_t tokens, int heads, int head_dim, int n_score_heads,
                               void* o_host, uint8_t* mask_bits_host_out, rp_stream stream);

/* Stage (b) of rp_pooled_select on its own: block means of the first n_heads
 * heads of x (bf16 [tokens, heads, d]) -> out_dev [S_b, n_heads * d] f32.
 * One pass over S * n_heads * d bf16 (HBM-bound; the bench's roofline for
 * the pooled selector). */
rp_status rp_block_mean_pool(const rp_grid* g, const rp_tensor* x, int n_heads,
                             float* out_dev, rp_stream stream);

/* ---------------------------------------------------- soft-mask attention --
 * masked_attention (attention.hpp:32-39, attention.cpp:59-81, 107-113): every
 * key takes part; logits get + log1p(epsilon) on active blocks and
 * + log(epsilon) on inactive ones, then row softmax and the value product.
 * epsilon must be > 0 (RP_INVALID_ARGUMENT "masked attention: epsilon must be
 * positive").  Same tensors, dtypes and kernels as rp_sparse_attention_fwd
 * (bf16: the tcgen05 kernel over dense row lists with a per-block logit
 * offset; f32: fp64 softmax, 1e-5 parity); mask_bits_dev is the bit-packed
 * block mask on the device. */
rp_status rp_soft_attention_fwd(const rp_grid* g, const rp_tensor* q,
                                const rp_tensor* k, const rp_tensor* v,
                                rp_tensor* o, const uint8_t* mask_bits_dev,
                                double epsilon, float softmax_scale,
                                rp_stream stream);

/* Host-buffer soft-mask attention (the reference's masked_attention calling
 * convention; buffers as in rp_masked_attention_exact_host). */
rp_status rp_masked_attention_host(const rp_grid* g,
                                   const uint8_t* mask_bits_host,
                                   const void* q_host, const void* k_host,
                                   const void* v_host, int dtype,
                                   int64_t tokens, int heads, int head_dim,
                                   double epsilon, void* o_host,
                                   rp_stream stream);

/* ------------------------------------------- profiler objective --
 * build_proxy_cache (profiler.hpp:58-66, profiler.cpp:49-78) and objective
 * (profiler.hpp:68-76, profiler.cpp:80-148) on the GPU.  The cache is
 * device-resident and opaque: per-(row, column block) sums of the dense
 * proxy attention numerators w and w^2, the diagonal, the row sums and
 * |A_dense|_F^2 -- everything a trial reads -- instead of the S x S matrix.
 * features_dev: the ProxyBatch features, [total_tokens, feature_dim] f32
 * row-major on the device.  The logits follow the reference's float GEMM
 * order, exp runs in double (see csrc/objective.cu for the contract). */
typedef struct rp_proxy_cache rp_proxy_cache;

typedef struct {
  double loss; /* mse + penalty_weight * max(0, sparsity_target - achieved) */
  double mse;  /* masked-vs-dense reconstruction error over real tokens */
  double achieved_sparsity; /* over the padded block grid */
} rp_trial;

/* Synchronous.  The grid is ProxyBatch::grid. */
rp_status rp_proxy_cache_create(const rp_grid* g, const float* features_dev,
                                int feature_dim, rp_proxy_cache** out,
                                rp_stream stream);

/* The reference's DenseProxyCache itself (build_proxy_cache): weights
 * [S, S] f32 row-major = exp(logit - row max), row_sums [S] f64 (device, may
 * be NULL) and reference_sq_norm (host, may be NULL).  Synchronous. */
rp_status rp_proxy_weights(const rp_grid* g, const float* features_dev, int feature_dim,
                           float* weights_dev, double* row_sums_dev,
                           double* reference_sq_norm, rp_stream stream);

/* From a reference-layout DenseProxyCache already on the device: weights
 * [S, S] f32 row-major, row_sums [S] f64, and its reference_sq_norm. */
rp_status rp_proxy_cache_from_weights(const rp_grid* g, const float* weights_dev,
                                      const double* row_sums_dev,
                                      double reference_sq_norm,
                                      rp_proxy_cache** out, rp_stream stream);

void rp_proxy_cache_destroy(rp_proxy_cache* cache);

/* Copies row_sums [S] (may be NULL) and reference_sq_norm to the host. */
rp_status rp_proxy_cache_stats(const rp_proxy_cache* cache, double* row_sums_host,
                               double* reference_sq_norm, rp_stream stream);

/* One trial: validates c, builds the mask with seed mix64(batch_seed,
 * 0x6d61736b) on the GPU (dynamic mode scores scoring_features(batch), i.e.
 * the features as one fused head), then the error and loss.  Synchronous.
 * mask_bits_dev (may be NULL) receives the trial's bit-packed mask. */
rp_status rp_objective(const rp_proxy_cache* cache, const rp_config* c,
                       uint64_t batch_seed, const float* features_dev,
                       int feature_dim, double penalty_weight,
                       double sparsity_target, rp_trial* out,
                       uint8_t* mask_bits_dev, rp_stream stream);

/* Number of CUDA kernels this library has launched in the calling process
 * (all entry points); used by bench.py to report gpu_launches. */
int64_t rp_kernel_launch_count(void);

/* Per-stage device timing (measurement support for bench.py).  While
 * enabled, the entry points record CUDA events on their launching stream
 * around each stage; rp_profile_read waits for them and returns, per stage
 * index, the summed milliseconds and the number of occurrences.  Stages:
 * 0 mask prep (base copy, norms), 1 tensor-core scoring pass 1 (stats),
 * 2 per-frame-pair thresholds, 3 tensor-core scoring pass 2 (select),
 * 4 exact recheck + fallback, 5 theta_c / theta_m apply, 6 CSR,
 * 7 stage-(d) attention, 8 exact fp64 scoring engine, 9 static build.
 * rp_profile_stages(1) clears previous records. */
void rp_profile_stages(int enable);
rp_status rp_profile_read(double* total_ms, int64_t* count, int n_stages);

#ifdef __cplusplus
}
#endif
#endif /* DYNRAD_H */
