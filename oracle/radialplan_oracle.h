/* TEST INFRASTRUCTURE ONLY — the CPU restatement of the DynamicRad hot path.
 *
 * Plain C11.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and only as
 * the checker or the timed CPU baseline, never as the product path.
 *
 * Pinned by: the compiled reference (oracle/_ref/libradialplan_ref.so, built
 * from /root/reference by oracle/Makefile) and the golden vectors under
 * tests/golden/ (generated from that build by tests/golden/make_golden.py).
 * tests/test_oracle.py checks this restatement against both.
 */
#ifndef RADIALPLAN_ORACLE_H
#define RADIALPLAN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int mode; /* 0 static ratio, 1 dynamic threshold */
  double decay_factor, long_range_factor, split_epsilon;
  double mask_threshold, col_threshold, near_param, far_param;
  int fallback_k;
} orc_cfg;

typedef struct {
  int n_frames, tokens_per_frame, block_size;
  int64_t total_tokens, padded_tokens, blocks_per_dim, row_bytes;
} orc_grid;

/* 0 ok, 1 invalid argument (message via orc_last_error). */
int orc_make_grid(int nf, int nt, int bs, orc_grid* g);
const char* orc_last_error(void);

/* Per ordered frame pair (i, j): window, retained, pair_count, tier,
 * split factor (radial.cpp:30-121, selection.cpp:34-59). */
void orc_frame_pair(const orc_grid* g, const orc_cfg* c, int i, int j,
                    int64_t out5[5]);

/* Algorithm 1 (mask.cpp:162-289).  q/k: [tokens, heads, d] float32, needed
 * only in dynamic mode.  out_bits: blocks_per_dim * row_bytes bytes.
 * threads >= 1 splits frame pairs across pthreads (result is independent of
 * it).  stats (may be NULL): [retained_frame_pairs, scored_pairs]. */
int orc_build_mask(const orc_grid* g, const orc_cfg* c, uint64_t seed,
                   int disable_split, const float* q, const float* k,
                   int64_t tokens, int heads, int d, uint8_t* out_bits,
                   int threads, int64_t* stats);

/* masked_attention_exact (attention.cpp:50-121) for query rows
 * [row_begin, row_end) of the padded axis.  q/k/v: [tokens, heads, d];
 * out: [(row_end-row_begin), heads, d].  Returns 3 on an empty row
 * (domain_error in the reference). */
void orc_expand_mask(const orc_grid* g, const uint8_t* bits, uint8_t* out);
int orc_masked_attention_exact(const orc_grid* g, const uint8_t* bits,
                               const float* q, const float* k, const float* v,
                               int64_t tokens, int heads, int d,
                               int64_t row_begin, int64_t row_end, float* out,
                               int threads);

/* masked_attention (attention.cpp:59-81, 107-113): soft mask, eps > 0. */
int orc_masked_attention(const orc_grid* g, const uint8_t* bits, const float* q,
                         const float* k, const float* v, int64_t tokens, int heads, int d,
                         double eps, int64_t row_begin, int64_t row_end, float* out,
                         int threads);

/* build_proxy_cache (profiler.cpp:49-78): features [S, dim] row-major;
 * weights [S, S] row-major (may be NULL: not stored), row_sums [S]. */
int orc_proxy_cache(int64_t tokens, int dim, const float* features, float* weights,
                    double* row_sums, double* sq_norm, int threads);

/* objective (profiler.cpp:80-148) with its own cache: out3 = {loss, mse,
 * achieved_sparsity}.  features: ProxyBatch::features [total_tokens, dim]. */
int orc_objective(const orc_grid* g, const orc_cfg* c, const float* features, int dim,
                  uint64_t batch_seed, double penalty_weight, double sparsity_target,
                  double* out3, int threads);

/* random_batch (attention.cpp:182-204): [tokens, heads, d] each. */
void orc_random_batch(int64_t tokens, int heads, int d, uint64_t seed,
                      float* q, float* k, float* v, int threads);

/* splitmix64 finalizer (rng.hpp:19-25). */
uint64_t orc_mix64(uint64_t z);

#ifdef __cplusplus
}
#endif
#endif
