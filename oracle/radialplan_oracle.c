/* TEST INFRASTRUCTURE ONLY — CPU restatement of the DynamicRad hot path.
 * See radialplan_oracle.h for who may load this and what pins it.
 *
 * Every function restates the reference algorithm from its definition; the
 * reference file:line it follows is cited beside it (paths relative to
 * /root/reference/proj).  Compiled with -ffp-contract=off so that the
 * double-precision score arithmetic rounds exactly as the reference's
 * (separate multiply then add).
 */
#define _GNU_SOURCE
#include "radialplan_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];
const char* orc_last_error(void) { return g_err; }

#define GOLDEN 0x9E3779B97F4A7C15ull

/* rng.hpp:19-25 */
uint64_t orc_mix64(uint64_t z) {
  z += GOLDEN;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* grid.hpp:23-42 */
int orc_make_grid(int nf, int nt, int bs, orc_grid* g) {
  if (nf < 1) { snprintf(g_err, sizeof g_err, "grid: n_frames must be >= 1"); return 1; }
  if (nt < 1) { snprintf(g_err, sizeof g_err, "grid: tokens_per_frame must be >= 1"); return 1; }
  if (bs < 2 || (bs & (bs - 1)) != 0) {
    snprintf(g_err, sizeof g_err, "grid: block_size must be a power of two >= 2");
    return 1;
  }
  g->n_frames = nf;
  g->tokens_per_frame = nt;
  g->block_size = bs;
  g->total_tokens = (int64_t)nf * nt;
  g->padded_tokens = (g->total_tokens + bs - 1) / bs * bs;
  g->blocks_per_dim = g->padded_tokens / bs;
  g->row_bytes = (g->blocks_per_dim + 7) / 8;
  return 0;
}

/* radial.cpp:10-28: octave index = bit width, L0 = next power of two,
 * decay = factor * L0 / 2^octave. */
static int bit_width(int64_t t) {
  int b = 0;
  while (t > 0) { ++b; t >>= 1; }
  return b;
}
static int64_t pow2_ceil(int64_t x) {
  int64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}
static double decay(int64_t t, double factor, int64_t base) {
  return factor * (double)base / (double)((int64_t)1 << bit_width(t));
}

typedef struct {
  int i, j;
  int64_t t, width, n;
  int tier;
  int retained;
} pair_info;

/* radial.cpp:30-62, 111-121; selection.cpp:34-41 */
static pair_info frame_pair(const orc_grid* g, const orc_cfg* c, int i, int j) {
  pair_info p;
  const int64_t nt = g->tokens_per_frame;
  const int64_t base = pow2_ceil(nt);
  p.i = i;
  p.j = j;
  p.t = i > j ? i - j : j - i;
  if (p.t <= 1) {
    p.width = nt;
  } else {
    int64_t r = llround(decay(p.t, c->decay_factor, base));
    p.width = r < g->block_size ? g->block_size : r;
  }
  if (p.t <= 1) {
    p.retained = 1;
  } else {
    const double raw = (double)g->block_size /
                       (decay(p.t, c->long_range_factor, base) + c->split_epsilon);
    int64_t sf = (int64_t)raw;
    if (sf < 1) sf = 1;
    p.retained = (p.t % sf) == 0;
  }
  if (p.t <= 1)
    p.tier = 0;
  else
    p.tier = decay(p.t, c->decay_factor, base) >= (double)g->block_size ? 1 : 2;
  if (!p.retained) {
    p.n = 0;
  } else if (p.width >= nt - 1) {
    p.n = nt * nt;
  } else {
    const int64_t m = nt - 1 - p.width;
    p.n = nt * nt - m * (m + 1);
  }
  return p;
}

void orc_frame_pair(const orc_grid* g, const orc_cfg* c, int i, int j,
                    int64_t out5[5]) {
  pair_info p = frame_pair(g, c, i, j);
  out5[0] = p.width;
  out5[1] = p.retained;
  out5[2] = p.n;
  out5[3] = p.tier;
  if (p.t >= 1) {
    const double raw =
        (double)g->block_size /
        (decay(p.t, c->long_range_factor, pow2_ceil(g->tokens_per_frame)) +
         c->split_epsilon);
    int64_t sf = (int64_t)raw;
    out5[4] = sf < 1 ? 1 : sf;
  } else {
    out5[4] = 1;
  }
}

static void set_bit(uint8_t* bits, int64_t row_bytes, int64_t r, int64_t col) {
  bits[r * row_bytes + col / 8] |= (uint8_t)(1u << (col % 8));
}

/* ---- per frame pair aggregation (mask.cpp:87-158) ---------------------- */

typedef struct {
  int64_t r0, c0, tr, tc;
  int bs;
  uint32_t* counts; /* [tr][tc][bs] */
} tiles_t;

static void tiles_reset(tiles_t* T, const orc_grid* g, int i, int j) {
  const int64_t nt = g->tokens_per_frame, bs = g->block_size;
  const int64_t qi = (int64_t)i * nt, kj = (int64_t)j * nt;
  T->bs = (int)bs;
  T->r0 = qi / bs;
  T->c0 = kj / bs;
  T->tr = (qi + nt - 1) / bs - T->r0 + 1;
  T->tc = (kj + nt - 1) / bs - T->c0 + 1;
  T->counts = (uint32_t*)calloc((size_t)(T->tr * T->tc * bs), sizeof(uint32_t));
}

static void tiles_add(tiles_t* T, int64_t grow, int64_t gcol) {
  const int64_t rr = grow / T->bs - T->r0, cc = gcol / T->bs - T->c0;
  T->counts[(rr * T->tc + cc) * T->bs + gcol % T->bs]++;
}

/* Column active iff count/B >= theta_c; tile iff active/B >= theta_m; both
 * denominators are B (mask.hpp:61-64). */
static void tiles_apply(const tiles_t* T, const orc_cfg* c, uint8_t* bits,
                        int64_t row_bytes) {
  for (int64_t r = 0; r < T->tr; ++r)
    for (int64_t cc = 0; cc < T->tc; ++cc) {
      const uint32_t* col = T->counts + (r * T->tc + cc) * T->bs;
      int active = 0;
      for (int k = 0; k < T->bs; ++k)
        if ((double)col[k] / T->bs >= c->col_threshold) ++active;
      if ((double)active / T->bs >= c->mask_threshold)
        set_bit(bits, row_bytes, T->r0 + r, T->c0 + cc);
    }
}

/* Closed-form counts of a fully kept band: column v of frame j is hit by
 * rows u in [v-w, v+w] of frame i (mask.cpp:132-158). */
static void tiles_full_band(tiles_t* T, const orc_grid* g, const pair_info* p) {
  const int64_t nt = g->tokens_per_frame, bs = T->bs;
  const int64_t qi = (int64_t)p->i * nt, kj = (int64_t)p->j * nt;
  for (int64_t v = 0; v < nt; ++v) {
    const int64_t gc = kj + v;
    const int64_t ulo = v - p->width < 0 ? 0 : v - p->width;
    const int64_t uhi = v + p->width > nt - 1 ? nt - 1 : v + p->width;
    if (ulo > uhi) continue;
    const int64_t cc = gc / bs - T->c0;
    for (int64_t r = 0; r < T->tr; ++r) {
      const int64_t lo0 = (T->r0 + r) * bs, hi0 = lo0 + bs - 1;
      const int64_t lo = qi + ulo > lo0 ? qi + ulo : lo0;
      const int64_t hi = qi + uhi < hi0 ? qi + uhi : hi0;
      if (lo > hi) continue;
      T->counts[(r * T->tc + cc) * bs + gc % bs] += (uint32_t)(hi - lo + 1);
    }
  }
}

/* Canonical row-major band enumeration (radial.cpp:64-79). */
static int64_t vlo(const pair_info* p, int64_t u) {
  return u - p->width < 0 ? 0 : u - p->width;
}
static int64_t* row_offsets(const orc_grid* g, const pair_info* p) {
  const int64_t nt = g->tokens_per_frame;
  int64_t* off = (int64_t*)malloc((size_t)(nt + 1) * sizeof(int64_t));
  off[0] = 0;
  for (int64_t u = 0; u < nt; ++u) {
    const int64_t hi = u + p->width > nt - 1 ? nt - 1 : u + p->width;
    off[u + 1] = off[u] + (hi - vlo(p, u) + 1);
  }
  return off;
}
/* upper_bound(off, flat) - 1 */
static int64_t row_of(const int64_t* off, int64_t nt, int64_t flat) {
  int64_t lo = 0, hi = nt; /* off[lo] <= flat < off[hi] */
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) / 2;
    if (off[mid] <= flat) lo = mid; else hi = mid;
  }
  return lo;
}

/* Static: partial Fisher-Yates over flat indices with the pair's splitmix64
 * stream (mask.cpp:224-252; selection.cpp:61-91; selection.hpp:45-48). */
static void select_static(tiles_t* T, const orc_grid* g, const pair_info* p,
                          double ratio, uint64_t seed) {
  const int64_t n = p->n, nt = g->tokens_per_frame;
  int64_t k = (int64_t)floor((double)n * ratio);
  if (k < 1) k = 1;
  uint32_t* fy = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
  for (int64_t x = 0; x < n; ++x) fy[x] = (uint32_t)x;
  uint64_t state =
      orc_mix64(orc_mix64(orc_mix64(seed) ^ (uint64_t)p->i) ^ (uint64_t)p->j);
  int64_t* off = row_offsets(g, p);
  const int64_t qi = (int64_t)p->i * nt, kj = (int64_t)p->j * nt;
  for (int64_t d = 0; d < k; ++d) {
    const uint64_t draw = orc_mix64(state);
    state += GOLDEN;
    const int64_t r = d + (int64_t)(draw % (uint64_t)(n - d));
    const uint32_t tmp = fy[d];
    fy[d] = fy[r];
    fy[r] = tmp;
    const int64_t flat = fy[d];
    const int64_t u = row_of(off, nt, flat);
    tiles_add(T, qi + u, kj + vlo(p, u) + (flat - off[u]));
  }
  free(off);
  free(fy);
}

typedef struct {
  double z;
  int64_t idx;
} zi_t;
static int zi_cmp(const void* a, const void* b) {
  const zi_t* x = (const zi_t*)a;
  const zi_t* y = (const zi_t*)b;
  if (x->z > y->z) return -1;
  if (x->z < y->z) return 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}
static int i64_cmp(const void* a, const void* b) {
  const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return x < y ? -1 : (x > y);
}

/* Dynamic: token-pair proxy scores in double (selection.cpp:93-123),
 * population z-score (:125-148), keep z >= tau else the fallback_k best,
 * ties to the lowest flat index (:150-185). */
static void select_dynamic(tiles_t* T, const orc_grid* g, const pair_info* p,
                           double tau, int fallback_k, const float* q,
                           const float* kf, int heads, int d) {
  const int64_t n = p->n, nt = g->tokens_per_frame;
  const int64_t qi = (int64_t)p->i * nt, kj = (int64_t)p->j * nt;
  const double inv_sqrt_d = 1.0 / sqrt((double)d);
  float* s = (float*)malloc((size_t)n * sizeof(float));
  int64_t x = 0;
  for (int64_t u = 0; u < nt; ++u) {
    const int64_t hi = u + p->width > nt - 1 ? nt - 1 : u + p->width;
    for (int64_t v = vlo(p, u); v <= hi; ++v) {
      double acc = 0.0;
      for (int h = 0; h < heads; ++h) {
        const float* qa = q + ((qi + u) * heads + h) * d;
        const float* kb = kf + ((kj + v) * heads + h) * d;
        double dot = 0.0;
        for (int e = 0; e < d; ++e) dot += (double)qa[e] * (double)kb[e];
        acc += dot * inv_sqrt_d;
      }
      s[x++] = (float)(acc / heads);
    }
  }
  double sum = 0.0;
  for (int64_t y = 0; y < n; ++y) sum += (double)s[y];
  const double mean = sum / (double)n;
  double sq = 0.0;
  for (int64_t y = 0; y < n; ++y) {
    const double dd = (double)s[y] - mean;
    sq += dd * dd;
  }
  const double denom = sqrt(sq / (double)n) + 1e-8;
  int64_t* off = row_offsets(g, p);
  int64_t kept = 0;
  for (int64_t y = 0; y < n; ++y) {
    if (((double)s[y] - mean) / denom >= tau) {
      const int64_t u = row_of(off, nt, y);
      tiles_add(T, qi + u, kj + vlo(p, u) + (y - off[u]));
      ++kept;
    }
  }
  if (kept == 0 && n > 0) {
    const int64_t k = fallback_k < n ? fallback_k : n;
    zi_t* zi = (zi_t*)malloc((size_t)n * sizeof(zi_t));
    for (int64_t y = 0; y < n; ++y) {
      zi[y].z = ((double)s[y] - mean) / denom;
      zi[y].idx = y;
    }
    qsort(zi, (size_t)n, sizeof(zi_t), zi_cmp);
    int64_t* pick = (int64_t*)malloc((size_t)k * sizeof(int64_t));
    for (int64_t y = 0; y < k; ++y) pick[y] = zi[y].idx;
    qsort(pick, (size_t)k, sizeof(int64_t), i64_cmp);
    for (int64_t y = 0; y < k; ++y) {
      const int64_t u = row_of(off, nt, pick[y]);
      tiles_add(T, qi + u, kj + vlo(p, u) + (pick[y] - off[u]));
    }
    free(pick);
    free(zi);
  }
  free(off);
  free(s);
}

/* ---- build_mask (mask.cpp:162-289) ------------------------------------- */

typedef struct {
  const orc_grid* g;
  const orc_cfg* c;
  uint64_t seed;
  const float *q, *k;
  int heads, d;
  const pair_info* jobs;
  int64_t begin, end;
  uint8_t* bits; /* private */
  int64_t scored;
} worker_t;

static void* worker_run(void* arg) {
  worker_t* w = (worker_t*)arg;
  const orc_grid* g = w->g;
  const orc_cfg* c = w->c;
  for (int64_t jx = w->begin; jx < w->end; ++jx) {
    const pair_info* p = &w->jobs[jx];
    tiles_t T;
    tiles_reset(&T, g, p->i, p->j);
    if (c->mode == 0) {
      const double ratio = p->tier == 0 ? 1.0 : (p->tier == 1 ? c->near_param : c->far_param);
      if (ratio >= 1.0) tiles_full_band(&T, g, p);
      else select_static(&T, g, p, ratio, w->seed);
    } else {
      if (p->tier == 0) {
        tiles_full_band(&T, g, p);
      } else {
        const double tau = p->tier == 1 ? c->near_param : c->far_param;
        if (p->n > 0)
          select_dynamic(&T, g, p, tau, c->fallback_k, w->q, w->k, w->heads, w->d);
        w->scored += p->n;
      }
    }
    tiles_apply(&T, c, w->bits, g->row_bytes);
    free(T.counts);
  }
  return NULL;
}

static int validate(const orc_cfg* c) {
  const char* msg = NULL;
  if (!(c->decay_factor > 0.0)) msg = "config: decay_factor must be positive";
  else if (!(c->long_range_factor > 0.0)) msg = "config: long_range_factor must be positive";
  else if (!(c->mask_threshold > 0.0 && c->mask_threshold <= 1.0)) msg = "config: mask_threshold must be in (0, 1]";
  else if (!(c->col_threshold > 0.0 && c->col_threshold <= 1.0)) msg = "config: col_threshold must be in (0, 1]";
  else if (c->fallback_k < 1) msg = "config: fallback_k must be >= 1";
  else if (c->mode == 0 && (!(c->near_param > 0.0 && c->near_param <= 1.0) ||
                            !(c->far_param > 0.0 && c->far_param <= 1.0)))
    msg = "config: static retention ratios must be in (0, 1]";
  else if (c->mode != 0 && (!isfinite(c->near_param) || !isfinite(c->far_param)))
    msg = "config: dynamic thresholds must be finite";
  if (msg) { snprintf(g_err, sizeof g_err, "%s", msg); return 1; }
  return 0;
}

int orc_build_mask(const orc_grid* g, const orc_cfg* c, uint64_t seed,
                   int disable_split, const float* q, const float* k,
                   int64_t tokens, int heads, int d, uint8_t* out_bits,
                   int threads, int64_t* stats) {
  if (validate(c)) return 1;
  if (c->mode != 0) {
    if (!q || !k) { snprintf(g_err, sizeof g_err, "build_mask: dynamic mode needs features"); return 1; }
    if (tokens < g->total_tokens) { snprintf(g_err, sizeof g_err, "build_mask: feature batch too short"); return 1; }
  }
  const int64_t S = g->blocks_per_dim, rb = g->row_bytes;
  memset(out_bits, 0, (size_t)(S * rb));
  /* intra-frame rectangles (mask.cpp:175-183) */
  for (int i = 0; i < g->n_frames; ++i) {
    const int64_t lo = (int64_t)i * g->tokens_per_frame;
    const int64_t hi = lo + g->tokens_per_frame - 1;
    for (int64_t r = lo / g->block_size; r <= hi / g->block_size; ++r)
      for (int64_t cb = lo / g->block_size; cb <= hi / g->block_size; ++cb)
        set_bit(out_bits, rb, r, cb);
  }
  /* job list: ordered pairs, t >= 1, split rule (mask.cpp:185-192) */
  const int nf = g->n_frames;
  pair_info* jobs = (pair_info*)malloc((size_t)nf * nf * sizeof(pair_info));
  int64_t nj = 0;
  for (int i = 0; i < nf; ++i)
    for (int j = 0; j < nf; ++j) {
      if (i == j) continue;
      pair_info p = frame_pair(g, c, i, j);
      /* With disable_split the pruned pair still becomes a job, but its
       * candidate set stays empty (candidate_set keeps retained=false,
       * radial.cpp:111-121): a full band is still counted in closed form
       * from the width, a sampled static pair would draw from an empty set
       * (the reference divides by zero there), a dynamic one keeps nothing. */
      if (!disable_split && !p.retained) continue;
      if (c->mode == 0 && !p.retained && p.tier != 0) {
        const double ratio = p.tier == 1 ? c->near_param : c->far_param;
        if (ratio < 1.0) {
          snprintf(g_err, sizeof g_err,
                   "build_mask: disable_split samples a pruned frame pair "
                   "(empty candidate set)");
          free(jobs);
          return 1;
        }
      }
      jobs[nj++] = p;
    }
  if (threads < 1) threads = 1;
  if (threads > nj) threads = nj > 0 ? (int)nj : 1;
  worker_t* ws = (worker_t*)calloc((size_t)threads, sizeof(worker_t));
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  const int64_t chunk = (nj + threads - 1) / threads;
  for (int w = 0; w < threads; ++w) {
    ws[w].g = g; ws[w].c = c; ws[w].seed = seed; ws[w].q = q; ws[w].k = k;
    ws[w].heads = heads; ws[w].d = d; ws[w].jobs = jobs;
    ws[w].begin = w * chunk;
    ws[w].end = (w + 1) * chunk < nj ? (w + 1) * chunk : nj;
    if (ws[w].begin > ws[w].end) ws[w].begin = ws[w].end;
    ws[w].bits = (uint8_t*)calloc((size_t)(S * rb), 1);
    if (threads == 1) worker_run(&ws[w]);
    else pthread_create(&th[w], NULL, worker_run, &ws[w]);
  }
  int64_t scored = 0;
  for (int w = 0; w < threads; ++w) {
    if (threads > 1) pthread_join(th[w], NULL);
    for (int64_t b = 0; b < S * rb; ++b) out_bits[b] |= ws[w].bits[b];
    scored += ws[w].scored;
    free(ws[w].bits);
  }
  if (stats) { stats[0] = nj; stats[1] = scored; }
  free(th);
  free(ws);
  free(jobs);
  return 0;
}

/* ---- masked_attention_exact (attention.cpp:43-121) --------------------- */

typedef struct {
  const orc_grid* g;
  const uint8_t* bits;
  const float *q, *k, *v;
  int64_t tokens;
  int heads, d;
  int64_t rb, re, row0;
  float* out;
  int status;
  int soft;            /* masked_attention (attention.cpp:59-81): log1p/log eps offsets */
  double log_active, log_inactive;
} attn_t;

static void* attn_run(void* arg) {
  attn_t* a = (attn_t*)arg;
  const int64_t n = a->g->padded_tokens, bs = a->g->block_size;
  const int64_t row_bytes = a->g->row_bytes;
  const int heads = a->heads, d = a->d;
  const double scale = 1.0 / sqrt((double)d);
  double* p = (double*)malloc((size_t)n * sizeof(double));
  double* acc = (double*)malloc((size_t)d * sizeof(double));
  for (int h = 0; h < heads; ++h)
    for (int64_t r = a->rb; r < a->re; ++r) {
      const int64_t br = r / bs;
      double m = -INFINITY;
      for (int64_t c = 0; c < n; ++c) {
        const int64_t bc = c / bs;
        const int active = (a->bits[br * row_bytes + bc / 8] >> (bc % 8)) & 1u;
        if (!a->soft && !active) {
          p[c] = -INFINITY;
          continue;
        }
        /* padded rows of Q/K are zero (attention.cpp:43-48) */
        float logit = 0.0f;
        if (r < a->tokens && c < a->tokens) {
          const float* qa = a->q + (r * heads + h) * d;
          const float* kb = a->k + (c * heads + h) * d;
          for (int e = 0; e < d; ++e) logit += qa[e] * kb[e];
        }
        const double l = (double)logit * scale +
                         (a->soft ? (active ? a->log_active : a->log_inactive) : 0.0);
        p[c] = l;
        if (l > m) m = l;
      }
      if (m == -INFINITY) { a->status = 3; goto done; }
      double sum = 0.0;
      for (int64_t c = 0; c < n; ++c) {
        p[c] = p[c] == -INFINITY ? 0.0 : exp(p[c] - m);
        sum += p[c];
      }
      for (int e = 0; e < d; ++e) acc[e] = 0.0;
      for (int64_t c = 0; c < n && c < a->tokens; ++c) {
        if (p[c] == 0.0) continue;
        const float* vb = a->v + (c * heads + h) * d;
        for (int e = 0; e < d; ++e) acc[e] += p[c] * (double)vb[e];
      }
      float* o = a->out + ((r - a->row0) * heads + h) * d;
      for (int e = 0; e < d; ++e) o[e] = (float)(acc[e] / sum);
    }
done:
  free(acc);
  free(p);
  return NULL;
}

static int attention(const orc_grid* g, const uint8_t* bits, const float* q, const float* k,
                     const float* v, int64_t tokens, int heads, int d, int soft, double eps,
                     int64_t row_begin, int64_t row_end, float* out, int threads) {
  if (tokens < 1 || heads < 1 || d < 1) {
    snprintf(g_err, sizeof g_err, "feature batch: empty dimensions");
    return 1;
  }
  if (g->padded_tokens < tokens) {
    snprintf(g_err, sizeof g_err, "masked attention: mask smaller than batch");
    return 1;
  }
  if (threads < 1) threads = 1;
  const int64_t rows = row_end - row_begin;
  if (threads > rows) threads = rows > 0 ? (int)rows : 1;
  attn_t* as = (attn_t*)calloc((size_t)threads, sizeof(attn_t));
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  const int64_t chunk = (rows + threads - 1) / threads;
  for (int w = 0; w < threads; ++w) {
    attn_t* a = &as[w];
    a->g = g; a->bits = bits; a->q = q; a->k = k; a->v = v; a->tokens = tokens;
    a->heads = heads; a->d = d; a->row0 = row_begin; a->out = out;
    a->soft = soft;
    a->log_active = soft ? log1p(eps) : 0.0;
    a->log_inactive = soft ? log(eps) : 0.0;
    a->rb = row_begin + w * chunk;
    a->re = row_begin + (w + 1) * chunk < row_end ? row_begin + (w + 1) * chunk : row_end;
    if (a->rb > a->re) a->rb = a->re;
    if (threads == 1) attn_run(a);
    else pthread_create(&th[w], NULL, attn_run, a);
  }
  int st = 0;
  for (int w = 0; w < threads; ++w) {
    if (threads > 1) pthread_join(th[w], NULL);
    if (as[w].status) st = as[w].status;
  }
  free(th);
  free(as);
  if (st == 3) snprintf(g_err, sizeof g_err, "masked attention: row has no active key");
  return st;
}

int orc_masked_attention_exact(const orc_grid* g, const uint8_t* bits,
                               const float* q, const float* k, const float* v,
                               int64_t tokens, int heads, int d,
                               int64_t row_begin, int64_t row_end, float* out,
                               int threads) {
  return attention(g, bits, q, k, v, tokens, heads, d, 0, 0.0, row_begin, row_end, out,
                   threads);
}

/* expand_mask (mask.cpp:52-66): every active block's bit broadcast to its
 * B x B token bits on the padded axis; out: padded_tokens rows of
 * ceil(padded_tokens / 8) bytes, LSB-first (TokenMask, mask.hpp:39-55). */
void orc_expand_mask(const orc_grid* g, const uint8_t* bits, uint8_t* out) {
  const int64_t n = g->padded_tokens, trb = (n + 7) / 8;
  memset(out, 0, (size_t)(n * trb));
  for (int64_t r = 0; r < n; ++r) {
    const int64_t br = r / g->block_size;
    for (int64_t bc = 0; bc < g->blocks_per_dim; ++bc) {
      if (!((bits[br * g->row_bytes + bc / 8] >> (bc % 8)) & 1u)) continue;
      for (int64_t c = bc * g->block_size; c < (bc + 1) * g->block_size && c < n; ++c)
        out[r * trb + c / 8] |= (uint8_t)(1u << (c % 8));
    }
  }
}

/* masked_attention (attention.cpp:107-113): epsilon must be positive. */
int orc_masked_attention(const orc_grid* g, const uint8_t* bits, const float* q,
                         const float* k, const float* v, int64_t tokens, int heads, int d,
                         double eps, int64_t row_begin, int64_t row_end, float* out,
                         int threads) {
  if (!(eps > 0.0)) {
    snprintf(g_err, sizeof g_err, "masked attention: epsilon must be positive");
    return 1;
  }
  return attention(g, bits, q, k, v, tokens, heads, d, 1, eps, row_begin, row_end, out,
                   threads);
}

/* ---- random_batch (attention.cpp:182-204; rng.hpp:84-91) --------------- */

static double gaussian_at(uint64_t key) {
  const uint64_t a = orc_mix64(key ^ 0x8D5CF3D2A3B1E601ull);
  const uint64_t b = orc_mix64(key ^ 0xC2B2AE3D27D4EB4Full);
  const double u1 = (double)((a >> 11) + 1) * 0x1.0p-53;
  const double u2 = (double)(b >> 11) * 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

typedef struct {
  int64_t tb, te;
  int heads, d;
  uint64_t seed;
  float *q, *k, *v;
} rb_t;

static void* rb_run(void* arg) {
  rb_t* r = (rb_t*)arg;
  float* dst[3] = {r->q, r->k, r->v};
  for (int role = 1; role <= 3; ++role) {
    float* out = dst[role - 1];
    if (!out) continue;
    for (int h = 0; h < r->heads; ++h) {
      const uint64_t base =
          orc_mix64(orc_mix64(orc_mix64(r->seed) ^ (uint64_t)role) ^ (uint64_t)h);
      for (int64_t t = r->tb; t < r->te; ++t) {
        const uint64_t bt = orc_mix64(orc_mix64(base) ^ (uint64_t)t);
        for (int e = 0; e < r->d; ++e)
          out[(t * r->heads + h) * r->d + e] =
              (float)gaussian_at(orc_mix64(bt ^ (uint64_t)e));
      }
    }
  }
  return NULL;
}

void orc_random_batch(int64_t tokens, int heads, int d, uint64_t seed,
                      float* q, float* k, float* v, int threads) {
  if (threads < 1) threads = 1;
  if (threads > tokens) threads = (int)tokens;
  rb_t* rs = (rb_t*)calloc((size_t)threads, sizeof(rb_t));
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  const int64_t chunk = (tokens + threads - 1) / threads;
  for (int w = 0; w < threads; ++w) {
    rs[w].tb = w * chunk;
    rs[w].te = (w + 1) * chunk < tokens ? (w + 1) * chunk : tokens;
    if (rs[w].tb > rs[w].te) rs[w].tb = rs[w].te;
    rs[w].heads = heads; rs[w].d = d; rs[w].seed = seed;
    rs[w].q = q; rs[w].k = k; rs[w].v = v;
    if (threads == 1) rb_run(&rs[w]);
    else pthread_create(&th[w], NULL, rb_run, &rs[w]);
  }
  if (threads > 1)
    for (int w = 0; w < threads; ++w) pthread_join(th[w], NULL);
  free(th);
  free(rs);
}

/* ---- profiler objective (profiler.cpp:49-148), SURVEY 8f3 ---------------- */

typedef struct {
  int64_t n, rb, re;
  int dim;
  const float* f;
  float* w;     /* [n, n] row-major */
  double* rs;
} cache_t;

static void* cache_run(void* arg) {
  cache_t* a = (cache_t*)arg;
  const int64_t n = a->n;
  const int dim = a->dim;
  const float scale = 1.0f / sqrtf((float)dim); /* profiler.cpp:52 (float) */
  for (int64_t r = a->rb; r < a->re; ++r) {
    float* wr = a->w + r * n;
    const float* fr = a->f + r * dim;
    /* scale * (F F^T): the float GEMM, ascending feature index */
    for (int64_t c = 0; c < n; ++c) {
      const float* fc = a->f + c * dim;
      float acc = 0.0f;
      for (int k = 0; k < dim; ++k) acc += fr[k] * fc[k];
      wr[c] = scale * acc;
    }
    double m = -INFINITY;
    for (int64_t c = 0; c < n; ++c)
      if ((double)wr[c] > m) m = (double)wr[c];
    double sum = 0.0;
    for (int64_t c = 0; c < n; ++c) {
      const double e = exp((double)wr[c] - m);
      wr[c] = (float)e;
      sum += e;
    }
    a->rs[r] = sum;
  }
  return NULL;
}

static void proxy_cache_fill(int64_t n, int dim, const float* f, float* w, double* rs,
                             double* sq, int threads) {
  if (threads < 1) threads = 1;
  if (threads > n) threads = (int)n;
  cache_t* as = (cache_t*)calloc((size_t)threads, sizeof(cache_t));
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  const int64_t chunk = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    cache_t* a = &as[t];
    a->n = n; a->dim = dim; a->f = f; a->w = w; a->rs = rs;
    a->rb = t * chunk < n ? t * chunk : n;
    a->re = (t + 1) * chunk < n ? (t + 1) * chunk : n;
    if (threads == 1) cache_run(a);
    else pthread_create(&th[t], NULL, cache_run, a);
  }
  if (threads > 1)
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(as);
  /* |A_dense|_F^2, sequential as profiler.cpp:70-76 */
  double acc = 0.0;
  for (int64_t r = 0; r < n; ++r)
    for (int64_t c = 0; c < n; ++c) {
      const double a = (double)w[r * n + c] / rs[r];
      acc += a * a;
    }
  *sq = acc;
}

int orc_proxy_cache(int64_t tokens, int dim, const float* features, float* weights,
                    double* row_sums, double* sq_norm, int threads) {
  if (tokens < 1 || dim < 1) {
    snprintf(g_err, sizeof g_err, "proxy cache: empty batch");
    return 1;
  }
  float* w = weights ? weights : (float*)malloc((size_t)(tokens * tokens) * sizeof(float));
  proxy_cache_fill(tokens, dim, features, w, row_sums, sq_norm, threads);
  if (!weights) free(w);
  return 0;
}

int orc_objective(const orc_grid* g, const orc_cfg* c, const float* features, int dim,
                  uint64_t batch_seed, double penalty_weight, double sparsity_target,
                  double* out3, int threads) {
  const int64_t n = g->total_tokens, bs = g->block_size;
  const uint64_t mask_seed = orc_mix64(orc_mix64(batch_seed) ^ 0x6d61736bull);
  uint8_t* bits = (uint8_t*)calloc((size_t)(g->blocks_per_dim * g->row_bytes), 1);
  int rc = c->mode == 1
               ? orc_build_mask(g, c, mask_seed, 0, features, features, n, 1, dim, bits,
                                threads, NULL)
               : orc_build_mask(g, c, mask_seed, 0, NULL, NULL, 0, 0, 0, bits, threads, NULL);
  if (rc) {
    free(bits);
    return rc;
  }
  float* w = (float*)malloc((size_t)(n * n) * sizeof(float));
  double* rs = (double*)malloc((size_t)n * sizeof(double));
  double sq = 0.0;
  proxy_cache_fill(n, dim, features, w, rs, &sq, threads);
  double num = 0.0;
  for (int64_t r = 0; r < n; ++r) {
    const int64_t br = r / bs;
    const double rd = rs[r];
    const float* wr = w + r * n;
    double rm = 0.0;
    for (int64_t cb = 0; cb * bs < n; ++cb) {
      if (!((bits[br * g->row_bytes + cb / 8] >> (cb % 8)) & 1u)) continue;
      const int64_t hi = (cb + 1) * bs < n ? (cb + 1) * bs : n;
      for (int64_t col = cb * bs; col < hi; ++col) rm += (double)wr[col];
    }
    if (rm == 0.0) {
      for (int64_t col = 0; col < n; ++col) {
        const double d = (double)wr[col] / rd - (col == r ? 1.0 : 0.0);
        num += d * d;
      }
      continue;
    }
    for (int64_t cb = 0; cb * bs < n; ++cb) {
      const int on = (bits[br * g->row_bytes + cb / 8] >> (cb % 8)) & 1u;
      const int64_t hi = (cb + 1) * bs < n ? (cb + 1) * bs : n;
      for (int64_t col = cb * bs; col < hi; ++col) {
        const double x = (double)wr[col];
        const double dense = x / rd;
        const double d = on ? dense - x / rm : dense;
        num += d * d;
      }
    }
  }
  int64_t active = 0;
  for (int64_t i = 0; i < g->blocks_per_dim * g->row_bytes; ++i)
    active += __builtin_popcount(bits[i]);
  const double sp =
      1.0 - (double)active / ((double)g->blocks_per_dim * (double)g->blocks_per_dim);
  out3[1] = num / sq;
  out3[2] = sp;
  out3[0] = out3[1] + penalty_weight * (sparsity_target - sp > 0.0 ? sparsity_target - sp : 0.0);
  free(w);
  free(rs);
  free(bits);
  return 0;
}

