// Stages (a)-(c) on the GPU: radialplan::build_mask (mask.cpp:162-289).
//
// Host side plans the frame-pair job table (plan.hpp, O(N_f^2) scalars with
// the reference's exact arithmetic).  Device side does all per-token / per-
// pair work:
//   K1  base mask: intra-frame rectangles (mask.cpp:175-183) and full-band
//       pairs (ratio >= 1 or tau = -inf) by closed-form column counts
//       (mask.cpp:132-158) -> theta_c / theta_m rule -> atomicOr.
//   K4  static ratio: exact partial Fisher-Yates (mask.cpp:224-252) resolved
//       in parallel: counter-form splitmix64 draws, a radix sort of
//       (pair, target, step) keys, then a pointer chase that recovers the
//       value each step swaps into its slot; per-column counts by atomics.
//   K2/K3 dynamic threshold, exact engine: fp64 token-pair proxy scores with
//       the reference's pinned operation order (selection.cpp:93-123),
//       sequential per-pair mean / population std (selection.cpp:125-148),
//       z >= tau, fallback_k best (selection.cpp:150-185).  The tensor-core
//       engine for large grids lives in mask_score_sm100.cu.
// Per-frame-pair counts are never merged across pairs (a tile straddling two
// frame pairs is judged per pair and OR-ed, mask.cpp:87-125).
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "internal.hpp"
#include "mask_build.cuh"
#include "mask_common.cuh"
#include "plan.hpp"

namespace rp {
namespace mask {

// ---------------------------------------------------- K1: base mask -------
__global__ void intra_kernel(uint32_t* words, int nf, int64_t nt, int bs, int64_t row_bytes,
                             int span) {
  const int f = blockIdx.x;
  const int64_t lo = static_cast<int64_t>(f) * nt, hi = lo + nt - 1;
  const int64_t b0 = lo / bs, b1 = hi / bs;
  for (int x = threadIdx.x; x < span * span; x += blockDim.x) {
    const int64_t r = b0 + x / span, c = b0 + x % span;
    if (r <= b1 && c <= b1) set_block(words, row_bytes, r, c);
  }
}

// ------------------------------------------ K4: exact partial Fisher-Yates --
// Draw d of job j: r_d = d + next_d % (n - d), next_d = stream call d of
// SplitMix64(pair_seed) (rng.hpp:40-48, mask.cpp:245-248).
RP_DEV int64_t fy_target(const DJob& jb, int64_t d) {
  const uint64_t x = stream_at(jb.seed, static_cast<uint64_t>(d));
  return d + static_cast<int64_t>(x % static_cast<uint64_t>(jb.n - d));
}

__global__ void fy_draw_kernel(const DJob* __restrict__ jobs, const int* __restrict__ batch_jobs,
                               const int64_t* __restrict__ off, int n_jobs, int64_t total,
                               int bits, uint64_t* __restrict__ keys) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= total) return;
  const int lj = find_job(off, n_jobs, x);
  const DJob& jb = jobs[batch_jobs[lj]];
  const int64_t d = x - off[lj];
  const int64_t r = fy_target(jb, d);
  keys[x] = (static_cast<uint64_t>(lj) << (2 * bits)) | (static_cast<uint64_t>(r) << bits) |
            static_cast<uint64_t>(d);
}

// After sorting by (job, target, step): prev[d] = previous step with the same
// target (or -1); tlast[p] (p < k) = last step e != p that targeted slot p.
__global__ void fy_link_kernel(const uint64_t* __restrict__ keys, int64_t total, int bits,
                               const int64_t* __restrict__ off, int32_t* __restrict__ prev,
                               int32_t* __restrict__ tlast, const DJob* __restrict__ jobs,
                               const int* __restrict__ batch_jobs) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const uint64_t mask = (uint64_t{1} << bits) - 1;
  const uint64_t key = keys[i];
  const uint64_t grp = key >> bits;  // (job, target)
  const int lj = static_cast<int>(key >> (2 * bits));
  const int64_t r = static_cast<int64_t>((key >> bits) & mask);
  const int64_t d = static_cast<int64_t>(key & mask);
  const bool has_prev = i > 0 && (keys[i - 1] >> bits) == grp;
  const int64_t dprev = has_prev ? static_cast<int64_t>(keys[i - 1] & mask) : -1;
  prev[off[lj] + d] = static_cast<int32_t>(dprev);
  const bool last = i + 1 == total || (keys[i + 1] >> bits) != grp;
  const int64_t k = jobs[batch_jobs[lj]].k;
  if (last && r < k) {
    const int64_t e = d != r ? d : dprev;  // exclude the slot's own step
    tlast[off[lj] + r] = static_cast<int32_t>(e);
  }
}

// Value swapped into slot d at step d: the target r_d itself when no
// earlier step touched it, else A(e) chased down the tlast links.
RP_DEV int64_t fy_slot_value(const DJob& jb, int64_t d, int32_t p, const int32_t* tl) {
  if (p < 0) return fy_target(jb, d);  // slot r_d untouched before step d
  int64_t e = p;  // A(e): value at slot e before step e
  while (tl[e] >= 0) e = tl[e];
  return e;
}

// ... then counted into its tile column (build_mask).
__global__ void fy_count_kernel(const DJob* __restrict__ jobs, const int* __restrict__ batch_jobs,
                                const int64_t* __restrict__ off, int n_jobs, int64_t total,
                                const int32_t* __restrict__ prev,
                                const int32_t* __restrict__ tlast, uint32_t* counts, int64_t nt,
                                int bs) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= total) return;
  const int lj = find_job(off, n_jobs, x);
  const DJob& jb = jobs[batch_jobs[lj]];
  const int64_t d = x - off[lj];
  const int64_t val = fy_slot_value(jb, d, prev[x], tlast + off[lj]);
  int64_t u, v;
  band_uv(val, nt, jb.width, &u, &v);
  add_count(jb, counts, nt, bs, u, v);
}

// ... or emitted as the (u, v) of slot d (static_select, one job).
__global__ void fy_value_kernel(const DJob* __restrict__ job, int64_t k,
                                const int32_t* __restrict__ prev,
                                const int32_t* __restrict__ tlast, int64_t nt,
                                int64_t* __restrict__ uv) {
  const int64_t d = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (d >= k) return;
  const int64_t val = fy_slot_value(*job, d, prev[d], tlast);
  band_uv(val, nt, job->width, &uv[2 * d], &uv[2 * d + 1]);
}

// ---------------------------------- per-frame-pair selection operators -----
// normalize_scores' z (selection.cpp:144-146) from the pinned stats.
__global__ void zscore_kernel(const float* __restrict__ s, int64_t n,
                              const double2* __restrict__ st, double* __restrict__ z) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x < n) z[x] = zscore(s[x], *st);
}

// dynamic_select keep set (selection.cpp:159-161), in flat order: per-CTA
// counts, then an ordered scatter after a host-side exclusive scan.
constexpr int kSelTile = 1024;
__global__ void keep_count_kernel(const double* __restrict__ z, int64_t n, double tau,
                                  int32_t* __restrict__ cta_count) {
  __shared__ int32_t c;
  if (threadIdx.x == 0) c = 0;
  __syncthreads();
  const int64_t x = static_cast<int64_t>(blockIdx.x) * kSelTile + threadIdx.x;
  int mine = 0;
  for (int64_t y = x; y < n && y < (static_cast<int64_t>(blockIdx.x) + 1) * kSelTile;
       y += blockDim.x)
    mine += z[y] >= tau;
  if (mine) atomicAdd(&c, mine);
  __syncthreads();
  if (threadIdx.x == 0) cta_count[blockIdx.x] = c;
}
__global__ void keep_scatter_kernel(const double* __restrict__ z, int64_t n, double tau,
                                    const int64_t* __restrict__ cta_off, int64_t nt, int64_t w,
                                    int64_t* __restrict__ uv) {
  // one warp-ordered pass per CTA tile keeps the flat order
  __shared__ int32_t base;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kSelTile;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int64_t y0 = t0; y0 < n && y0 < t0 + kSelTile; y0 += blockDim.x) {
    const int64_t y = y0 + threadIdx.x;
    const bool keep = y < n && y < t0 + kSelTile && z[y] >= tau;
    const unsigned m = __ballot_sync(0xFFFFFFFFu, keep);
    __shared__ int32_t warp_tot[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) warp_tot[wid] = __popc(m);
    __syncthreads();
    int before = base;
    for (int q = 0; q < wid; ++q) before += warp_tot[q];
    if (keep) {
      const int64_t slot = cta_off[blockIdx.x] + before + __popc(m & ((1u << lane) - 1));
      band_uv(y, nt, w, &uv[2 * slot], &uv[2 * slot + 1]);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) tot += warp_tot[q];
      base += tot;
    }
    __syncthreads();
  }
}
// Fallback (selection.cpp:163-175): the fallback_k best z, ties to the lower
// flat index, emitted in ascending flat order.  One CTA, k argmax rounds.
__global__ void fallback_pick_kernel(const double* __restrict__ z, int64_t n, int k, int64_t nt,
                                     int64_t w, int64_t* __restrict__ uv) {
  __shared__ double bz[32];
  __shared__ int64_t bi[32];
  __shared__ int64_t last_pick;
  __shared__ double last_z;
  if (threadIdx.x == 0) {
    last_pick = -1;
    last_z = INFINITY;
  }
  __syncthreads();
  for (int round = 0; round < k; ++round) {
    double best = -INFINITY;
    int64_t besti = -1;
    for (int64_t x = threadIdx.x; x < n; x += blockDim.x) {
      const double zz = z[x];
      if (!(zz < last_z || (zz == last_z && x > last_pick))) continue;
      if (besti < 0 || zz > best || (zz == best && x < besti)) {
        best = zz;
        besti = x;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double oz = __shfl_xor_sync(0xFFFFFFFFu, best, o);
      const int64_t oi = __shfl_xor_sync(0xFFFFFFFFu, besti, o);
      if (oi >= 0 && (besti < 0 || oz > best || (oz == best && oi < besti))) {
        best = oz;
        besti = oi;
      }
    }
    if ((threadIdx.x & 31) == 0) {
      bz[threadIdx.x >> 5] = best;
      bi[threadIdx.x >> 5] = besti;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int q = 1; q < static_cast<int>(blockDim.x >> 5); ++q)
        if (bi[q] >= 0 && (bi[0] < 0 || bz[q] > bz[0] || (bz[q] == bz[0] && bi[q] < bi[0]))) {
          bz[0] = bz[q];
          bi[0] = bi[q];
        }
      uv[2 * round] = bi[0];  // flat index; converted below
      last_pick = bi[0];
      last_z = bz[0];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    for (int a = 1; a < k; ++a)  // ascending flat order (selection.cpp:174)
      for (int b = a; b > 0 && uv[2 * (b - 1)] > uv[2 * b]; --b) {
        const int64_t t = uv[2 * b];
        uv[2 * b] = uv[2 * (b - 1)];
        uv[2 * (b - 1)] = t;
      }
    for (int a = 0; a < k; ++a) {
      const int64_t flat = uv[2 * a];
      band_uv(flat, nt, w, &uv[2 * a], &uv[2 * a + 1]);
    }
  }
}

// Token mask (S' x S' bits) -> block mask at block size B: the block bit is
// its top-left token bit; `bad` counts blocks that are not uniform.
__global__ void token_to_block_kernel(const uint8_t* __restrict__ tok, int64_t dim,
                                      int64_t trb, int bs, int64_t nb, int64_t brb,
                                      uint32_t* __restrict__ words,
                                      unsigned long long* __restrict__ bad) {
  const int64_t blk = blockIdx.x;  // block row * nb + block col
  const int64_t br = blk / nb, bc = blk % nb;
  const auto bit = [&](int64_t r, int64_t c) { return (tok[r * trb + c / 8] >> (c % 8)) & 1; };
  const int ref = bit(br * bs, bc * bs);
  int diff = 0;
  for (int64_t e = threadIdx.x; e < static_cast<int64_t>(bs) * bs; e += blockDim.x)
    diff |= bit(br * bs + e / bs, bc * bs + e % bs) != ref;
  diff = __syncthreads_or(diff);
  if (threadIdx.x == 0) {
    if (diff) atomicAdd(bad, 1ull);
    if (ref) set_block(words, brb, br, bc);
  }
}

// ------------------------------------ K2/K3 exact engine (fp64 SIMT) -------
// One thread per band pair of the batch (flat index x).  The frame pair and
// the band row are searched once per warp (lane 0) and each lane narrows
// from there: a warp's 32 consecutive pairs span at most 32 band rows.
__global__ void exact_scores_kernel(const DJob* __restrict__ jobs,
                                    const int* __restrict__ batch_jobs,
                                    const int64_t* __restrict__ off, int n_jobs, int64_t total,
                                    Feat f, int64_t nt, float* __restrict__ scores) {
  const int lane = threadIdx.x & 31;
  const int64_t x0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + (threadIdx.x & ~31);
  if (x0 >= total) return;
  int lj0 = 0;
  int64_t u0 = 0;
  if (lane == 0) {
    lj0 = find_job(off, n_jobs, x0);
    int64_t v0;
    band_uv(x0 - off[lj0], nt, jobs[batch_jobs[lj0]].width, &u0, &v0);
  }
  lj0 = __shfl_sync(0xFFFFFFFFu, lj0, 0);
  u0 = __shfl_sync(0xFFFFFFFFu, u0, 0);
  const int64_t x = x0 + lane;
  if (x >= total) return;
  int lj = lj0;
  while (x >= off[lj + 1]) ++lj;
  const DJob& jb = jobs[batch_jobs[lj]];
  int64_t u, v;
  if (lj == lj0) band_uv(x - off[lj], nt, jb.width, &u, &v, u0, u0 + 32);
  else band_uv(x - off[lj], nt, jb.width, &u, &v);
  scores[x] = exact_score(f, static_cast<int64_t>(jb.i) * nt + u,
                          static_cast<int64_t>(jb.j) * nt + v);
}

// selection.cpp:133-142, sequential like the reference: bit-identical stats.
// The two fp64 chains (the sum, then the squared deviations from the mean)
// stay in one thread in the reference's order; the block's other warps stage
// the scores into shared memory chunk by chunk (double-buffered), so the
// chain runs at the DADD latency instead of waiting on a global load per
// score.  One block per frame pair.
constexpr int kSeqChunk = 4096;
constexpr int kSeqThreads = 256;
__global__ void __launch_bounds__(kSeqThreads) seq_stats_kernel(const int64_t* __restrict__ off,
                                                                int n_jobs,
                                                                const float* __restrict__ scores,
                                                                double2* __restrict__ stats,
                                                                double* __restrict__ inv_den) {
  __shared__ __align__(16) float buf[2][kSeqChunk];
  const int lj = blockIdx.x;
  if (lj >= n_jobs) return;
  const float* s = scores + off[lj];
  const int64_t n = off[lj + 1] - off[lj];
  const int64_t nch = (n + kSeqChunk - 1) / kSeqChunk;
  auto fill = [&](int b, int64_t c) {  // warps 1.. only: warp 0 runs the chain
    if (threadIdx.x < 32) return;
    const int64_t base = c * kSeqChunk;
    const int cnt = static_cast<int>(n - base < kSeqChunk ? n - base : kSeqChunk);
    for (int i = threadIdx.x - 32; i < cnt; i += kSeqThreads - 32) buf[b][i] = s[base + i];
  };
  double sum = 0.0, mean = 0.0, sq = 0.0;
  for (int pass = 0; pass < 2; ++pass) {
    if (nch > 0) fill(0, 0);
    __syncthreads();
    for (int64_t c = 0; c < nch; ++c) {
      if (c + 1 < nch) fill(static_cast<int>((c + 1) & 1), c + 1);
      if (threadIdx.x == 0) {
        const float* b = buf[c & 1];
        const int cnt = static_cast<int>(n - c * kSeqChunk < kSeqChunk ? n - c * kSeqChunk
                                                                       : kSeqChunk);
        int i = 0;
        if (pass == 0) {
#pragma unroll 4
          for (; i + 4 <= cnt; i += 4) {
            const float4 v = *reinterpret_cast<const float4*>(b + i);
            sum = __dadd_rn(sum, static_cast<double>(v.x));
            sum = __dadd_rn(sum, static_cast<double>(v.y));
            sum = __dadd_rn(sum, static_cast<double>(v.z));
            sum = __dadd_rn(sum, static_cast<double>(v.w));
          }
          for (; i < cnt; ++i) sum = __dadd_rn(sum, static_cast<double>(b[i]));
        } else {
          auto step = [&](float x) {
            const double dd = __dsub_rn(static_cast<double>(x), mean);
            sq = __dadd_rn(sq, __dmul_rn(dd, dd));
          };
#pragma unroll 4
          for (; i + 4 <= cnt; i += 4) {
            const float4 v = *reinterpret_cast<const float4*>(b + i);
            step(v.x);
            step(v.y);
            step(v.z);
            step(v.w);
          }
          for (; i < cnt; ++i) step(b[i]);
        }
      }
      __syncthreads();
    }
    if (pass == 0) mean = __ddiv_rn(sum, static_cast<double>(n));
  }
  if (threadIdx.x == 0) {
    const double sd = __dsqrt_rn(__ddiv_rn(sq, static_cast<double>(n)));
    stats[lj] = make_double2(mean, sd);
    if (inv_den) inv_den[lj] = 1.0 / __dadd_rn(sd, 1e-8);
  }
}

// z >= tau per pair (selection.cpp:144-161).  z is the reference's
// correctly rounded (s - mean) / (sd + 1e-8); a multiply by the frame pair's
// reciprocal decides every pair whose z is not within 1e-13 (relative) of
// tau, the rest take the exact division.  The frame pair's kept counter is
// bumped once per warp and job.
__global__ void exact_select_kernel(const DJob* __restrict__ jobs,
                                    const int* __restrict__ batch_jobs,
                                    const int64_t* __restrict__ off, int n_jobs, int64_t total,
                                    const float* __restrict__ scores,
                                    const double2* __restrict__ stats,
                                    const double* __restrict__ inv_den, uint32_t* counts,
                                    unsigned long long* kept, int64_t nt, int bs) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool valid = x < total;
  const int lj = valid ? find_job(off, n_jobs, x) : -1;
  bool keep = false;
  if (valid) {
    const DJob& jb = jobs[batch_jobs[lj]];
    const double2 st = stats[lj];
    const double num = __dsub_rn(static_cast<double>(scores[x]), st.x);
    const double tau = jb.param;
    double z = __dmul_rn(num, inv_den[lj]);
    if (fabs(z - tau) <= 1e-13 * (fabs(z) + fabs(tau)) || !isfinite(z))
      z = __ddiv_rn(num, __dadd_rn(st.y, 1e-8));
    keep = z >= tau;
    if (keep) {
      int64_t u, v;
      band_uv(x - off[lj], nt, jb.width, &u, &v);
      add_count(jb, counts, nt, bs, u, v);
    }
  }
  const unsigned km = __ballot_sync(0xFFFFFFFFu, keep);
  const unsigned same = __match_any_sync(0xFFFFFFFFu, lj);
  const int lane = threadIdx.x & 31;
  if (lj >= 0 && lane == __ffs(same) - 1 && (km & same))
    atomicAdd(&kept[lj], static_cast<unsigned long long>(__popc(km & same)));
}

// selection.cpp:163-175: if nothing cleared tau keep the fallback_k best z,
// ties to the lowest flat index.  One CTA per job; k rounds of argmax.
__global__ void exact_fallback_kernel(const DJob* __restrict__ jobs,
                                      const int* __restrict__ batch_jobs,
                                      const int64_t* __restrict__ off,
                                      const float* __restrict__ scores,
                                      const double2* __restrict__ stats,
                                      const unsigned long long* __restrict__ kept,
                                      uint32_t* counts, int64_t nt, int bs, int fallback_k,
                                      unsigned long long* n_fallback) {
  const int lj = blockIdx.x;
  if (kept[lj] != 0) return;
  const DJob& jb = jobs[batch_jobs[lj]];
  const int64_t n = off[lj + 1] - off[lj];
  const float* s = scores + off[lj];
  const double2 st = stats[lj];
  __shared__ double bz[32];
  __shared__ int64_t bi[32];
  __shared__ int64_t last_pick;
  __shared__ double last_z;
  const int k = static_cast<int>(fallback_k < n ? fallback_k : n);
  if (threadIdx.x == 0) {
    last_pick = -1;
    last_z = INFINITY;
    atomicAdd(n_fallback, 1ull);
  }
  __syncthreads();
  for (int round = 0; round < k; ++round) {
    // best (z, -index) strictly after (last_z, last_pick) in the order
    // z descending then index ascending.
    double best = -INFINITY;
    int64_t besti = -1;
    for (int64_t x = threadIdx.x; x < n; x += blockDim.x) {
      const double z = zscore(s[x], st);
      const bool after = z < last_z || (z == last_z && x > last_pick);
      if (!after) continue;
      if (besti < 0 || z > best || (z == best && x < besti)) {
        best = z;
        besti = x;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double oz = __shfl_xor_sync(0xFFFFFFFFu, best, o);
      const int64_t oi = __shfl_xor_sync(0xFFFFFFFFu, besti, o);
      if (oi >= 0 && (besti < 0 || oz > best || (oz == best && oi < besti))) {
        best = oz;
        besti = oi;
      }
    }
    if (threadIdx.x % 32 == 0) {
      bz[threadIdx.x / 32] = best;
      bi[threadIdx.x / 32] = besti;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < static_cast<int>(blockDim.x / 32); ++w)
        if (bi[w] >= 0 && (bi[0] < 0 || bz[w] > bz[0] || (bz[w] == bz[0] && bi[w] < bi[0]))) {
          bz[0] = bz[w];
          bi[0] = bi[w];
        }
      if (bi[0] >= 0) {
        int64_t u, v;
        band_uv(bi[0], nt, jb.width, &u, &v);
        add_count(jb, counts, nt, bs, u, v);
      }
      last_pick = bi[0];
      last_z = bz[0];
    }
    __syncthreads();
  }
}

}  // namespace mask
}  // namespace rp

// =========================================================================
using namespace rp;
using namespace rp::mask;

namespace {

// Device buffer: stream-ordered (temporaries of one build) or, with
// persistent = true, a plain allocation owned by a plan.
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  bool persistent = false;
  DevBuf() = default;
  DevBuf(size_t count, cudaStream_t st, bool keep = false) : n(count), s(st), persistent(keep) {
    if (!count) return;
    if (keep) RP_CUDA(cudaMalloc(reinterpret_cast<void**>(&p), sizeof(T) * count));
    else RP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(T) * count, st));
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), s(o.s), persistent(o.persistent) {
    o.p = nullptr;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    std::swap(p, o.p);
    std::swap(n, o.n);
    std::swap(s, o.s);
    std::swap(persistent, o.persistent);
    return *this;
  }
  ~DevBuf() {
    if (!p) return;
    if (persistent) cudaFree(p);
    else cudaFreeAsync(p, s);
  }
  void upload(const T* h, size_t count) {
    RP_CUDA(cudaMemcpyAsync(p, h, sizeof(T) * count, cudaMemcpyHostToDevice, s));
  }
};

int bit_length(uint64_t x) {
  int b = 0;
  while (x) {
    ++b;
    x >>= 1;
  }
  return b;
}

}  // namespace

struct rp_plan_s {
  rp_grid g{};
  rp_config c{};
  uint64_t seed = 0;
  rp_build_options o{};
  std::vector<plan::Job> jobs;
  std::vector<DJob> djobs;
  int cmin = 0, amin = 0;
  size_t words = 0;  // 32-bit words of the padded mask buffer
  // device state (allocated with the stream of the first build)
  cudaStream_t s = nullptr;
  DevBuf<DJob> d_jobs;
  DevBuf<uint32_t> base;    // intra-frame + full-band bits
  DevBuf<uint32_t> cached;  // static mode: the full mask
  bool base_ready = false, static_ready = false;
  int64_t retained = 0, sampled = 0, scored = 0;
  FastEngine* fast = nullptr;
  int fast_heads = 0, fast_dim = 0;
  // Builds of one plan may come from any stream: they are serialised on the
  // host (mu) and on the device (each build's stream first waits for the
  // previous build's completion event), because they share the cached masks
  // and the fast engine's scratch buffers.  A plan belongs to the device of
  // its first build.
  std::mutex mu;
  cudaEvent_t done_ev = nullptr;
  int dev = -1;
  ~rp_plan_s() {
    if (done_ev) {
      cudaEventSynchronize(done_ev);
      cudaEventDestroy(done_ev);
    }
    fast_engine_destroy(fast);
  }
};

namespace {

void make_jobs(rp_plan_s& P) {
  const rp_grid& g = P.g;
  const rp_config& c = P.c;
  const int64_t nt = g.tokens_per_frame;
  int64_t score_ordinal = 0;
  for (int i = 0; i < g.n_frames; ++i)
    for (int j = 0; j < g.n_frames; ++j) {
      const int64_t t = std::llabs(static_cast<long long>(i) - j);
      if (t < 1) continue;
      const bool ret = plan::frame_retained(t, c, g);
      if (!P.o.disable_split && !ret) continue;
      plan::Job jb{};
      jb.i = i;
      jb.j = j;
      jb.tier = plan::distance_tier(i, j, c, g);
      jb.width = plan::window_width(i, j, c, g);
      jb.n = ret ? plan::band_pairs(nt, jb.width) : 0;
      jb.stream_seed = pair_seed(P.seed, i, j);
      if (c.mode == RP_STATIC_RATIO) {
        jb.param = jb.tier == 0 ? 1.0 : (jb.tier == 1 ? c.near_param : c.far_param);
        if (jb.param >= 1.0) {
          jb.kind = plan::kFullBand;
        } else {
          if (jb.n == 0)
            throw std::invalid_argument(
                "build_mask: disable_split samples a pruned frame pair (empty candidate set; "
                "the reference divides by zero here)");
          jb.kind = plan::kSample;
          jb.k = static_cast<int64_t>(std::floor(static_cast<double>(jb.n) * jb.param));
          if (jb.k < 1) jb.k = 1;
        }
      } else {
        jb.param = jb.tier == 0 ? -std::numeric_limits<double>::infinity()
                                : (jb.tier == 1 ? c.near_param : c.far_param);
        if (jb.tier == 0) jb.kind = plan::kFullBand;
        else jb.kind = jb.n > 0 ? plan::kScore : plan::kEmpty;
        // multi-GPU split: another shard scores this pair
        if (jb.kind == plan::kScore && (score_ordinal++ % P.o.shard_count) != P.o.shard_index)
          jb.kind = plan::kEmpty;
      }
      P.jobs.push_back(jb);
    }
  const int bs = g.block_size;
  for (const plan::Job& jb : P.jobs) {
    DJob d{};
    d.i = jb.i;
    d.j = jb.j;
    d.kind = jb.kind;
    d.width = jb.width;
    d.n = jb.n;
    d.k = jb.k;
    d.param = jb.param;
    d.seed = jb.stream_seed;
    const int64_t qi = static_cast<int64_t>(jb.i) * nt, kj = static_cast<int64_t>(jb.j) * nt;
    d.r0 = static_cast<int32_t>(qi / bs);
    d.c0 = static_cast<int32_t>(kj / bs);
    d.tr = static_cast<int32_t>((qi + nt - 1) / bs - d.r0 + 1);
    d.tc = static_cast<int32_t>((kj + nt - 1) / bs - d.c0 + 1);
    P.djobs.push_back(d);
  }
  P.cmin = plan::count_threshold(c.col_threshold, bs);
  P.amin = plan::count_threshold(c.mask_threshold, bs);
  P.retained = static_cast<int64_t>(P.jobs.size());
}

int apply_threads(int bs) { return bs >= 1024 ? 1024 : (bs < 32 ? 32 : bs); }

void launch_apply(rp_plan_s& P, const std::vector<Item>& items, const uint32_t* counts,
                  uint32_t* words, int mode, cudaStream_t s) {
  if (items.empty()) return;
  DevBuf<Item> d_items(items.size(), s);
  d_items.upload(items.data(), items.size());
  const int64_t chunk = 1 << 30;  // grid.x limit safety
  for (int64_t b = 0; b < static_cast<int64_t>(items.size()); b += chunk) {
    const int64_t nb = std::min<int64_t>(chunk, items.size() - b);
    apply_kernel<<<static_cast<unsigned>(nb), apply_threads(P.g.block_size), 0, s>>>(
        P.d_jobs.p, d_items.p + b, counts, words, P.g.tokens_per_frame, P.g.block_size,
        P.g.row_bytes, P.cmin, P.amin, mode);
    RP_LAUNCHED();
  }
}

void tiles_of(const rp_plan_s& P, int job, std::vector<Item>& out) {
  const DJob& d = P.djobs[job];
  for (int32_t r = 0; r < d.tr; ++r)
    for (int32_t c = 0; c < d.tc; ++c) out.push_back(Item{job, r, c});
}

// Intra-frame rectangles + every full-band pair, once per plan.
void build_base(rp_plan_s& P, cudaStream_t s) {
  const rp_grid& g = P.g;
  P.base = DevBuf<uint32_t>(P.words, s, true);
  RP_CUDA(cudaMemsetAsync(P.base.p, 0, P.words * 4, s));
  const int span = static_cast<int>((g.tokens_per_frame + g.block_size - 1) / g.block_size + 1);
  intra_kernel<<<g.n_frames, 256, 0, s>>>(P.base.p, g.n_frames, g.tokens_per_frame,
                                          g.block_size, g.row_bytes, span);
  RP_LAUNCHED();
  std::vector<Item> items;
  for (int jx = 0; jx < static_cast<int>(P.djobs.size()); ++jx)
    if (P.djobs[jx].kind == plan::kFullBand) tiles_of(P, jx, items);
  launch_apply(P, items, nullptr, P.base.p, 0, s);
  P.base_ready = true;
}

// Batches of jobs of one kind whose per-job sizes (`size(job)`) sum to at
// most `cap` elements (a single oversized job forms its own batch).
template <class F>
std::vector<std::vector<int>> batches(const rp_plan_s& P, int kind, int64_t cap, F size) {
  std::vector<std::vector<int>> out;
  std::vector<int> cur;
  int64_t tot = 0;
  for (int jx = 0; jx < static_cast<int>(P.djobs.size()); ++jx) {
    if (P.djobs[jx].kind != kind) continue;
    const int64_t sz = size(P.djobs[jx]);
    if (!cur.empty() && tot + sz > cap) {
      out.push_back(cur);
      cur.clear();
      tot = 0;
    }
    cur.push_back(jx);
    tot += sz;
  }
  if (!cur.empty()) out.push_back(cur);
  return out;
}

// Count buffers for a batch: one [tr][tc][B] block per job.
int64_t assign_counts(rp_plan_s& P, const std::vector<int>& batch) {
  int64_t off = 0;
  for (int jx : batch) {
    P.djobs[jx].cnt_off = off;
    off += static_cast<int64_t>(P.djobs[jx].tr) * P.djobs[jx].tc * P.g.block_size;
  }
  return off;
}

constexpr int64_t kDrawCap = int64_t{1} << 28;   // draws per static batch
// scores per exact batch (8 GB of fp32): every frame pair of a batch runs its
// sequential stats chains concurrently, so fewer, larger batches cost less
constexpr int64_t kScoreCap = int64_t{1} << 31;

void build_static(rp_plan_s& P, uint32_t* words, cudaStream_t s) {
  const int bs = P.g.block_size;
  const int64_t nt = P.g.tokens_per_frame;
  auto bl = batches(P, plan::kSample, kDrawCap, [](const DJob& d) { return d.k; });
  for (auto& batch : bl) {
    const int nj = static_cast<int>(batch.size());
    std::vector<int64_t> off(nj + 1, 0);
    int64_t max_n = 1;
    for (int x = 0; x < nj; ++x) {
      off[x + 1] = off[x] + P.djobs[batch[x]].k;
      max_n = std::max(max_n, P.djobs[batch[x]].n);
    }
    const int64_t total = off[nj];
    const int bits = std::max(1, bit_length(static_cast<uint64_t>(max_n - 1)));
    const int jbits = std::max(1, bit_length(static_cast<uint64_t>(nj - 1)));
    if (2 * bits + jbits > 64 || max_n > (int64_t{1} << 31))
      throw std::out_of_range("build_mask: frame pair too large for the sampling key");
    const int64_t ncnt = assign_counts(P, batch);
    P.d_jobs.upload(P.djobs.data(), P.djobs.size());
    DevBuf<int> d_batch(nj, s);
    d_batch.upload(batch.data(), nj);
    DevBuf<int64_t> d_off(nj + 1, s);
    d_off.upload(off.data(), nj + 1);
    DevBuf<uint64_t> keys(total, s), sorted(total, s);
    DevBuf<int32_t> prev(total, s), tlast(total, s);
    DevBuf<uint32_t> counts(ncnt, s);
    RP_CUDA(cudaMemsetAsync(tlast.p, 0xFF, sizeof(int32_t) * total, s));
    RP_CUDA(cudaMemsetAsync(counts.p, 0, sizeof(uint32_t) * ncnt, s));
    const unsigned grid = static_cast<unsigned>((total + 255) / 256);
    fy_draw_kernel<<<grid, 256, 0, s>>>(P.d_jobs.p, d_batch.p, d_off.p, nj, total, bits, keys.p);
    RP_LAUNCHED();
    size_t tmp_bytes = 0;
    const int end_bit = 2 * bits + jbits;
    // Only the (job, target) bits are sorted: the keys are generated in
    // (job, step) order and the LSD radix sort is stable, so each target's
    // steps stay in step order without sorting the low `bits` step bits
    // (4 passes instead of 7 at the Wan grid).
    RP_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, keys.p, sorted.p, total, bits,
                                           end_bit, s));
    DevBuf<uint8_t> tmp(tmp_bytes, s);
    RP_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, keys.p, sorted.p, total, bits, end_bit,
                                           s));
    count_launch();
    fy_link_kernel<<<grid, 256, 0, s>>>(sorted.p, total, bits, d_off.p, prev.p, tlast.p,
                                        P.d_jobs.p, d_batch.p);
    RP_LAUNCHED();
    fy_count_kernel<<<grid, 256, 0, s>>>(P.d_jobs.p, d_batch.p, d_off.p, nj, total, prev.p,
                                         tlast.p, counts.p, nt, bs);
    RP_LAUNCHED();
    std::vector<Item> items;
    for (int jx : batch) tiles_of(P, jx, items);
    launch_apply(P, items, counts.p, words, 1, s);
    P.sampled += total;
  }
}

Feat make_feat(const rp_tensor* q, const rp_tensor* k, int heads) {
  Feat f;
  f.q = q->data;
  f.k = k->data;
  f.dtype = q->dtype;
  f.q_ts = q->token_stride;
  f.q_hs = q->head_stride;
  f.k_ts = k->token_stride;
  f.k_hs = k->head_stride;
  f.heads = heads;
  f.d = q->head_dim;
  f.inv_sqrt_d = 1.0 / std::sqrt(static_cast<double>(q->head_dim));
  return f;
}

void build_dynamic_exact(rp_plan_s& P, const Feat& f, uint32_t* words, int64_t* rechecked,
                         int64_t* fallbacks, cudaStream_t s) {
  const int bs = P.g.block_size;
  const int64_t nt = P.g.tokens_per_frame;
  auto bl = batches(P, plan::kScore, kScoreCap, [](const DJob& d) { return d.n; });
  (void)rechecked;
  for (auto& batch : bl) {
    const int nj = static_cast<int>(batch.size());
    std::vector<int64_t> off(nj + 1, 0);
    for (int x = 0; x < nj; ++x) off[x + 1] = off[x] + P.djobs[batch[x]].n;
    const int64_t total = off[nj];
    const int64_t ncnt = assign_counts(P, batch);
    P.d_jobs.upload(P.djobs.data(), P.djobs.size());
    DevBuf<int> d_batch(nj, s);
    d_batch.upload(batch.data(), nj);
    DevBuf<int64_t> d_off(nj + 1, s);
    d_off.upload(off.data(), nj + 1);
    DevBuf<float> scores(total, s);
    DevBuf<double2> stats(nj, s);
    DevBuf<double> inv_den(nj, s);
    DevBuf<uint32_t> counts(ncnt, s);
    DevBuf<unsigned long long> kept(nj + 1, s);
    RP_CUDA(cudaMemsetAsync(counts.p, 0, sizeof(uint32_t) * ncnt, s));
    RP_CUDA(cudaMemsetAsync(kept.p, 0, sizeof(unsigned long long) * (nj + 1), s));
    const unsigned grid = static_cast<unsigned>((total + 255) / 256);
    exact_scores_kernel<<<grid, 256, 0, s>>>(P.d_jobs.p, d_batch.p, d_off.p, nj, total, f, nt,
                                             scores.p);
    RP_LAUNCHED();
    seq_stats_kernel<<<nj, kSeqThreads, 0, s>>>(d_off.p, nj, scores.p, stats.p, inv_den.p);
    RP_LAUNCHED();
    exact_select_kernel<<<grid, 256, 0, s>>>(P.d_jobs.p, d_batch.p, d_off.p, nj, total,
                                             scores.p, stats.p, inv_den.p, counts.p, kept.p, nt, bs);
    RP_LAUNCHED();
    exact_fallback_kernel<<<nj, 256, 0, s>>>(P.d_jobs.p, d_batch.p, d_off.p, scores.p, stats.p,
                                             kept.p, counts.p, nt, bs, P.c.fallback_k,
                                             kept.p + nj);
    RP_LAUNCHED();
    std::vector<Item> items;
    for (int jx : batch) tiles_of(P, jx, items);
    launch_apply(P, items, counts.p, words, 1, s);
    if (fallbacks) {
      unsigned long long h = 0;
      RP_CUDA(cudaMemcpyAsync(&h, kept.p + nj, sizeof(h), cudaMemcpyDeviceToHost, s));
      RP_CUDA(cudaStreamSynchronize(s));
      *fallbacks += static_cast<int64_t>(h);
    }
    P.scored += total;
  }
}

}  // namespace

extern "C" {

void rp_build_options_defaults(rp_build_options* o) {
  o->disable_split = 0;
  o->score_engine = 0;
  o->recheck_delta = 0.0;
  o->shard_index = 0;
  o->shard_count = 1;
}

rp_status rp_plan_create(const rp_grid* g, const rp_config* c, uint64_t seed,
                         const rp_build_options* opt, rp_plan* out) {
  return guarded([&] {
    check_grid(g);
    if (!c) throw std::invalid_argument("config: null");
    plan::validate(*c);
    std::unique_ptr<rp_plan_s> p(new rp_plan_s);
    p->g = *g;
    p->c = *c;
    p->seed = seed;
    if (opt) p->o = *opt;
    else rp_build_options_defaults(&p->o);
    if (p->o.shard_count < 1 || p->o.shard_index < 0 || p->o.shard_index >= p->o.shard_count)
      throw std::invalid_argument("build options: shard_index must be in [0, shard_count)");
    make_jobs(*p);
    p->words = static_cast<size_t>((g->blocks_per_dim * g->row_bytes + 3) / 4);
    *out = p.release();
  });
}

void rp_plan_destroy(rp_plan p) {
  delete p;  // waits for the last build (done_ev) before freeing device state
}

rp_status rp_plan_build_mask(rp_plan P, const rp_tensor* q, const rp_tensor* k,
                             int n_score_heads, uint8_t* mask_bits_dev, rp_build_stats* stats,
                             rp_stream stream) {
  return guarded([&] {
    require_device();
    if (!P) throw std::invalid_argument("build_mask: null plan");
    if (!mask_bits_dev) throw std::invalid_argument("build_mask: null mask buffer");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const rp_grid& g = P->g;
    const bool dynamic = P->c.mode == RP_DYNAMIC_THRESHOLD;
    if (dynamic) {
      if (!q || !k || !q->data || !k->data)
        throw std::invalid_argument("build_mask: dynamic mode needs features");
      if (n_score_heads < 1 || n_score_heads > q->heads || q->heads != k->heads ||
          q->head_dim != k->head_dim || q->dtype != k->dtype || q->head_dim < 1)
        throw std::invalid_argument("feature batch: queries/keys shape mismatch");
      if (q->tokens < g.total_tokens || k->tokens < g.total_tokens)
        throw std::invalid_argument("build_mask: feature batch too short");
    }
    std::lock_guard<std::mutex> lock(P->mu);
    int dev = 0;
    RP_CUDA(cudaGetDevice(&dev));
    if (P->dev < 0) P->dev = dev;
    if (P->dev != dev)
      throw std::invalid_argument("build_mask: plan was created on another device");
    if (P->done_ev) RP_CUDA(cudaStreamWaitEvent(s, P->done_ev, 0));
    else RP_CUDA(cudaEventCreateWithFlags(&P->done_ev, cudaEventDisableTiming));
    // whatever happens below, later builds order after this one's work
    struct Record {
      rp_plan_s* P;
      cudaStream_t s;
      ~Record() { cudaEventRecord(P->done_ev, s); }
    } record{P, s};
    if (!P->d_jobs.p) {
      P->s = s;
      P->d_jobs = DevBuf<DJob>(std::max<size_t>(P->djobs.size(), 1), s, true);
      if (!P->djobs.empty()) P->d_jobs.upload(P->djobs.data(), P->djobs.size());
    }
    if (!P->base_ready) build_base(*P, s);
    const size_t bytes = static_cast<size_t>(g.blocks_per_dim * g.row_bytes);
    int64_t rechecked = 0, fallbacks = 0;
    if (!dynamic) {
      if (!P->static_ready) {
        P->cached = DevBuf<uint32_t>(P->words, s, true);
        RP_CUDA(cudaMemcpyAsync(P->cached.p, P->base.p, P->words * 4, cudaMemcpyDeviceToDevice, s));
        stage_begin(kStageStatic, s);
        build_static(*P, P->cached.p, s);
        stage_end(kStageStatic, s);
        P->static_ready = true;
      }
      RP_CUDA(cudaMemcpyAsync(mask_bits_dev, P->cached.p, bytes, cudaMemcpyDeviceToDevice, s));
    } else {
      P->scored = 0;  // BuildTimings::scored_pairs of this build
      DevBuf<uint32_t> work(P->words, s);
      RP_CUDA(cudaMemcpyAsync(work.p, P->base.p, P->words * 4, cudaMemcpyDeviceToDevice, s));
      const Feat f = make_feat(q, k, n_score_heads);
      int engine = P->o.score_engine;
      if (engine == 0)
        engine = (q->dtype == RP_BF16 && fast_engine_supported(g, q->head_dim, n_score_heads))
                     ? 1 : 2;
      if (engine == 1) {
        if (q->dtype != RP_BF16 || !fast_engine_supported(g, q->head_dim, n_score_heads))
          throw std::invalid_argument(
              "build_mask: tensor-core scoring needs bf16 features, B in {32,64,128} and "
              "head_dim*heads in {64..512, multiple of 64}");
        if (!P->fast || P->fast_heads != n_score_heads || P->fast_dim != q->head_dim) {
          fast_engine_destroy(P->fast);
          P->fast = nullptr;
          P->fast = fast_engine_create(g, P->djobs, P->cmin, P->amin, n_score_heads,
                                       q->head_dim, s);
          P->fast_heads = n_score_heads;
          P->fast_dim = q->head_dim;
        }
        for (const DJob& d : P->djobs)
          if (d.kind == plan::kScore) P->scored += d.n;
        FastResult fr;
        fast_engine_run(P->fast, q, k, f, work.p, s,
                        P->o.recheck_delta > 0 ? P->o.recheck_delta : 1e-5, P->c.fallback_k,
                        stats != nullptr, &fr);
        rechecked = fr.rechecked;
        fallbacks = fr.fallbacks;
      } else {
        stage_begin(kStageExactScore, s);
        build_dynamic_exact(*P, f, work.p, &rechecked, stats ? &fallbacks : nullptr, s);
        stage_end(kStageExactScore, s);
      }
      RP_CUDA(cudaMemcpyAsync(mask_bits_dev, work.p, bytes, cudaMemcpyDeviceToDevice, s));
    }
    if (stats) {
      std::vector<uint8_t> h(bytes);
      RP_CUDA(cudaMemcpyAsync(h.data(), mask_bits_dev, bytes, cudaMemcpyDeviceToHost, s));
      RP_CUDA(cudaStreamSynchronize(s));
      int64_t act = 0;
      for (uint8_t b : h) act += __builtin_popcount(b);
      stats->retained_frame_pairs = P->retained;
      stats->scored_pairs = P->scored;
      stats->sampled_pairs = P->sampled;
      stats->rechecked_pairs = rechecked;
      stats->fallback_frame_pairs = fallbacks;
      stats->active_blocks = act;
    }
  });
}

rp_status rp_build_mask(const rp_grid* g, const rp_config* c, uint64_t seed,
                        const rp_build_options* opt, const rp_tensor* q, const rp_tensor* k,
                        int n, uint8_t* bits, rp_build_stats* st, rp_stream s) {
  rp_plan p = nullptr;
  rp_status r = rp_plan_create(g, c, seed, opt, &p);
  if (r != RP_OK) return r;
  r = rp_plan_build_mask(p, q, k, n, bits, st, s);
  if (r == RP_OK) {
    const cudaError_t e = cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(s));
    if (e != cudaSuccess) {
      set_error(cudaGetErrorString(e));
      r = RP_CUDA_ERROR;
    }
  }
  rp_plan_destroy(p);
  return r;
}

// ------------------------------------------------ selection operators ------
namespace {

int64_t band_count(const rp_band* b) {
  if (!b) throw std::invalid_argument("band: null");
  if (b->tokens_per_frame < 1 || b->width < 0)
    throw std::invalid_argument("band: bad geometry");
  return b->retained ? plan::band_pairs(b->tokens_per_frame, b->width) : 0;
}

}  // namespace

rp_status rp_static_select(const rp_band* band, double ratio, uint64_t seed, int64_t* uv_dev,
                           int64_t cap, int64_t* count, rp_stream stream) {
  return guarded([&] {
    require_device();
    if (!count) throw std::invalid_argument("static_select: null count");
    const int64_t n = band_count(band);
    *count = 0;
    if (n == 0) return;
    if (!(ratio > 0.0 && ratio <= 1.0))
      throw std::invalid_argument("static_select: ratio must be in (0, 1]");
    int64_t k = static_cast<int64_t>(std::floor(static_cast<double>(n) * ratio));
    if (k < 1) k = 1;
    if (k > cap || !uv_dev) throw std::out_of_range("static_select: output capacity");
    if (n > (int64_t{1} << 31)) throw std::out_of_range("static_select: band too large");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    DJob jb{};
    jb.i = band->frame_i;
    jb.j = band->frame_j;
    jb.width = band->width;
    jb.n = n;
    jb.k = k;
    jb.seed = pair_seed(seed, band->frame_i, band->frame_j);
    const int bits = std::max(1, bit_length(static_cast<uint64_t>(n - 1)));
    DevBuf<DJob> d_job(1, s);
    d_job.upload(&jb, 1);
    const int zero = 0;
    DevBuf<int> d_batch(1, s);
    d_batch.upload(&zero, 1);
    const int64_t off[2] = {0, k};
    DevBuf<int64_t> d_off(2, s);
    d_off.upload(off, 2);
    DevBuf<uint64_t> keys(k, s), sorted(k, s);
    DevBuf<int32_t> prev(k, s), tlast(k, s);
    RP_CUDA(cudaMemsetAsync(tlast.p, 0xFF, sizeof(int32_t) * k, s));
    const unsigned grid = static_cast<unsigned>((k + 255) / 256);
    fy_draw_kernel<<<grid, 256, 0, s>>>(d_job.p, d_batch.p, d_off.p, 1, k, bits, keys.p);
    RP_LAUNCHED();
    size_t tmp_bytes = 0;
    RP_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, keys.p, sorted.p, k, bits,
                                           2 * bits + 1, s));  // stable: see build_static
    DevBuf<uint8_t> tmp(tmp_bytes, s);
    RP_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, keys.p, sorted.p, k, bits,
                                           2 * bits + 1, s));
    count_launch();
    fy_link_kernel<<<grid, 256, 0, s>>>(sorted.p, k, bits, d_off.p, prev.p, tlast.p, d_job.p,
                                        d_batch.p);
    RP_LAUNCHED();
    fy_value_kernel<<<grid, 256, 0, s>>>(d_job.p, k, prev.p, tlast.p, band->tokens_per_frame,
                                         uv_dev);
    RP_LAUNCHED();
    RP_CUDA(cudaStreamSynchronize(s));
    *count = k;
  });
}

rp_status rp_proxy_scores(const rp_tensor* q, const rp_tensor* k, int n_heads,
                          const rp_band* band, float* scores_dev, rp_stream stream) {
  return guarded([&] {
    require_device();
    if (n_heads < 1) throw std::invalid_argument("proxy_scores: batch has no heads");
    if (!q || !k || !q->data || !k->data || q->heads < n_heads || k->heads < n_heads ||
        q->head_dim != k->head_dim || q->dtype != k->dtype)
      throw std::invalid_argument("feature batch: queries/keys shape mismatch");
    const int64_t n = band_count(band);
    const int64_t nt = band->tokens_per_frame;
    const int64_t qi = static_cast<int64_t>(band->frame_i) * nt;
    const int64_t kj = static_cast<int64_t>(band->frame_j) * nt;
    if (band->frame_i < 0 || band->frame_j < 0 || qi + nt > q->tokens || kj + nt > k->tokens)
      throw std::out_of_range("proxy_scores: frame outside feature batch");
    if (n == 0) return;
    if (!scores_dev) throw std::invalid_argument("proxy_scores: null output");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    DJob jb{};
    jb.i = band->frame_i;
    jb.j = band->frame_j;
    jb.width = band->width;
    jb.n = n;
    DevBuf<DJob> d_job(1, s);
    d_job.upload(&jb, 1);
    const int zero = 0;
    DevBuf<int> d_batch(1, s);
    d_batch.upload(&zero, 1);
    const int64_t off[2] = {0, n};
    DevBuf<int64_t> d_off(2, s);
    d_off.upload(off, 2);
    const Feat f = make_feat(q, k, n_heads);
    exact_scores_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(
        d_job.p, d_batch.p, d_off.p, 1, n, f, nt, scores_dev);
    RP_LAUNCHED();
    RP_CUDA(cudaStreamSynchronize(s));
  });
}

rp_status rp_normalize_scores(const float* scores_dev, int64_t n, double* z_dev, double* mean,
                              double* stddev, rp_stream stream) {
  return guarded([&] {
    require_device();
    if (n < 0) throw std::invalid_argument("normalize_scores: negative count");
    if (n == 0) {
      if (mean) *mean = 0.0;
      if (stddev) *stddev = 0.0;
      return;
    }
    if (!scores_dev || !z_dev) throw std::invalid_argument("normalize_scores: null buffer");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t off[2] = {0, n};
    DevBuf<int64_t> d_off(2, s);
    d_off.upload(off, 2);
    DevBuf<double2> st(1, s);
    seq_stats_kernel<<<1, kSeqThreads, 0, s>>>(d_off.p, 1, scores_dev, st.p, nullptr);
    RP_LAUNCHED();
    zscore_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(scores_dev, n, st.p,
                                                                          z_dev);
    RP_LAUNCHED();
    double2 h;
    RP_CUDA(cudaMemcpyAsync(&h, st.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    RP_CUDA(cudaStreamSynchronize(s));
    if (mean) *mean = h.x;
    if (stddev) *stddev = h.y;
  });
}

rp_status rp_dynamic_select(const rp_band* band, const double* z_dev, int64_t n,
                            double threshold, int fallback_k, int64_t* uv_dev, int64_t cap,
                            int64_t* count, rp_stream stream) {
  return guarded([&] {
    require_device();
    if (!count) throw std::invalid_argument("dynamic_select: null count");
    const int64_t pc = band_count(band);
    if (n != pc) throw std::invalid_argument("dynamic_select: score count mismatch");
    *count = 0;
    if (n == 0) return;
    if (!z_dev || !uv_dev) throw std::invalid_argument("dynamic_select: null buffer");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t tiles = (n + kSelTile - 1) / kSelTile;
    DevBuf<int32_t> cnt(tiles, s);
    keep_count_kernel<<<static_cast<unsigned>(tiles), 256, 0, s>>>(z_dev, n, threshold, cnt.p);
    RP_LAUNCHED();
    std::vector<int32_t> hc(tiles);
    RP_CUDA(cudaMemcpyAsync(hc.data(), cnt.p, sizeof(int32_t) * tiles, cudaMemcpyDeviceToHost, s));
    RP_CUDA(cudaStreamSynchronize(s));
    std::vector<int64_t> off(tiles);
    int64_t kept = 0;
    for (int64_t t = 0; t < tiles; ++t) {
      off[t] = kept;
      kept += hc[t];
    }
    if (kept > 0) {
      if (kept > cap) throw std::out_of_range("dynamic_select: output capacity");
      DevBuf<int64_t> d_off(tiles, s);
      d_off.upload(off.data(), tiles);
      keep_scatter_kernel<<<static_cast<unsigned>(tiles), 256, 0, s>>>(
          z_dev, n, threshold, d_off.p, band->tokens_per_frame, band->width, uv_dev);
      RP_LAUNCHED();
      RP_CUDA(cudaStreamSynchronize(s));
      *count = kept;
      return;
    }
    const int64_t k = std::min<int64_t>(std::max(fallback_k, 0), n);
    if (k > cap) throw std::out_of_range("dynamic_select: output capacity");
    if (k > 0) {
      fallback_pick_kernel<<<1, 1024, 0, s>>>(z_dev, n, static_cast<int>(k),
                                              band->tokens_per_frame, band->width, uv_dev);
      RP_LAUNCHED();
      RP_CUDA(cudaStreamSynchronize(s));
    }
    *count = k;
  });
}

rp_status rp_token_mask_to_blocks(const uint8_t* token_bits_dev, int64_t dim, int block_size,
                                  uint8_t* block_bits_dev, int* uniform, rp_stream stream) {
  return guarded([&] {
    require_device();
    if (block_size < 1 || dim < 1 || dim % block_size)
      throw std::invalid_argument("token mask: block size must divide the mask dimension");
    if (!token_bits_dev || !block_bits_dev) throw std::invalid_argument("token mask: null buffer");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t nb = dim / block_size, brb = (nb + 7) / 8;
    const size_t words = static_cast<size_t>((nb * brb + 3) / 4);
    DevBuf<uint32_t> w(words, s);
    DevBuf<unsigned long long> bad(1, s);
    RP_CUDA(cudaMemsetAsync(w.p, 0, words * 4, s));
    RP_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(unsigned long long), s));
    token_to_block_kernel<<<static_cast<unsigned>(nb * nb), 256, 0, s>>>(
        token_bits_dev, dim, (dim + 7) / 8, block_size, nb, brb, w.p, bad.p);
    RP_LAUNCHED();
    RP_CUDA(cudaMemcpyAsync(block_bits_dev, w.p, static_cast<size_t>(nb * brb),
                            cudaMemcpyDeviceToDevice, s));
    unsigned long long h = 0;
    RP_CUDA(cudaMemcpyAsync(&h, bad.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    RP_CUDA(cudaStreamSynchronize(s));
    if (uniform) *uniform = h == 0;
  });
}

}  // extern "C"
