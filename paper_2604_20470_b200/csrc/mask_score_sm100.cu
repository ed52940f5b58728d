// K2/K3: dynamic-threshold proxy scoring on the tensor cores (sm_100a).
//
// Reference semantics (selection.cpp:93-185): per ordered frame pair (i, j)
// every band pair (u, v), |u - v| <= w, gets s = mean_h(q_u . k_v)/sqrt(d)
// over the H_f scoring heads; s is standardised by the pair's population
// mean / std and kept iff z >= tau; kept pairs are counted per tile column
// and aggregated by the theta_c / theta_m rule (mask.cpp:87-125).
//
// B200 mapping.  The band of a frame pair is covered by 128 x 128 token tiles
// (items).  One tcgen05 MMA chain per item computes S = Q' K'^T with
// Q' = [q_h0 | q_h1 | ...] (the first H_f heads are adjacent in the [S, H, d]
// layout, so the concatenation is one TMA box per head and 64-wide chunk):
// K = H_f * d.  Bf16 products are exact, so a fast score differs from the
// reference's double-accumulated score only by the fp32 accumulation inside
// the tensor core, bounded per pair by kappa * |q'_u| |k'_v| (Cauchy-Schwarz).
//   pass 1 (stats): per row fp32 sums of a tile, carried in fp64 across the
//          unit (one frame pair, one tile row), reduced once per unit to
//          (n, mean, M2); units are then Chan-merged per frame pair in a
//          fixed order (deterministic mu / sigma).
//   pass 2 (select): z = (s - mu)/(sigma + 1e-8); decided directly when
//          |z - tau| exceeds the pair's error bound + delta_floor, otherwise
//          appended to the CTA's undecided region; kept bits -> per-column
//          counts by 32 x 32 bit transposes -> the frame pair's [tile][B]
//          count buffer.
//   recheck: every queued pair is re-scored exactly as the reference does
//          (fp64, sequential d, separate multiply / add, float cast).
//   apply: theta_c / theta_m per tile, one warp per tile.
// Frame pairs with no kept pair take the fallback_k rule on exact scores
// (it can only change a tile when fallback_k >= ceil(theta_c * B)).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "internal.hpp"
#include "mask_build.cuh"
#include "mask_common.cuh"
#include "plan.hpp"
#include "tmap.hpp"

namespace rp {
namespace mask {

// Everything the epilogue needs about one 128 x 128 item, precomputed on the
// host so an item costs three 16-byte loads and 32-bit index math only.
struct alignas(16) ScoreItem {
  int32_t job;       // index into the engine's job array
  int32_t tr;        // 128-token tile row (global)
  int32_t tc;        // 128-token tile column (global)
  int32_t width;     // the job's band half-width, clamped to N_t
  int32_t u0, v0;    // tr * 128 - first token of frame i, tc * 128 - first of frame j
  int32_t rr0, cc0;  // the tile's first block row / column in the job's count rectangle
  int32_t jtr, jtc;  // the job's count rectangle (block rows / columns)
  long long cnt_off; // the job's [tr][tc][B] count offset
};
static_assert(sizeof(ScoreItem) == 48, "ScoreItem is loaded as three int4");

RP_DEV ScoreItem load_item(const ScoreItem* items, long long i) {
  const int4* src = reinterpret_cast<const int4*>(items + i);
  ScoreItem x;
  int4* dst = reinterpret_cast<int4*>(&x);
  dst[0] = __ldg(src);
  dst[1] = __ldg(src + 1);
  dst[2] = __ldg(src + 2);
  return x;
}

struct SParams {
  const DJob* jobs;
  const ScoreItem* items;
  long long n_items;
  const int2* units;  // [n_units] item ranges [x, y), see UnitCursor
  int n_units;
  int nt, bs, lg_bs, cph;  // tokens per frame, block size (32/64/128) and its log2,
                           // 64-wide chunks per head
  float score_scale;     // inv_sqrt_d / H_f
  double* item_stats;    // pass 1: [n_items][3] (n, mean, M2)
  const double2* job_stats;  // pass 2: mean, stddev per job
  const float2* job_thr;     // pass 2: (raw-unit threshold, raw-unit delta margin) per job
  uint32_t* counts;
  unsigned long long* job_kept;
  uint2* upairs;       // undecided pairs (job, u * nt + v): one region of ucap per CTA
  unsigned ucap;       // region capacity (pairs beyond it are decided in place)
  unsigned* ucount;    // [grid] pairs in each CTA's region
  const float* qnorm;
  const float* kmax;  // per 128-token tile: max |k'_v|
  float kappa;
  float delta_floor;
  Feat feat;  // exact re-score in place when the undecided list is full
};

// Capacity of the undecided-pair list per item (the mean at the Hunyuan
// shape is ~3.4 per item); pairs beyond it are decided in place.
#ifndef RP_SCORE_ABL
#define RP_SCORE_ABL 0
#endif
constexpr int kSlotsPerItem = 32;

// Epilogue shape: 4 * CG warps, warp w reads TMEM lanes 32 (w % 4) .. (its
// 32 rows) and column group w / 4 (128 / CG columns), so CG > 1 puts CG
// warps on each sub-partition (latency hiding) and splits the per-row work.
// Warp 4 CG issues TMA, warp 4 CG + 1 the MMAs.
template <int CG>
struct Epi {
  static constexpr int kWarps = 4 * CG;
  static constexpr int kThreads = 32 * (kWarps + 2);
  static constexpr int kNW = 4 / CG;                    // 32-column words per warp
};
constexpr int kChunkBytes = 128 * 128;

template <int NC>
struct SLayout {
  static constexpr int kTileBytes = NC * kChunkBytes;
  static constexpr int kStages = 2;
  static constexpr int kSmemData = (1 + kStages) * kTileBytes;
  static constexpr int kNumBars = 2 * kStages + 6;
  // bars | tmem slot (16 B) | 512 B (word 0: undecided-pair counter) | wcnt[2][4][128] |
  // red[2][16][3] doubles
  // (wcnt / red double-buffered by item parity: one epilogue barrier per item)
  static constexpr int kExtra = kNumBars * 8 + 16 + 128 * 4 + 2 * 4 * 128 * 4 + 2 * 16 * 3 * 8;
  static constexpr int kSmemBytes = kSmemData + kExtra + 1024;
};

template <int CG>
RP_DEV void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(32 * Epi<CG>::kWarps) : "memory"); }

struct Welford {
  double n, mean, m2;
};
RP_DEV Welford chan(Welford a, Welford b) {
  if (b.n == 0.0) return a;
  if (a.n == 0.0) return b;
  const double n = a.n + b.n;
  const double delta = b.mean - a.mean;
  Welford r;
  r.n = n;
  r.mean = a.mean + delta * (b.n / n);
  r.m2 = a.m2 + b.m2 + delta * delta * (a.n * b.n / n);
  return r;
}

// Overflowing undecided pair: decided here with the exact fp64 score.  Out
// of line so the epilogue's unrolled loops stay compact.
__device__ __noinline__ bool decide_exact(const SParams& p, int job, long long gr, long long gc) {
  return zscore(exact_score(p.feat, gr, gc), p.job_stats[job]) >= p.jobs[job].param;
}

// Work order: units (one frame pair's items of one 128-token tile row, so
// consecutive items share the Q' tile) are dealt round-robin to the CTAs.
// The host sorts the units so that neighbouring units touch few frames:
// all CTAs then work on a narrow window of Q / K frames at once and K
// tiles come from L2 instead of HBM.
struct UnitCursor {
  const int2* units;
  int n, u, it, lo, hi;
  RP_DEV explicit UnitCursor(const SParams& p)
      : units(p.units), n(p.n_units), u(static_cast<int>(blockIdx.x)), it(0), lo(0), hi(0) {
    load();
  }
  RP_DEV void load() {
    if (u < n) {
      const int2 x = units[u];
      it = x.x;
      lo = x.x;
      hi = x.y;
    }
  }
  RP_DEV bool valid() const { return u < n; }
  RP_DEV void next() {
    if (++it >= hi) {
      u += static_cast<int>(gridDim.x);
      load();
    }
  }
};

template <int NC, int MODE, int CG>
__global__ void __launch_bounds__(Epi<CG>::kThreads, 1)
    score_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                 const SParams p) {
  using L = SLayout<NC>;
  using E = Epi<CG>;
  constexpr int kTma = E::kWarps, kMma = E::kWarps + 1, NW = E::kNW;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sq = smem;
  uint8_t* sk = smem + L::kTileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kSmemData);
  uint64_t* kv_full = bars;
  uint64_t* kv_empty = bars + L::kStages;
  uint64_t* q_full = bars + 2 * L::kStages;
  uint64_t* q_empty = q_full + 1;
  uint64_t* s_full = q_full + 2;   // [2]
  uint64_t* s_empty = q_full + 4;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + L::kNumBars);
  unsigned* s_ucnt = tmem_slot + 4;  // pass 2: pairs in this CTA's undecided region
  uint32_t* wcnt_base = reinterpret_cast<uint32_t*>(tmem_slot + 4 + 128);  // [2][4][128]
  double* red_base = reinterpret_cast<double*>(wcnt_base + 2 * 4 * 128);  // [2][16][3]

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    for (int s = 0; s < L::kStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    *s_ucnt = 0;
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_empty[b], E::kWarps);
    }
    fence_barrier_init();
  }
  if (warp == kMma) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kTma) {
    {
      // ------------------------------------------------------ TMA producer
      // (whole warp in uniform control flow, one elected lane issues)
      const uint64_t pol = policy_evict_normal();
      uint32_t kv_it = 0, qcnt = 0;
      int prev_tr = -1;
      for (UnitCursor cur(p); cur.valid(); cur.next()) {
        const long long it = cur.it;
        const int item_tr = shfl0(p.items[it].tr);
        const int item_tc = shfl0(p.items[it].tc);
        if (item_tr != prev_tr) {
          mbar_wait(q_empty, (qcnt & 1) ^ 1);
          mbar_arrive_expect_tx_w(q_full, L::kTileBytes);
#pragma unroll
          for (int c = 0; c < NC; ++c)
            tma_load_3d_w(sq + c * kChunkBytes, &tq, q_full, (c % p.cph) * 64, c / p.cph,
                        item_tr * 128, pol);
          ++qcnt;
          prev_tr = item_tr;
        }
        const uint32_t st = kv_it % L::kStages;
        mbar_wait(&kv_empty[st], ((kv_it / L::kStages) & 1) ^ 1);
        mbar_arrive_expect_tx_w(&kv_full[st], L::kTileBytes);
#pragma unroll
        for (int c = 0; c < NC; ++c)
          tma_load_3d_w(sk + st * L::kTileBytes + c * kChunkBytes, &tk, &kv_full[st],
                      (c % p.cph) * 64, c / p.cph, item_tc * 128, pol);
        ++kv_it;
      }
    }
  } else if (warp == kMma) {
    {
      // ------------------------------------------------------- MMA issuer
      // (whole warp: descriptors stay in uniform registers, see common.cuh)
      const uint32_t idesc = idesc_bf16(128, 128, false, false);
      const uint32_t qa = smem_u32(sq), kb0 = smem_u32(sk);
      uint32_t kv_it = 0, qcnt = 0, n = 0;
      int prev_tr = -1;
      for (UnitCursor cur(p); cur.valid(); cur.next(), ++n) {
        const long long it = cur.it;
        const int item_tr = shfl0(p.items[it].tr);
        const int item_tc = shfl0(p.items[it].tc);
        if (item_tr != prev_tr) {
          if (prev_tr >= 0) umma_commit_w(q_empty);  // old Q' no longer read
          mbar_wait(q_full, qcnt & 1);
          ++qcnt;
          prev_tr = item_tr;
        }
        const uint32_t st = kv_it % L::kStages;
        const uint32_t buf = n & 1;
        mbar_wait(&kv_full[st], (kv_it / L::kStages) & 1);
        mbar_wait(&s_empty[buf], ((n >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t kb = kb0 + st * L::kTileBytes;
#pragma unroll
        for (int kk = 0; kk < (RP_SCORE_ABL == 2 ? 1 : NC * 4); ++kk) {  // ABL 2: one MMA
          const uint32_t off = (kk / 4) * kChunkBytes + (kk % 4) * 32;
          umma_ss_w(tmem + buf * 128, smem_desc_sw128(qa + off, 0, 1024),
                  smem_desc_sw128(kb + off, 0, 1024), idesc, kk > 0);
        }
        umma_commit_w(&kv_empty[st]);
        umma_commit_w(&s_full[buf]);
        ++kv_it;
      }
    }
  } else {
    // ----------------------------------------------------------- epilogue
    // Branch-free over the 128 columns of the thread's row: the unrolled
    // loops carry no calls or rare-path code, so the kernel stays small
    // enough for the instruction cache (an earlier version that inlined the
    // exact re-score into every unrolled column ran at IPC 0.26, stalled on
    // instruction fetch).
    const int rw = warp & 3, cg = warp >> 2;  // row group (TMEM lanes), column group
    const int r = rw * 32 + lane;             // row within the tile
    const int et = warp * 32 + lane;          // epilogue thread index
    const uint32_t trow = tmem + (static_cast<uint32_t>(rw * 32) << 16) + cg * 32 * NW;
    uint32_t n = 0;
    double u1 = 0.0, u2 = 0.0;  // pass 1: this row's sums over the current unit
    int un = 0;
    uint32_t nu = 0;  // units reduced (red[] parity)
    // Item metadata is software-pipelined: item n + 2 is loaded while item n
    // is processed, and the loads that depend on it (its frame pair, the
    // pass-2 threshold, |q'| of the row, max |k'| of the tile) one item
    // later, so no global-load latency sits on an item's critical path.
    ScoreItem itm0{}, itm1{};
    float2 thr0 = make_float2(0.f, 0.f);
    float qn0 = 0.f, km0 = 0.f;
    auto job_loads = [&](const ScoreItem& x) {
      if (MODE == 1) {
        thr0 = __ldg(p.job_thr + x.job);
        qn0 = __ldg(p.qnorm + x.tr * 128 + r);
        km0 = __ldg(p.kmax + x.tc);
      }
    };
    UnitCursor ahead(p);
    if (ahead.valid()) {
      itm0 = load_item(p.items, ahead.it);
      job_loads(itm0);
      ahead.next();
    }
    bool has1 = ahead.valid();
    if (has1) {
      itm1 = load_item(p.items, ahead.it);
      ahead.next();
    }
    for (UnitCursor cur(p); cur.valid(); cur.next(), ++n) {
      const long long it = cur.it;
      const ScoreItem item = itm0;
      const float2 thr = thr0;
      const float qk = qn0 * p.kappa * km0;
      if (has1) job_loads(itm1);
      itm0 = itm1;
      has1 = ahead.valid();
      if (has1) {
        itm1 = load_item(p.items, ahead.it);
        ahead.next();
      }
      const uint32_t buf = n & 1;
      mbar_wait(&s_full[buf], (n >> 1) & 1);
      tc_fence_after();
      uint32_t sv[NW][32];
#pragma unroll
      for (int c = 0; c < NW; ++c) tmem_ld32(trow + buf * 128 + c * 32, sv[c]);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[buf]);
#if RP_SCORE_ABL == 1  // timing ablation only: no epilogue work
      if (sv[0][0] == 0x7fffffffu && sv[NW - 1][31] == 0x7fffffffu) p.counts[0] = 1;
      continue;
#endif
      // valid columns of this row: contiguous [c_lo, c_hi] (band + frames)
      const int u = item.u0 + r;  // row within frame i
      int c_lo = 1, c_hi = 0;
      if (u >= 0 && u < p.nt) {
        c_lo = max(max(u - item.width, 0) - item.v0, 0);
        c_hi = min(min(u + item.width, p.nt - 1) - item.v0, 127);
      }
      uint32_t inm[NW];
      int cnt = 0;
#pragma unroll
      for (int w4 = 0; w4 < NW; ++w4) {
        const int wb = 32 * (cg * NW + w4);
        const int lo = max(c_lo - wb, 0), hi = min(c_hi - wb, 31);
        inm[w4] = lo > hi ? 0u : ((hi == 31 ? 0xFFFFFFFFu : ((2u << hi) - 1u)) & ~((1u << lo) - 1u));
        cnt += __popc(inm[w4]);
      }
      if (MODE == 0) {
        // per-row sum and sum of squares of the valid scores (fp32, four
        // independent chains), then (n, sum, sumsq) reduced in fp64
        float a1[4] = {0.f, 0.f, 0.f, 0.f}, a2[4] = {0.f, 0.f, 0.f, 0.f};
        // 32-column words outside the band / frame for the whole warp are
        // skipped (they would add zeros: same sums bit for bit)
#pragma unroll
        for (int w4 = 0; w4 < NW; ++w4) {
          if (!__any_sync(0xFFFFFFFFu, inm[w4] != 0u)) continue;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float x = (inm[w4] >> i) & 1u ? __uint_as_float(sv[w4][i]) * p.score_scale : 0.f;
            a1[i & 3] += x;
            a2[i & 3] = fmaf(x, x, a2[i & 3]);
          }
        }
        // the row's sums are carried in fp64 across the items of the unit
        // (one frame pair, one tile row) and reduced once per unit: the
        // unit's stats go to its first item, the others keep n = 0 (zeroed
        // before the pass), which the per-job Chan merge skips
        u1 += static_cast<double>((a1[0] + a1[1]) + (a1[2] + a1[3]));
        u2 += static_cast<double>((a2[0] + a2[1]) + (a2[2] + a2[3]));
        un += cnt;
        if (it + 1 == cur.hi) {
          const int tn = __reduce_add_sync(0xFFFFFFFFu, un);
          double t1 = u1, t2 = u2;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {  // fixed butterfly -> deterministic lane 0
            t1 += __shfl_xor_sync(0xFFFFFFFFu, t1, o);
            t2 += __shfl_xor_sync(0xFFFFFFFFu, t2, o);
          }
          double* red = red_base + (nu & 1) * 16 * 3;
          if (lane == 0) {
            red[warp * 3 + 0] = static_cast<double>(tn);
            red[warp * 3 + 1] = t1;
            red[warp * 3 + 2] = t2;
          }
          epi_bar<CG>();
          if (et == 0) {
            double N = 0.0, S1 = 0.0, S2 = 0.0;
            for (int x = 0; x < E::kWarps; ++x) {
              N += red[3 * x];
              S1 += red[3 * x + 1];
              S2 += red[3 * x + 2];
            }
            const double mean = N > 0.0 ? S1 / N : 0.0;
            const long long first = cur.lo;
            p.item_stats[3 * first + 0] = N;
            p.item_stats[3 * first + 1] = mean;
            p.item_stats[3 * first + 2] = N > 0.0 ? fmax(S2 - S1 * mean, 0.0) : 0.0;
          }
          // no trailing barrier: the next unit writes the other red buffer,
          // and this one is rewritten only after the next unit's barrier
          u1 = 0.0;
          u2 = 0.0;
          un = 0;
          ++nu;
        }
      } else {
        // Decision thresholds of this row in raw accumulator units.  The
        // fast score differs from the reference's by at most
        // kappa |q'_u| |k'_v| (fp32 accumulation) plus the mu/sigma and
        // float-rounding floor delta (1 + |z|); only |z - tau| < 1 can be
        // undecided, so in z units B = qn kmax(tile) kappa scale / sd +
        // delta (2 + |tau|).  In raw units z >= tau + B <=> raw >= base + m
        // with base = (tau sd + mu) / scale and m = qn kmax kappa + c_job
        // (job_stats_kernel); the fp32 evaluation is inflated by 2^-20
        // relative so rounding can only widen the undecided band.
        const float m = fmaf(qk, 1.f + 0x1p-20f, thr.y) + 0x1p-20f * fabsf(thr.x);
        const float hi_raw = thr.x + m;
        const float lo_raw = thr.x - m;
        uint32_t kb[NW], ub[NW];
#pragma unroll
        for (int w4 = 0; w4 < NW; ++w4) {
          uint32_t k1 = 0u, u1 = 0u;
          // words empty for the whole warp (band edge, frame boundary) skip
          // the compares
          const bool any = __any_sync(0xFFFFFFFFu, inm[w4] != 0u);
#pragma unroll
          for (int i = 0; i < 32 && any; ++i) {
            // compare + predicated OR per mask (2 instructions per bit)
            asm("{\n\t.reg .pred pk, pu;\n\t"
                "setp.ge.f32 pk, %2, %3;\n\t"
                "setp.gt.f32 pu, %2, %4;\n\t"
                "@pk or.b32 %0, %0, %5;\n\t"
                "@pu or.b32 %1, %1, %5;\n\t}"
                : "+r"(k1), "+r"(u1)
                : "f"(__uint_as_float(sv[w4][i])), "f"(hi_raw), "f"(lo_raw), "r"(1u << i));
          }
          kb[w4] = k1 & inm[w4];
          ub[w4] = u1 & inm[w4] & ~k1;
        }
        // rare path: undecided pairs are appended to one compact list for the
        // exact fp64 re-score (one atomic per warp, warp scan for the offsets)
        int mine = 0;
#pragma unroll
        for (int w4 = 0; w4 < NW; ++w4) mine += __popc(ub[w4]);
        if (__any_sync(0xFFFFFFFFu, mine != 0)) {
          int incl = mine;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += y;
          }
          unsigned base = 0;
          if (lane == 31) base = atomicAdd(s_ucnt, static_cast<unsigned>(incl));
          base = __shfl_sync(0xFFFFFFFFu, base, 31);
          if (mine) {
            unsigned at = base + static_cast<unsigned>(incl - mine);
#pragma unroll
            for (int w4 = 0; w4 < NW; ++w4) {
              uint32_t m = ub[w4];
              while (m) {
                const int i = __ffs(m) - 1;
                m &= m - 1;
                const int v = item.v0 + 32 * (cg * NW + w4) + i;
                if (at < p.ucap)
                  p.upairs[static_cast<long long>(blockIdx.x) * p.ucap + at] = make_uint2(static_cast<uint32_t>(item.job),
                                            static_cast<uint32_t>(u) * p.nt + v);
                else if (decide_exact(p, item.job, static_cast<long long>(item.tr) * 128 + r,
                                      static_cast<long long>(item.tc) * 128 +
                                          32 * (cg * NW + w4) + i))
                  kb[w4] |= 1u << i;
                ++at;
              }
            }
          }
        }
        // per-column counts within the warp: transpose each 32 x 32 bit block
        // (lane = row -> lane = column) and count
        unsigned kept_total = 0;
#pragma unroll
        for (int w4 = 0; w4 < NW; ++w4) {
          uint32_t x = kb[w4];
          kept_total += __popc(x);
#pragma unroll
          for (int j = 16; j > 0; j >>= 1) {
            const uint32_t m = j == 16 ? 0x0000FFFFu : j == 8 ? 0x00FF00FFu
                             : j == 4 ? 0x0F0F0F0Fu : j == 2 ? 0x33333333u : 0x55555555u;
            const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x, j);
            x = (lane & j) ? ((x & ~m) | ((y >> j) & m)) : ((x & m) | ((y & m) << j));
          }
          wcnt_base[(n & 1) * 512 + rw * 128 + (cg * NW + w4) * 32 + lane] = __popc(x);
        }
        epi_bar<CG>();
        // thread et < 128 owns column et: sum the row groups of each block
        // row (bs = 32 << k: 128 / bs block rows of bs / 32 row groups)
        if (et < 128) {
          const int lg = p.lg_bs;
          const int cc = item.cc0 + (et >> lg);
          if (cc >= 0 && cc < item.jtc) {
            const int wpb = p.bs >> 5;
            const int within = et & (p.bs - 1);
            for (int br = 0; br < (128 >> lg); ++br) {
              uint32_t c2 = 0;
              for (int x = 0; x < wpb; ++x) c2 += wcnt_base[(n & 1) * 512 + (br * wpb + x) * 128 + et];
              const int rr = item.rr0 + br;
              if (rr >= 0 && rr < item.jtr && c2)
                p.counts[item.cnt_off + (static_cast<long long>(rr * item.jtc + cc) << lg) + within] = c2;
            }
          }
        }
        kept_total = __reduce_add_sync(0xFFFFFFFFu, kept_total);
        if (lane == 0 && kept_total) atomicAdd(&p.job_kept[item.job], static_cast<unsigned long long>(kept_total));
        // no trailing barrier (wcnt is double-buffered, see red above)
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (MODE == 1 && threadIdx.x == 0) p.ucount[blockIdx.x] = *s_ucnt;
  if (warp == kMma) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

// Per-token L2 norm of the concatenated scoring features (H_f heads x d).
__global__ void norm_kernel(const __nv_bfloat16* __restrict__ x, long long tokens,
                            long long ts, long long hs, int heads, int d,
                            float* __restrict__ out) {
  const long long t = static_cast<long long>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (t >= tokens) return;
  float acc = 0.f;
  for (int h = 0; h < heads; ++h)
    for (int e = lane; e < d; e += 32) {
      const float v = __bfloat162float(x[t * ts + h * hs + e]);
      acc = fmaf(v, v, acc);
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
  if (lane == 0) out[t] = sqrtf(acc);
}

// Deterministic per-frame-pair merge of item statistics: one warp per job,
// lane l Chan-merges items l, l + 32, ... (only each unit's first item
// carries stats), then a fixed butterfly.
__global__ void job_stats_kernel(const double* __restrict__ item_stats,
                                 const long long* __restrict__ job_item_off, int n_jobs,
                                 const DJob* __restrict__ jobs, double score_scale,
                                 double delta_floor, double2* __restrict__ job_stats,
                                 float2* __restrict__ job_thr) {
  const int j = static_cast<int>((blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= n_jobs) return;
  Welford a{0.0, 0.0, 0.0};
  for (long long it = job_item_off[j] + lane; it < job_item_off[j + 1]; it += 32)
    a = chan(a, Welford{item_stats[3 * it], item_stats[3 * it + 1], item_stats[3 * it + 2]});
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Welford b;
    b.n = __shfl_xor_sync(0xFFFFFFFFu, a.n, o);
    b.mean = __shfl_xor_sync(0xFFFFFFFFu, a.mean, o);
    b.m2 = __shfl_xor_sync(0xFFFFFFFFu, a.m2, o);
    a = (lane & o) ? chan(b, a) : chan(a, b);  // lower lanes' items first on both sides
  }
  if (lane != 0) return;
  const double sd = a.n > 0 ? sqrt(a.m2 / a.n) : 0.0;
  job_stats[j] = make_double2(a.mean, sd);
  // pass-2 thresholds in raw accumulator units (see score_kernel)
  const double tau = jobs[j].param, sde = sd + 1e-8;
  job_thr[j] = make_float2(__double2float_rn((tau * sde + a.mean) / score_scale),
                           __double2float_ru(delta_floor * (2.0 + fabs(tau)) * sde / score_scale));
}

// theta_c / theta_m per block tile from the count buffer (mask.cpp:87-125,
// as apply_kernel mode 1): one warp per tile, bs / 32 columns per lane.
__global__ void apply_tiles_kernel(const DJob* __restrict__ jobs, const Item* __restrict__ tiles,
                                   long long n_tiles, const uint32_t* __restrict__ counts,
                                   uint32_t* words, int bs, int64_t row_bytes, uint32_t cmin,
                                   int amin) {
  const long long t = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= n_tiles) return;
  const Item it = tiles[t];
  const DJob& jb = jobs[it.job];
  const uint32_t* c = counts + jb.cnt_off + (static_cast<int64_t>(it.tr) * jb.tc + it.tc) * bs;
  int mine;
  if (bs == 128) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(c) + lane);
    mine = (v.x >= cmin) + (v.y >= cmin) + (v.z >= cmin) + (v.w >= cmin);
  } else if (bs == 64) {
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(c) + lane);
    mine = (v.x >= cmin) + (v.y >= cmin);
  } else {
    mine = __ldg(c + lane) >= cmin;
  }
  const int active = __reduce_add_sync(0xFFFFFFFFu, mine);
  if (lane == 0 && active >= amin) set_block(words, row_bytes, jb.r0 + it.tr, jb.c0 + it.tc);
}

// Max of the per-token norms over each 128-token tile (one warp per tile).
__global__ void tile_max_kernel(const float* __restrict__ norms, long long tokens,
                                long long tiles, float* __restrict__ out) {
  const long long t = static_cast<long long>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (t >= tiles) return;
  float m = 0.f;
  for (int x = lane; x < 128; x += 32) {
    const long long i = t * 128 + x;
    if (i < tokens) m = fmaxf(m, norms[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
  if (lane == 0) out[t] = m;
}

// Exact re-score of every undecided pair (reference operation order): one
// thread per pair; blockIdx.y = the scoring CTA whose undecided region this
// block walks.
__global__ void recheck_kernel(const DJob* __restrict__ jobs, const uint2* __restrict__ upairs,
                               const unsigned* __restrict__ ucount, unsigned ucap, Feat f,
                               const double2* __restrict__ job_stats, uint32_t* counts,
                               unsigned long long* job_kept, unsigned long long* rechecked,
                               int nt, int bs) {
  const unsigned n = min(ucount[blockIdx.y], ucap);
  upairs += static_cast<long long>(blockIdx.y) * ucap;
  unsigned done = 0;
  for (unsigned x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
    const uint2 sl = upairs[x];
    const DJob& jb = jobs[sl.x];
    const int64_t u = sl.y / nt, v = sl.y % nt;
    const float sc = exact_score(f, static_cast<int64_t>(jb.i) * nt + u,
                                 static_cast<int64_t>(jb.j) * nt + v);
    if (zscore(sc, job_stats[sl.x]) >= jb.param) {
      add_count(jb, counts, nt, bs, u, v);
      atomicAdd(&job_kept[sl.x], 1ull);
    }
    ++done;
  }
  done = __reduce_add_sync(0xFFFFFFFFu, done);
  if ((threadIdx.x & 31) == 0 && done) atomicAdd(rechecked, static_cast<unsigned long long>(done));
}

// Exact fallback for frame pairs that kept nothing: exact scores of the
// whole band, then the fallback_k best z (ties to the lowest flat index).
__global__ void fb_scores_kernel(const DJob* __restrict__ jobs, int job, Feat f, int nt,
                                 float* __restrict__ scores) {
  const DJob& jb = jobs[job];
  for (long long x = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; x < jb.n;
       x += static_cast<long long>(gridDim.x) * blockDim.x) {
    int64_t u, v;
    band_uv(x, nt, jb.width, &u, &v);
    scores[x] = exact_score(f, static_cast<int64_t>(jb.i) * nt + u,
                            static_cast<int64_t>(jb.j) * nt + v);
  }
}

__global__ void fb_select_kernel(const DJob* __restrict__ jobs, int job,
                                 const float* __restrict__ scores,
                                 const double2* __restrict__ job_stats, uint32_t* counts, int nt,
                                 int bs, int fallback_k) {
  const DJob& jb = jobs[job];
  const int64_t n = jb.n;
  const double2 st = job_stats[job];
  __shared__ double bz[32];
  __shared__ int64_t bi[32];
  __shared__ int64_t last_pick;
  __shared__ double last_z;
  const int k = static_cast<int>(fallback_k < n ? fallback_k : n);
  if (threadIdx.x == 0) {
    last_pick = -1;
    last_z = INFINITY;
  }
  __syncthreads();
  for (int round = 0; round < k; ++round) {
    double best = -INFINITY;
    int64_t besti = -1;
    for (int64_t x = threadIdx.x; x < n; x += blockDim.x) {
      const double z = zscore(scores[x], st);
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

// ------------------------------------------------------------ host side ---
class FastEngine {
 public:
  rp_grid g{};
  int cmin = 0, amin = 0, heads = 0, dim = 0, nc = 0;
  std::vector<DJob> jobs;        // score jobs only (cnt_off set)
  std::vector<ScoreItem> items;
  std::vector<int2> units;       // item ranges of one (job, tile row), locality order
  std::vector<long long> job_item_off;
  std::vector<Item> tiles;       // block tiles of every score job (apply)
  int64_t ncounts = 0;
  DJob* d_jobs = nullptr;
  ScoreItem* d_items = nullptr;
  int2* d_units = nullptr;
  long long* d_job_item_off = nullptr;
  Item* d_tiles = nullptr;
  uint32_t* d_counts = nullptr;
  double* d_item_stats = nullptr;
  double2* d_job_stats = nullptr;
  float2* d_job_thr = nullptr;
  unsigned long long* d_kept = nullptr;  // [jobs + 1]: per job, then rechecked pairs
  uint2* d_upairs = nullptr;
  unsigned* d_ucount = nullptr;
  float* d_qn = nullptr;
  float* d_kn = nullptr;
  float* d_kmax = nullptr;

  ~FastEngine() {
    for (void* p : {static_cast<void*>(d_jobs), static_cast<void*>(d_items),
                    static_cast<void*>(d_job_item_off), static_cast<void*>(d_tiles),
                    static_cast<void*>(d_units),
                    static_cast<void*>(d_counts), static_cast<void*>(d_item_stats),
                    static_cast<void*>(d_job_stats), static_cast<void*>(d_kept),
                    static_cast<void*>(d_job_thr),
                    static_cast<void*>(d_upairs), static_cast<void*>(d_ucount),
                    static_cast<void*>(d_qn),
                    static_cast<void*>(d_kn), static_cast<void*>(d_kmax)})
      if (p) cudaFree(p);
  }
};

bool fast_engine_supported(const rp_grid& g, int head_dim, int heads) {
  const int bs = g.block_size;
  if (bs != 32 && bs != 64 && bs != 128) return false;
  if (static_cast<int64_t>(g.tokens_per_frame) * g.tokens_per_frame >= (int64_t{1} << 32))
    return false;  // recheck slots pack u * N_t + v into 32 bits
  if (head_dim % 64 != 0 || heads < 1) return false;
  const int nc = heads * head_dim / 64;
  return nc >= 1 && nc <= 4;
}

template <class T>
static void dalloc(T** p, size_t n) {
  RP_CUDA(cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * std::max<size_t>(n, 1)));
}

FastEngine* fast_engine_create(const rp_grid& g, const std::vector<DJob>& all, int cmin,
                               int amin, int heads, int head_dim, cudaStream_t s) {
  (void)s;
  std::unique_ptr<FastEngine> e(new FastEngine);
  e->g = g;
  e->cmin = cmin;
  e->amin = amin;
  e->heads = heads;
  e->dim = head_dim;
  e->nc = heads * head_dim / 64;
  const int64_t nt = g.tokens_per_frame;
  const int bs = g.block_size;
  int64_t off = 0;
  for (const DJob& d0 : all) {
    if (d0.kind != plan::kScore) continue;
    DJob d = d0;
    d.cnt_off = off;
    off += static_cast<int64_t>(d.tr) * d.tc * bs;
    const int job = static_cast<int>(e->jobs.size());
    e->jobs.push_back(d);
    e->job_item_off.push_back(static_cast<long long>(e->items.size()));
    // 128-token tiles intersecting the band of frames (i, j)
    const int64_t qi = d.i * nt, kj = d.j * nt;
    const int64_t tr0 = qi / 128, tr1 = (qi + nt - 1) / 128;
    const int64_t tc0 = kj / 128, tc1 = (kj + nt - 1) / 128;
    for (int64_t tr = tr0; tr <= tr1; ++tr) {
      const int64_t ua = std::max<int64_t>(tr * 128, qi) - qi;
      const int64_t ub = std::min<int64_t>(tr * 128 + 127, qi + nt - 1) - qi;
      for (int64_t tc = tc0; tc <= tc1; ++tc) {
        const int64_t va = std::max<int64_t>(tc * 128, kj) - kj;
        const int64_t vb = std::min<int64_t>(tc * 128 + 127, kj + nt - 1) - kj;
        if (va - ub > d.width || ua - vb > d.width) continue;  // no |u - v| <= w
        ScoreItem x{};
        x.job = job;
        x.tr = static_cast<int32_t>(tr);
        x.tc = static_cast<int32_t>(tc);
        x.width = static_cast<int32_t>(std::min<int64_t>(d.width, nt));
        x.u0 = static_cast<int32_t>(tr * 128 - qi);
        x.v0 = static_cast<int32_t>(tc * 128 - kj);
        x.rr0 = static_cast<int32_t>(tr * 128 / bs - d.r0);
        x.cc0 = static_cast<int32_t>(tc * 128 / bs - d.c0);
        x.jtr = d.tr;
        x.jtc = d.tc;
        x.cnt_off = d.cnt_off;
        e->items.push_back(x);
      }
    }
    for (int32_t r = 0; r < d.tr; ++r)
      for (int32_t c = 0; c < d.tc; ++c) e->tiles.push_back(Item{job, r, c});
  }
  e->job_item_off.push_back(static_cast<long long>(e->items.size()));
  e->ncounts = off;
  // units: runs of items with the same (job, tile row)
  for (size_t a = 0; a < e->items.size();) {
    size_t b = a + 1;
    while (b < e->items.size() && e->items[b].job == e->items[a].job &&
           e->items[b].tr == e->items[a].tr)
      ++b;
    e->units.push_back(make_int2(static_cast<int>(a), static_cast<int>(b)));
    a = b;
  }
  // Locality order: frame pairs in F x F blocks of (key frame, query frame),
  // F chosen so the block's Q' and K' frames (2 F frames of heads * d bf16
  // per token) stay well inside L2; concurrent CTAs then share K tiles.
  {
    const double frame_bytes = static_cast<double>(nt) * heads * head_dim * 2.0;
    const int F = std::max(1, static_cast<int>((32.0 * (1 << 20)) / (2.0 * frame_bytes)));
    auto key = [&](const int2& u) {
      const ScoreItem& it = e->items[u.x];
      const DJob& d = e->jobs[it.job];
      return std::make_tuple(d.j / F, d.i / F, d.j, d.i, it.tr);
    };
    const char* order = std::getenv("DYNRAD_SCORE_ORDER");  // "plain": item order (A/B)
    if (!(order && std::strcmp(order, "plain") == 0))
      std::stable_sort(e->units.begin(), e->units.end(),
                       [&](const int2& a, const int2& b) { return key(a) < key(b); });
  }
  const size_t nj = e->jobs.size();
  dalloc(&e->d_jobs, nj);
  dalloc(&e->d_items, e->items.size());
  dalloc(&e->d_units, e->units.size());
  dalloc(&e->d_job_item_off, nj + 1);
  dalloc(&e->d_tiles, e->tiles.size());
  dalloc(&e->d_counts, static_cast<size_t>(off));
  dalloc(&e->d_item_stats, 3 * e->items.size());
  dalloc(&e->d_job_stats, nj);
  dalloc(&e->d_job_thr, nj);
  dalloc(&e->d_kept, nj + 1);
  dalloc(&e->d_upairs, e->items.size() * kSlotsPerItem);
  dalloc(&e->d_ucount, 1024);  // one per scoring CTA (grid <= SM count)
  dalloc(&e->d_qn, static_cast<size_t>(g.padded_tokens));
  dalloc(&e->d_kn, static_cast<size_t>(g.padded_tokens));
  dalloc(&e->d_kmax, static_cast<size_t>((g.padded_tokens + 127) / 128));
  RP_CUDA(cudaMemcpy(e->d_jobs, e->jobs.data(), sizeof(DJob) * nj, cudaMemcpyHostToDevice));
  RP_CUDA(cudaMemcpy(e->d_items, e->items.data(), sizeof(ScoreItem) * e->items.size(),
                     cudaMemcpyHostToDevice));
  RP_CUDA(cudaMemcpy(e->d_units, e->units.data(), sizeof(int2) * e->units.size(),
                     cudaMemcpyHostToDevice));
  RP_CUDA(cudaMemcpy(e->d_job_item_off, e->job_item_off.data(), sizeof(long long) * (nj + 1),
                     cudaMemcpyHostToDevice));
  RP_CUDA(cudaMemcpy(e->d_tiles, e->tiles.data(), sizeof(Item) * e->tiles.size(),
                     cudaMemcpyHostToDevice));
  return e.release();
}

void fast_engine_destroy(FastEngine* e) { delete e; }

template <int NC, int CG>
static void launch_pass_cg(const CUtensorMap& mq, const CUtensorMap& mk, const SParams& p,
                           int mode, int grid, cudaStream_t s) {
  const int smem = SLayout<NC>::kSmemBytes;
  const int threads = Epi<CG>::kThreads;
  if (mode == 0) {
    prepare_kernel(reinterpret_cast<const void*>(score_kernel<NC, 0, CG>), smem);
    score_kernel<NC, 0, CG><<<grid, threads, smem, s>>>(mq, mk, p);
  } else {
    prepare_kernel(reinterpret_cast<const void*>(score_kernel<NC, 1, CG>), smem);
    score_kernel<NC, 1, CG><<<grid, threads, smem, s>>>(mq, mk, p);
  }
  RP_LAUNCHED();
}

// Epilogue column groups (warps per sub-partition, see Epi) per pass.
// Measured at the Hunyuan shape (ncu, profiles/r2_score_notes.md): two warps
// per sub-partition for both passes (stats 5.38 -> 4.99 ms once its
// reduction moved to one per unit; select 8.26 ms at CG = 1, 6.82 at 2,
// 7.61 at 4).  DYNRAD_SCORE_CG in {1, 2, 4} forces both.
static int score_cg(int mode) {
  static const int forced = [] {
    const char* e = std::getenv("DYNRAD_SCORE_CG");
    const int v = e ? std::atoi(e) : 0;
    return (v == 1 || v == 2 || v == 4) ? v : 0;
  }();
  (void)mode;
  return forced ? forced : 2;
}

template <int NC>
static void launch_pass(const CUtensorMap& mq, const CUtensorMap& mk, const SParams& p, int mode,
                        int grid, cudaStream_t s) {
  switch (score_cg(mode)) {
    case 1: launch_pass_cg<NC, 1>(mq, mk, p, mode, grid, s); break;
    case 4: launch_pass_cg<NC, 4>(mq, mk, p, mode, grid, s); break;
    default: launch_pass_cg<NC, 2>(mq, mk, p, mode, grid, s); break;
  }
}

void fast_engine_run(FastEngine* e, const rp_tensor* q, const rp_tensor* k, const Feat& f,
                     uint32_t* words, cudaStream_t s, double delta_floor, int fallback_k,
                     bool want_stats, FastResult* res) {
  const rp_grid& g = e->g;
  const int nj = static_cast<int>(e->jobs.size());
  if (nj == 0 || e->items.empty()) return;
  // views restricted to the scoring heads
  rp_tensor qv = *q, kv = *k;
  qv.heads = e->heads;
  kv.heads = e->heads;
  const CUtensorMap mq = make_map_bf16(qv), mk = make_map_bf16(kv);
  stage_begin(kStageMaskPrep, s);
  RP_CUDA(cudaMemsetAsync(e->d_counts, 0, sizeof(uint32_t) * std::max<int64_t>(e->ncounts, 1), s));
  RP_CUDA(cudaMemsetAsync(e->d_kept, 0, sizeof(unsigned long long) * (nj + 1), s));
  RP_CUDA(cudaMemsetAsync(e->d_qn, 0, sizeof(float) * g.padded_tokens, s));
  RP_CUDA(cudaMemsetAsync(e->d_kn, 0, sizeof(float) * g.padded_tokens, s));
  const unsigned ngrid = static_cast<unsigned>((g.total_tokens + 7) / 8);
  norm_kernel<<<ngrid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(q->data), g.total_tokens,
                                    q->token_stride, q->head_stride, e->heads, e->dim, e->d_qn);
  RP_LAUNCHED();
  norm_kernel<<<ngrid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(k->data), g.total_tokens,
                                    k->token_stride, k->head_stride, e->heads, e->dim, e->d_kn);
  RP_LAUNCHED();
  const long long ktiles = (g.padded_tokens + 127) / 128;
  tile_max_kernel<<<static_cast<unsigned>((ktiles + 7) / 8), 256, 0, s>>>(e->d_kn, g.total_tokens,
                                                                         ktiles, e->d_kmax);
  RP_LAUNCHED();
  stage_end(kStageMaskPrep, s);

  SParams p{};
  p.jobs = e->d_jobs;
  p.items = e->d_items;
  p.n_items = static_cast<long long>(e->items.size());
  p.units = e->d_units;
  p.n_units = static_cast<int>(e->units.size());
  p.nt = g.tokens_per_frame;
  p.bs = g.block_size;
  p.lg_bs = g.block_size == 32 ? 5 : g.block_size == 64 ? 6 : 7;
  p.cph = e->dim / 64;
  p.score_scale = static_cast<float>((1.0 / std::sqrt(static_cast<double>(e->dim))) / e->heads);
  p.item_stats = e->d_item_stats;
  p.job_stats = e->d_job_stats;
  p.job_thr = e->d_job_thr;
  p.counts = e->d_counts;
  p.job_kept = e->d_kept;
  p.upairs = e->d_upairs;
  p.ucount = e->d_ucount;
  p.qnorm = e->d_qn;
  p.kmax = e->d_kmax;
  // fp32 accumulation of K = H_f * d exact bf16 products, each rounding
  // (or truncating) step off by <= 2^-23 relative: |err| <= 2 K 2^-23
  // sum|q k| <= 2 K 2^-23 |q| |k|.
  p.kappa = static_cast<float>(2.0 * e->heads * e->dim * std::ldexp(1.0, -23));
  p.delta_floor = static_cast<float>(delta_floor);
  p.feat = f;
  int dev = 0, sms = 0;
  RP_CUDA(cudaGetDevice(&dev));
  RP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int grid = std::min(p.n_units, std::min(sms, 1024));
  p.ucap = static_cast<unsigned>(
      std::min<long long>(static_cast<long long>(e->items.size()) * kSlotsPerItem / grid,
                          0x7fffffffLL));
  // DYNRAD_SCORE_UCAP: smaller per-CTA capacity (tests drive the in-place
  // exact decision of pairs that overflow the list)
  if (const char* cap = std::getenv("DYNRAD_SCORE_UCAP"))
    p.ucap = std::min<unsigned>(p.ucap, static_cast<unsigned>(std::max(0, std::atoi(cap))));
  for (int mode = 0; mode < 2; ++mode) {
    const int st = mode == 0 ? kStageScoreStats : kStageScoreSelect;
    stage_begin(st, s);
    if (mode == 0)  // per-unit stats land on each unit's first item
      RP_CUDA(cudaMemsetAsync(e->d_item_stats, 0, sizeof(double) * 3 * e->items.size(), s));
    switch (e->nc) {
      case 1: launch_pass<1>(mq, mk, p, mode, grid, s); break;
      case 2: launch_pass<2>(mq, mk, p, mode, grid, s); break;
      case 3: launch_pass<3>(mq, mk, p, mode, grid, s); break;
      default: launch_pass<4>(mq, mk, p, mode, grid, s); break;
    }
    stage_end(st, s);
    if (mode == 0) {
      stage_begin(kStageJobStats, s);
      job_stats_kernel<<<(nj + 7) / 8, 256, 0, s>>>(e->d_item_stats, e->d_job_item_off, nj,
                                                       e->d_jobs, p.score_scale, delta_floor,
                                                       e->d_job_stats, e->d_job_thr);
      RP_LAUNCHED();
      stage_end(kStageJobStats, s);
    }
  }
  // exact re-score of the pairs within their error bound of tau
  stage_begin(kStageRecheck, s);
  {
    recheck_kernel<<<dim3(8, static_cast<unsigned>(grid)), 256, 0, s>>>(
        e->d_jobs, e->d_upairs, e->d_ucount, p.ucap, f, e->d_job_stats, e->d_counts, e->d_kept,
        e->d_kept + nj, g.tokens_per_frame, g.block_size);
    RP_LAUNCHED();
  }
  // fallback_k: only when it can activate a column (fallback_k >= cmin)
  const bool fb_matters = fallback_k >= e->cmin;
  std::vector<unsigned long long> kept;
  if (fb_matters || want_stats) {
    kept.resize(nj + 1);
    RP_CUDA(cudaMemcpyAsync(kept.data(), e->d_kept, sizeof(unsigned long long) * (nj + 1),
                            cudaMemcpyDeviceToHost, s));
    RP_CUDA(cudaStreamSynchronize(s));
    if (res) res->rechecked = static_cast<int64_t>(kept[nj]);
    for (int j = 0; j < nj; ++j) {
      if (kept[j] != 0) continue;
      if (res) ++res->fallbacks;
      if (!fb_matters) continue;
      float* sc = nullptr;
      RP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&sc), sizeof(float) * e->jobs[j].n, s));
      fb_scores_kernel<<<std::min<int64_t>((e->jobs[j].n + 255) / 256, 4096), 256, 0, s>>>(
          e->d_jobs, j, f, g.tokens_per_frame, sc);
      RP_LAUNCHED();
      fb_select_kernel<<<1, 256, 0, s>>>(e->d_jobs, j, sc, e->d_job_stats, e->d_counts,
                                         g.tokens_per_frame, g.block_size, fallback_k);
      RP_LAUNCHED();
      RP_CUDA(cudaFreeAsync(sc, s));
    }
  }
  stage_end(kStageRecheck, s);
  // theta_c / theta_m per block tile of every scored frame pair
  stage_begin(kStageApply, s);
  {
    const long long nt_ = static_cast<long long>(e->tiles.size());
    apply_tiles_kernel<<<static_cast<unsigned>((nt_ + 7) / 8), 256, 0, s>>>(
        e->d_jobs, e->d_tiles, nt_, e->d_counts, words, g.block_size, g.row_bytes,
        static_cast<uint32_t>(e->cmin), e->amin);
    RP_LAUNCHED();
  }
  stage_end(kStageApply, s);
}

}  // namespace mask
}  // namespace rp
