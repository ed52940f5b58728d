// K6: block-sparse flash-attention forward, bf16 in / fp32 softmax, sm_100a.
//
// Replaces radialplan::masked_attention_exact (attention.cpp:50-121) on the
// tensor cores.  Semantics kept from the reference:
//   * only blocks listed in the row's CSR list are attended (exact mask,
//     -inf elsewhere; the mask is constant within a B x B block so no
//     element masking is needed);
//   * query/key/value rows >= S (the padding of the last block) are zeros:
//     TMA's out-of-bounds fill produces them, and padded keys take part with
//     logit 0 whenever their block is active (attention.cpp:43-48, 66-68).
//
// Design (one persistent CTA per SM, 384 threads, FA4-style warp roles):
//   warps 0-3  softmax for tile A  (thread t owns query row t = TMEM lane t)
//   warps 4-7  softmax for tile B
//   warp  8    TMA producer (Q tiles, K/V ring of kStages 128-row tiles)
//   warp  9    TMEM allocator + tcgen05.mma issuer (one thread)
//   warps 10-11 idle (complete the producer warpgroup for setmaxnreg)
// A work unit is (row block r, head pair {2p, 2p+1}): tiles A and B share
// the same KV block list and ping-pong on the tensor core.  TMEM (512 cols):
// S_A 0-127, S_B 128-255, O_A 256-(256+D), O_B 384-(384+D).  P (bf16)
// overwrites the first 64 columns of its S tile and feeds O += P V straight
// from TMEM (A operand in TMEM), so shared memory only serves Q, K and V
// (the tensor core's shared-memory read bandwidth is the scarce resource for
// 1-SM 128x128 MMAs; a P operand in shared memory measured ~8% slower).
// MMA issue order per step j: O_A += P_A(j) V(j), S_A(j+1), O_B += P_B(j)
// V(j), S_B(j+1) (S_x(j+1) overwrites P_x(j), so it follows the P.V that
// reads it; tcgen05 MMAs of one CTA execute in issue order).
// Online softmax with lazy rescaling: O and l are rescaled only when the row
// max grows by more than 2^8 (exact: numerator and denominator share the
// stale max).
#include "common.cuh"

namespace rp {
namespace attn {

constexpr int kThreads = 384;  // 3 warpgroups: softmax A, softmax B, producer/MMA
constexpr int kBM = 128;  // query rows per tile (= block size B)
constexpr int kBN = 128;  // keys per KV tile (= block size B)
// Which of every 8 consecutive element pairs take the polynomial exp2 on the
// FMA pipe instead of MUFU.EX2 (bit i set -> pair i mod 8 uses the
// polynomial): balances the two pipes, FA4-style.
#ifndef RP_POLY_MASK
#define RP_POLY_MASK 0x00u
#endif
constexpr uint32_t kPolyMask = RP_POLY_MASK;
// Keys of P after which the softmax signals the MMA warp (p_split) so that
// P.V on them overlaps the last chunk's exponentials (multiple of 32, < 128).
#ifndef RP_SPLIT_KEYS
#define RP_SPLIT_KEYS 128
#endif
constexpr int kSplitKeys = RP_SPLIT_KEYS;

template <int D>
struct Layout {
  static constexpr int kChunks = D / 64;           // 128-byte K chunks
  static constexpr int kTileBytes = 128 * D * 2;   // one 128-row bf16 tile
  static constexpr int kChunkBytes = 128 * 128;    // 128 rows x 128 B
  static constexpr int kStages = D == 128 ? 5 : 10;
  static constexpr int kSmemData = 2 * kTileBytes + kStages * kTileBytes;
  static constexpr int kNumBars = 2 * kStages + 14;
  static constexpr int kSmemBytes = kSmemData + kNumBars * 8 + 16 + 1024;
  RP_HD static uint32_t s_col(int x) { return x ? 128u : 0u; }
  RP_HD static uint32_t o_col(int x) { return x ? 384u : 256u; }
};

#ifdef RP_TRACE
// Debug-only event trace (tools/trace_k6.py): clock64 stamps of the softmax
// and MMA roles of the first kTraceCtas CTAs.
constexpr int kTraceCtas = 4, kTraceEv = 12, kTraceSteps = 512;
__device__ unsigned long long g_trace[kTraceCtas][kTraceEv][kTraceSteps];
#define RP_TR(ev, idx)                                                        \
  do {                                                                        \
    if (blockIdx.x < kTraceCtas && (idx) < kTraceSteps)                       \
      g_trace[blockIdx.x][ev][idx] = clock64();                               \
  } while (0)
#else
#define RP_TR(ev, idx) \
  do {                 \
  } while (0)
#endif

struct Params {
  const int32_t* row_ptr;
  const int32_t* col_idx;
  const int32_t* row_order;  // may be null
  int n_rows;                // S_b
  int heads;
  int n_pairs;               // ceil(heads / 2)
  long long n_units;         // n_pairs * n_rows
  __nv_bfloat16* out;
  long long out_tok_stride;  // elements
  long long out_head_stride;
  float scale_log2;          // softmax_scale * log2(e)
};

struct Unit {
  int row, h0, h1, beg, n;
  bool has_b;
};

RP_DEV Unit decode(const Params& p, long long u) {
  Unit w;
  const int pair = static_cast<int>(u / p.n_rows);
  const int ri = static_cast<int>(u % p.n_rows);
  w.row = p.row_order ? __ldg(p.row_order + ri) : ri;
  w.h0 = 2 * pair;
  w.h1 = 2 * pair + 1;
  w.has_b = w.h1 < p.heads;
  w.beg = __ldg(p.row_ptr + w.row);
  w.n = __ldg(p.row_ptr + w.row + 1) - w.beg;
  return w;
}

// decode() for a whole role warp: the row-list lookups are broadcast from
// lane 0 so every derived value is provably warp-uniform.
RP_DEV Unit decode_warp(const Params& p, long long u) {
  Unit w = decode(p, u);
  w.row = shfl0(w.row);
  w.beg = shfl0(w.beg);
  w.n = shfl0(w.n);
  return w;
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    bsfa_fwd_kernel(const __grid_constant__ CUtensorMap tq,
                    const __grid_constant__ CUtensorMap tk,
                    const __grid_constant__ CUtensorMap tv, const Params p) {
  using L = Layout<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sq = smem;                                  // [2][tile]
  uint8_t* skv = smem + 2 * L::kTileBytes;             // [kStages][tile]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kSmemData);
  uint64_t* kv_full = bars;
  uint64_t* kv_empty = bars + L::kStages;
  uint64_t* q_full = bars + 2 * L::kStages;  // [2] each below
  uint64_t* q_empty = q_full + 2;
  uint64_t* s_full = q_full + 4;    // MMA -> softmax: S_x ready in TMEM
  uint64_t* p_full = q_full + 6;    // softmax -> MMA: P_x written to TMEM
  uint64_t* o_done = q_full + 8;    // MMA -> softmax: unit's last P.V done
  uint64_t* o_free = q_full + 10;   // softmax -> MMA: epilogue read O_x
  uint64_t* p_split = q_full + 12;  // softmax -> MMA: P_x keys [0, kSplitKeys) written
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + L::kNumBars);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    for (int s = 0; s < L::kStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(&q_full[x], 1);
      mbar_init(&q_empty[x], 1);
      mbar_init(&s_full[x], 1);
      mbar_init(&p_full[x], 4);
      mbar_init(&o_done[x], 1);
      mbar_init(&o_free[x], 4);
      mbar_init(&p_split[x], 4);
    }
    fence_barrier_init();
  }
  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&tq);
    tma_prefetch_desc(&tk);
    tma_prefetch_desc(&tv);
  }
  if (warp == 9) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // Register budget per role: the launch allocates 168 regs x 384 threads;
  // the producer warpgroup gives back to 88 so the two softmax warpgroups
  // (128-wide score row + packed P) can grow to 208:
  // 2 * 128 * 208 + 128 * 88 == 384 * 168 (an over-ask would block forever).
  if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;" ::: "memory");
    if (warp == 8) {
      // ---------------------------------------------------- TMA producer --
      // (whole warp, uniform control flow; one elected lane issues)
      const uint64_t pol_q = policy_evict_first();
#ifdef RP_KV_EVICT_NORMAL
      const uint64_t pol_kv = policy_evict_normal();
#else
      const uint64_t pol_kv = policy_evict_last();
#endif
      uint32_t kv_it = 0;
      uint32_t ucnt[2] = {0, 0};
      auto load_kv = [&](const CUtensorMap* m, int h, int blk) {
        const uint32_t st = kv_it % L::kStages;
        const uint32_t ph = (kv_it / L::kStages) & 1;
        mbar_wait(&kv_empty[st], ph ^ 1);
#ifdef RP_ABL_NOLOAD
        // ablation: after the ring's first fill, reuse stale tiles (timing only)
        if (kv_it >= L::kStages) {
          if (lane == 0) mbar_arrive(&kv_full[st]);
          ++kv_it;
          return;
        }
#endif
        mbar_arrive_expect_tx_w(&kv_full[st], L::kTileBytes);
        uint8_t* dst = skv + st * L::kTileBytes;
#pragma unroll
        for (int c = 0; c < L::kChunks; ++c)
          tma_load_3d_w(dst + c * L::kChunkBytes, m, &kv_full[st], c * 64, h, blk * kBN, pol_kv);
        ++kv_it;
      };
      for (long long u = blockIdx.x; u < p.n_units; u += gridDim.x) {
        const Unit w = decode_warp(p, u);
        for (int x = 0; x < 2; ++x) {
          if (x == 1 && !w.has_b) continue;
          mbar_wait(&q_empty[x], (ucnt[x] & 1) ^ 1);
          mbar_arrive_expect_tx_w(&q_full[x], L::kTileBytes);
#pragma unroll
          for (int c = 0; c < L::kChunks; ++c)
            tma_load_3d_w(sq + x * L::kTileBytes + c * L::kChunkBytes, &tq, &q_full[x], c * 64,
                        x ? w.h1 : w.h0, w.row * kBM, pol_q);
          ++ucnt[x];
        }
        // order must match the MMA issue order below
        const int32_t* cols = p.col_idx + w.beg;
        int cj = shfl0(__ldg(cols));
        load_kv(&tk, w.h0, cj);
        if (w.has_b) load_kv(&tk, w.h1, cj);
        for (int j = 0; j < w.n; ++j) {
          const int cn = j + 1 < w.n ? shfl0(__ldg(cols + j + 1)) : 0;
          load_kv(&tv, w.h0, cj);
          if (j + 1 < w.n) load_kv(&tk, w.h0, cn);
          if (w.has_b) {
            load_kv(&tv, w.h1, cj);
            if (j + 1 < w.n) load_kv(&tk, w.h1, cn);
          }
          cj = cn;
        }
      }
    } else if (warp == 9) {
      // ----------------------------------------------------- MMA issuer ---
      // (whole warp, uniform control flow; one elected lane issues)
      const uint32_t idesc_qk = idesc_bf16(128, 128, false, false);
      const uint32_t idesc_pv = idesc_bf16(128, D, false, true);
      const uint32_t sq_addr = smem_u32(sq);
      const uint32_t skv_addr = smem_u32(skv);
      uint32_t kv_it = 0;
      uint32_t ucnt[2] = {0, 0};
      uint32_t pcnt[2] = {0, 0};
      // S_x = Q_x . K^T : 128 x 128, K = D in steps of 16.
      auto issue_s = [&](int x, bool last_s) {
        const uint32_t st = kv_it % L::kStages;
        mbar_wait(&kv_full[st], (kv_it / L::kStages) & 1);
        tc_fence_after();
        const uint32_t qa = sq_addr + x * L::kTileBytes;
        const uint32_t kb = skv_addr + st * L::kTileBytes;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk / 4) * L::kChunkBytes + (kk % 4) * 32;
          umma_ss_w(tmem + L::s_col(x), smem_desc_sw128(qa + off, 0, 1024),
                  smem_desc_sw128(kb + off, 0, 1024), idesc_qk, kk > 0);
        }
        umma_commit_w(&kv_empty[st]);
        umma_commit_w(&s_full[x]);
        if (last_s) umma_commit_w(&q_empty[x]);
        ++kv_it;
      };
      // O_x (+)= P_x . V : 128 x D, K = 128 keys in steps of 16; P in TMEM
      // (bf16 pairs packed in the S_x columns 0..63).
      auto issue_pv = [&](int x, bool first, bool last, uint32_t ph) {
        const uint32_t st = kv_it % L::kStages;
        mbar_wait(&kv_full[st], (kv_it / L::kStages) & 1);
        tc_fence_after();
        const uint32_t vb = skv_addr + st * L::kTileBytes;
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk) {
          if (kk == kSplitKeys / 16) {
            // the tail of P_x: written after the split arrive
            mbar_wait(&p_full[x], ph);
            tc_fence_after();
          }
          umma_ts_w(tmem + L::o_col(x), tmem + L::s_col(x) + kk * 8,
                  smem_desc_sw128(vb + kk * 16 * 128, L::kChunkBytes, 1024), idesc_pv,
                  (!first) || kk > 0);
        }
        umma_commit_w(&kv_empty[st]);
        if (last) umma_commit_w(&o_done[x]);
        ++kv_it;
      };
      for (long long u = blockIdx.x; u < p.n_units; u += gridDim.x) {
        const Unit w = decode_warp(p, u);
        const int nx = w.has_b ? 2 : 1;
        for (int x = 0; x < nx; ++x) {
          mbar_wait(&q_full[x], ucnt[x] & 1);
          issue_s(x, w.n == 1);
        }
        for (int j = 0; j < w.n; ++j) {
          for (int x = 0; x < nx; ++x) {
            RP_TR(6 + 2 * x, pcnt[x]);
            const uint32_t ph = pcnt[x] & 1;
            mbar_wait(&p_split[x], ph);
            RP_TR(7 + 2 * x, pcnt[x]);
            ++pcnt[x];
            if (j == 0) mbar_wait(&o_free[x], (ucnt[x] & 1) ^ 1);
            tc_fence_after();
            issue_pv(x, j == 0, j == w.n - 1, ph);
            if (j + 1 < w.n) issue_s(x, j + 1 == w.n - 1);
          }
        }
        for (int x = 0; x < nx; ++x) ++ucnt[x];
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;" ::: "memory");
    // --------------------------------------------------------- softmax ----
    const int x = warp / 4;  // tile
    const int wq = warp % 4; // TMEM lane quarter
    const int r = wq * 32 + lane;  // row within the tile
    const uint32_t trow = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    const float sl2 = p.scale_log2;
    uint32_t scnt = 0, ucnt = 0;
    for (long long u = blockIdx.x; u < p.n_units; u += gridDim.x) {
      const Unit w = decode(p, u);
      if (x == 1 && !w.has_b) continue;
      float m = -INFINITY;  // running max (raw logit units), possibly stale
      float l = 0.f;
      for (int j = 0; j < w.n; ++j) {
        if (lane == 0 && wq == 0) RP_TR(3 * x + 0, scnt);
        mbar_wait(&s_full[x], scnt & 1);
        if (lane == 0 && wq == 0) RP_TR(3 * x + 1, scnt);
        ++scnt;
        tc_fence_after();
#ifdef RP_ABL_NOSOFT
        // ablation: no softmax work, P = stale S bits (timing only)
        __syncwarp();
        if (lane == 0) { mbar_arrive(&p_split[x]); mbar_arrive(&p_full[x]); }
        if (lane == 0 && wq == 0) RP_TR(3 * x + 2, scnt - 1);
        continue;
#endif
        uint32_t s0[32], s1[32], s2[32], s3[32];
        tmem_ld32(trow + L::s_col(x) + 0, s0);
        tmem_ld32(trow + L::s_col(x) + 32, s1);
        tmem_ld32(trow + L::s_col(x) + 64, s2);
        tmem_ld32(trow + L::s_col(x) + 96, s3);
        tmem_wait_ld();
        if (lane == 0 && wq == 0 && x == 0) RP_TR(10, scnt - 1);
        auto S = [&](int e) -> float {
          const uint32_t v = e < 32 ? s0[e] : e < 64 ? s1[e - 32] : e < 96 ? s2[e - 64] : s3[e - 96];
          return __uint_as_float(v);
        };
        // row max: four independent 3-input-max chains
        float mq[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float a = S(32 * c);
#pragma unroll
          for (int i = 1; i < 31; i += 2) a = fmaxf(a, fmaxf(S(32 * c + i), S(32 * c + i + 1)));
          mq[c] = fmaxf(a, S(32 * c + 31));
        }
        const float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
        const float m_new = fmaxf(m, mx);
        bool need = false;
        float alpha = 1.0f;
        if (j == 0) {
          m = m_new;
        } else if ((m_new - m) * sl2 > 8.0f) {
          need = true;
          alpha = ex2((m - m_new) * sl2);
          m = m_new;
          l *= alpha;
        }
        // Rescale O before any part of P is published: the P.V that follows
        // the split arrive accumulates into O_x.  (O_x is stable here: S_x(j)
        // was issued after O_x += P_x(j-1) V(j-1) and its commit covers every
        // earlier MMA.)
        if (__any_sync(0xFFFFFFFFu, need)) {
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            tmem_ld32(trow + L::o_col(x) + c * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(trow + L::o_col(x) + c * 32, o);
          }
        }
        // p = 2^(s*scale*log2e - m*scale*log2e), 32 keys per chunk: the
        // chunk's exponentials (MUFU or polynomial on the FMA pipe) issue back
        // to back, then the chunk is summed, packed to bf16 pairs and stored
        // into TMEM columns [16c, 16c+16) of S_x (the A operand of P.V).
        // After kSplitKeys keys the MMA may start P.V on them.
        const float2 sc2 = make_float2(sl2, sl2);
        const float2 ng2 = make_float2(-m * sl2, -m * sl2);
        float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        // Software pipeline over 4 chunks of 32 keys: step c issues chunk c's
        // exponentials and, in the MUFU gaps, sums / packs / stores chunk
        // c-1 (whose MUFU results have long retired).
        float2 pv_prev[16];
#pragma unroll
        for (int c = 0; c <= 4; ++c) {
          float2 pv_cur[16];
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (c < 4) {
              const int e = 32 * c + 2 * i;
              const float2 xv = ffma2v(make_float2(S(e), S(e + 1)), sc2, ng2);
              if (kPolyMask & (1u << (i & 7))) {
                pv_cur[i] = ex2_poly2(xv);
              } else {
                pv_cur[i].x = ex2v(xv.x);
                pv_cur[i].y = ex2v(xv.y);
              }
            }
            if (c > 0) {
              acc[i & 1] = fadd2v(acc[i & 1], pv_prev[i]);
              pk[i] = pack_bf16v(pv_prev[i].x, pv_prev[i].y);
            }
          }
          if (c > 0) {
            tmem_st16(trow + L::s_col(x) + 16 * (c - 1), pk);
            if (32 * c == kSplitKeys) {
              tmem_wait_st();
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&p_split[x]);
            }
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) pv_prev[i] = pv_cur[i];
        }
        if (lane == 0 && wq == 0 && x == 0) RP_TR(11, scnt - 1);
        const float2 at = fadd2(acc[0], acc[1]);
        l += at.x + at.y;
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[x]);
        if (lane == 0 && wq == 0) RP_TR(3 * x + 2, scnt - 1);
      }
      // epilogue: wait for the unit's last P.V, O / l -> bf16 -> global
      mbar_wait(&o_done[x], ucnt & 1);
      ++ucnt;
      tc_fence_after();
      const float inv = 1.0f / l;
      const int h = x ? w.h1 : w.h0;
      const long long tok = static_cast<long long>(w.row) * kBM + r;
      __nv_bfloat16* orow = p.out + tok * p.out_tok_stride + h * p.out_head_stride;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(trow + L::o_col(x) + c * 32, o);
        tmem_wait_ld();
        uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint4 pkt;
          pkt.x = pack_bf16(__uint_as_float(o[8 * v + 0]) * inv, __uint_as_float(o[8 * v + 1]) * inv);
          pkt.y = pack_bf16(__uint_as_float(o[8 * v + 2]) * inv, __uint_as_float(o[8 * v + 3]) * inv);
          pkt.z = pack_bf16(__uint_as_float(o[8 * v + 4]) * inv, __uint_as_float(o[8 * v + 5]) * inv);
          pkt.w = pack_bf16(__uint_as_float(o[8 * v + 6]) * inv, __uint_as_float(o[8 * v + 7]) * inv);
          dst[v] = pkt;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_free[x]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// --------------------------------------------------------------------------
// Descriptor probe (test support): one CTA computes C1 = A . B^T (both
// K-major, SS) and C2 = P . V (P from TMEM, V MN-major) with operands staged
// by plain stores in the same 128B-swizzled layout TMA produces.  Used by the
// GPU tests to pin the UMMA descriptor conventions independently of TMA.
__global__ void __launch_bounds__(128, 1)
    umma_probe_kernel(const __nv_bfloat16* A, const __nv_bfloat16* B,
                      const __nv_bfloat16* P, const __nv_bfloat16* V, float* C1,
                      float* C2) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + 32768;
  uint8_t* sv = smem + 65536;
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int t = threadIdx.x;
  // K-major / MN-major share the physical pattern: row r (128 B per chunk),
  // 16-byte unit XOR (r % 8), chunk c at c * 128 rows * 128 B.
  auto put = [](uint8_t* base, int r, int col, __nv_bfloat16 val) {
    const int chunk = col / 64, b = (col % 64) * 2;
    const int off = chunk * 16384 + r * 128 + (((b / 16) ^ (r % 8)) * 16) + b % 16;
    *reinterpret_cast<__nv_bfloat16*>(base + off) = val;
  };
  for (int i = t; i < 128 * 128; i += 128) {
    const int r = i / 128, c = i % 128;
    put(sa, r, c, A[i]);
    put(sb, r, c, B[i]);
    put(sv, r, c, V[i]);  // row = key, col = d
  }
  if (t == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (t < 32) tmem_alloc<512>(&slot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t idesc_qk = idesc_bf16(128, 128, false, false);
  const uint32_t idesc_pv = idesc_bf16(128, 128, false, true);
  if (t == 0) {
    for (int kk = 0; kk < 8; ++kk) {
      const uint32_t off = (kk / 4) * 16384 + (kk % 4) * 32;
      umma_ss(tmem, smem_desc_sw128(smem_u32(sa) + off, 0, 1024),
              smem_desc_sw128(smem_u32(sb) + off, 0, 1024), idesc_qk, kk > 0);
    }
    umma_commit(&bar);
  }
  // P rows into TMEM columns 256.. (packed bf16 pairs)
  {
    const int wq = t / 32;
    const uint32_t trow = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    uint32_t pk[32];
    for (int half = 0; half < 2; ++half) {
      for (int i = 0; i < 32; ++i) {
        const int k0 = half * 64 + 2 * i;
        __nv_bfloat162 v2;
        v2.x = P[t * 128 + k0];
        v2.y = P[t * 128 + k0 + 1];
        pk[i] = *reinterpret_cast<uint32_t*>(&v2);
      }
      tmem_st32(trow + 256 + half * 32, pk);
    }
    tmem_wait_st();
  }
  mbar_wait(&bar, 0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (t == 0) {
    for (int kk = 0; kk < 8; ++kk)
      umma_ts(tmem + 128, tmem + 256 + kk * 8,
              smem_desc_sw128(smem_u32(sv) + kk * 16 * 128, 16384, 1024), idesc_pv,
              kk > 0);
    umma_commit(&bar);
  }
  mbar_wait(&bar, 1);
  tc_fence_after();
  {
    const int wq = t / 32;
    const uint32_t trow = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    for (int c = 0; c < 8; ++c) {
      uint32_t o[32];
      tmem_ld32(trow + c * 32, o);
      tmem_wait_ld();
      float* dst = c < 4 ? C1 + t * 128 + c * 32 : C2 + t * 128 + (c - 4) * 32;
      for (int i = 0; i < 32; ++i) dst[i] = __uint_as_float(o[i]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (t < 32) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace attn
}  // namespace rp
