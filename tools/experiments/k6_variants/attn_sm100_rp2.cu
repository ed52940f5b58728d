// K6 (v4, "rp2"): block-sparse flash-attention forward with two query row
// blocks of one head sharing every K/V tile AND a double-buffered score tile
// per query tile (bf16 in / fp32 softmax, sm_100a).
//
// Same semantics as attn_sm100_db.cu / attn_sm100_rp.cu (attention.cpp:50-121,
// exact mask, zero-padded keys attended when their block is active).
//
// Why.  db (one query tile per CTA, S double-buffered) streams a 32 KB K and a
// 32 KB V tile through L2 per 128 x 128 step -- ~7.6 TB/s at the Wan shape,
// near the L2 cap (ablation: skipping the reloads is worth 16 %).  rp shares
// K/V between the row pair (2p, 2p+1) but, with one S buffer per tile, each
// tile's chain softmax -> P.V -> S -> softmax serialises; union entries held
// by one row of the pair leave the other tile idle.  Here each tile keeps TWO
// score buffers, which fit only at half-block granularity: a KV block is
// processed as two 64-key half-steps (S: M=128, N=64, K=D; P.V: K=64), so
//   TMEM  S_A0 0-63 | S_A1 64-127 | S_B0 128-191 | S_B1 192-255 |
//         O_A 256-(256+D) | O_B 384-(384+D)
// and each tile runs db's pipeline (S of half-step g+2 is issued right after
// P.V of half-step g, so the softmax never waits on the tensor core) while
// the pair shares K/V.  P (bf16) overwrites the first 32 columns of its S
// buffer and is the TMEM A operand of P.V.
//
// MMA order per union entry e (flags say which tile holds the block):
//   for hs in {0, 1}:  P_A(e-1, hs) V, S_A(e, hs), P_B(e-1, hs) V, S_B(e, hs)
// so the ring stays FIFO (V(e-1) then K(e)), every S buffer is rewritten only
// after the P.V that read it was issued, and a rescale (which needs the
// previous half-step's P.V retired) waits on a per-tile pv_done barrier.
//
//   warps 0-3  softmax / epilogue of tile A (row 2p)   warp 8  TMA producer
//   warps 4-7  softmax / epilogue of tile B (row 2p+1) warp 9  MMA issuer
//   warps 10-11 idle (setmaxnreg group)
// One softmax warp per tile per SM sub-partition: a thread owns one query row
// for the whole unit (no cross-warp max exchange), 64 keys per half-step.
#include "common.cuh"

namespace rp {
namespace attn4 {

using attn3::Params;
using attn3::Unit;
using attn3::decode;

constexpr int kThreads = 384;
constexpr int kBM = 128;
constexpr int kBN = 128;
#ifndef RP_RP2_POLY_MASK
#define RP_RP2_POLY_MASK 0x01u
#endif
constexpr uint32_t kPolyMask = RP_RP2_POLY_MASK;

template <int D>
struct Layout {
  static constexpr int kChunks = D / 64;
  static constexpr int kTileBytes = 128 * D * 2;
  static constexpr int kChunkBytes = 128 * 128;
  static constexpr int kHalfRows = 64 * 128;  // byte offset of key row 64 in a chunk
  static constexpr int kStages = D == 128 ? 5 : 10;
  static constexpr int kSmemData = 2 * kTileBytes + kStages * kTileBytes;
  static constexpr int kNumBars = 2 * kStages + 18;
  static constexpr int kSmemBytes = kSmemData + kNumBars * 8 + 16 + 1024;
  static_assert(kSmemBytes <= 232448, "exceeds the 227 KB opt-in shared memory");
  RP_HD static uint32_t s_col(int x, uint32_t b) { return 128u * x + 64u * b; }
  RP_HD static uint32_t o_col(int x) { return x ? 384u : 256u; }
};

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    bsfa_fwd_rp2_kernel(const __grid_constant__ CUtensorMap tq,
                        const __grid_constant__ CUtensorMap tk,
                        const __grid_constant__ CUtensorMap tv, const Params p) {
  using L = Layout<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sq = smem;
  uint8_t* skv = smem + 2 * L::kTileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kSmemData);
  uint64_t* kv_full = bars;
  uint64_t* kv_empty = bars + L::kStages;
  uint64_t* q_full = bars + 2 * L::kStages;  // [2] per tile
  uint64_t* q_empty = q_full + 2;            // [2]
  uint64_t* s_full = q_full + 4;             // [2 tiles][2 buffers]
  uint64_t* p_full = q_full + 8;             // [2 tiles][2 buffers], 4 warps each
  uint64_t* pv_done = q_full + 12;           // [2] a P.V of the tile retired
  uint64_t* o_done = q_full + 14;            // [2] the unit's last P.V retired
  uint64_t* o_free = q_full + 16;            // [2] epilogue read O (4 warps)
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
      for (int b = 0; b < 2; ++b) {
        mbar_init(&s_full[2 * x + b], 1);
        mbar_init(&p_full[2 * x + b], 4);
      }
      mbar_init(&pv_done[x], 1);
      mbar_init(&o_done[x], 1);
      mbar_init(&o_free[x], 4);
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

  if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;" ::: "memory");
    if (warp == 8) {
      // ---------------------------------------------------- TMA producer --
      // ring order = MMA consumption order: K(0), then V(e-1), K(e), ...
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();
      uint32_t kv_it = 0;
      uint32_t ucnt[2] = {0, 0};
      auto load_kv = [&](const CUtensorMap* m, int h, int blk) {
        const uint32_t st = kv_it % L::kStages;
        mbar_wait(&kv_empty[st], ((kv_it / L::kStages) & 1) ^ 1);
        mbar_arrive_expect_tx_w(&kv_full[st], L::kTileBytes);
        uint8_t* dst = skv + st * L::kTileBytes;
#pragma unroll
        for (int c = 0; c < L::kChunks; ++c)
          tma_load_3d_w(dst + c * L::kChunkBytes, m, &kv_full[st], c * 64, h, blk * kBN, pol_kv);
        ++kv_it;
      };
      for (long long u = blockIdx.x; u < p.n_units; u += gridDim.x) {
        const Unit w = decode(p, u, true);
        if (w.n == 0) continue;
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          if (!w.has[x]) continue;
          mbar_wait(&q_empty[x], (ucnt[x] & 1) ^ 1);
          mbar_arrive_expect_tx_w(&q_full[x], L::kTileBytes);
#pragma unroll
          for (int c = 0; c < L::kChunks; ++c)
            tma_load_3d_w(sq + x * L::kTileBytes + c * L::kChunkBytes, &tq, &q_full[x], c * 64,
                          w.h, w.row[x] * kBM, pol_q);
          ++ucnt[x];
        }
        const int32_t* cols = p.pcol + w.beg;
        int prev = 0;
        for (int e = 0; e <= w.n; ++e) {
          if (e > 0) load_kv(&tv, w.h, prev);
          if (e < w.n) {
            const int c = shfl0(__ldg(cols + e));
            load_kv(&tk, w.h, c);
            prev = c;
          }
        }
      }
    } else if (warp == 9) {
      // ----------------------------------------------------- MMA issuer ---
      const uint32_t idesc_qk = idesc_bf16(128, 64, false, false);
      const uint32_t idesc_pv = idesc_bf16(128, D, false, true);
      const uint32_t sq_addr = smem_u32(sq);
      const uint32_t skv_addr = smem_u32(skv);
      uint32_t kv_it = 0;
      uint32_t ucnt[2] = {0, 0};
      uint32_t sg[2] = {0, 0};  // S half-steps issued per tile (running)
      uint32_t pg[2] = {0, 0};  // P.V half-steps issued per tile (running)
      for (long long u = blockIdx.x; u < p.n_units; u += gridDim.x) {
        const Unit w = decode(p, u, true);
        if (w.n == 0) continue;
        const uint8_t* flags = p.pflag + w.beg;
        int ds[2] = {0, 0}, dp[2] = {0, 0};  // half-steps of this unit
        const int nh[2] = {2 * w.cnt[0], 2 * w.cnt[1]};
        uint32_t pfl = 0;
        for (int e = 0; e <= w.n; ++e) {
          const uint32_t fl = e < w.n ? static_cast<uint32_t>(shfl0(__ldg(flags + e))) : 0u;
          uint32_t v_st = 0, k_st = 0;
          if (e > 0) {
            v_st = kv_it % L::kStages;
            mbar_wait(&kv_full[v_st], (kv_it / L::kStages) & 1);
            ++kv_it;
          }
          if (e < w.n) {
            k_st = kv_it % L::kStages;
            mbar_wait(&kv_full[k_st], (kv_it / L::kStages) & 1);
            ++kv_it;
          }
          tc_fence_after();
#pragma unroll
          for (int hs = 0; hs < 2; ++hs) {
#pragma unroll
            for (int x = 0; x < 2; ++x) {
              if (e > 0 && ((pfl >> x) & 1)) {
                // O_x (+)= P_x(e-1, hs) . V(e-1)[64 hs .. 64 hs + 63]
                const uint32_t b = pg[x] & 1;
                mbar_wait(&p_full[2 * x + b], (pg[x] >> 1) & 1);
                if (dp[x] == 0) mbar_wait(&o_free[x], (ucnt[x] & 1) ^ 1);
                tc_fence_after();
                const uint32_t vb = skv_addr + v_st * L::kTileBytes;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                  umma_ts_w(tmem + L::o_col(x), tmem + L::s_col(x, b) + kk * 8,
                            smem_desc_sw128(vb + (4 * hs + kk) * 16 * 128, L::kChunkBytes, 1024),
                            idesc_pv, dp[x] > 0 || kk > 0);
                umma_commit_w(&pv_done[x]);
                ++dp[x];
                ++pg[x];
                if (dp[x] == nh[x]) umma_commit_w(&o_done[x]);
              }
              if (e < w.n && ((fl >> x) & 1)) {
                // S_x(e, hs) = Q_x K(e)[64 hs .. 64 hs + 63]^T into buffer sg % 2
                // (per tile right after its own P.V: a tile never waits on the
                // other tile's softmax for its next score tile)
                const uint32_t b = sg[x] & 1;
                if (ds[x] == 0) mbar_wait(&q_full[x], ucnt[x] & 1);
                tc_fence_after();
                const uint32_t qa = sq_addr + x * L::kTileBytes;
                const uint32_t kb = skv_addr + k_st * L::kTileBytes + hs * L::kHalfRows;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                  const uint32_t off = (kk / 4) * L::kChunkBytes + (kk % 4) * 32;
                  umma_ss_w(tmem + L::s_col(x, b), smem_desc_sw128(qa + off, 0, 1024),
                            smem_desc_sw128(kb + off, 0, 1024), idesc_qk, kk > 0);
                }
                umma_commit_w(&s_full[2 * x + b]);
                ++ds[x];
                ++sg[x];
                if (ds[x] == nh[x]) umma_commit_w(&q_empty[x]);
              }
            }
          }
          if (e > 0) umma_commit_w(&kv_empty[v_st]);
          if (e < w.n) umma_commit_w(&kv_empty[k_st]);
          pfl = fl;
        }
#pragma unroll
        for (int x = 0; x < 2; ++x)
          if (w.has[x]) ++ucnt[x];
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;" ::: "memory");
    // --------------------------------------------------------- softmax ----
    const int x = warp / 4;
    const int wq = warp % 4;
    const int r = wq * 32 + lane;
    const uint32_t trow = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    const float sl2 = p.scale_log2;
    uint32_t g = 0, ucnt = 0;
    for (long long u = blockIdx.x; u < p.n_units; u += gridDim.x) {
      const Unit w = decode(p, u, false);
      // (selects, not w.row[x]: a runtime index would put the Unit in local memory)
      const int my_row = x ? w.row[1] : w.row[0];
      const int my_cnt = x ? w.cnt[1] : w.cnt[0];
      const bool my_has = x ? w.has[1] : w.has[0];
      if (my_row >= p.n_rows) continue;
      __nv_bfloat16* orow = p.out + (static_cast<long long>(my_row) * kBM + r) *
                                         p.out_tok_stride + w.h * p.out_head_stride;
      if (!my_has) {  // empty block row: defined output (zeros)
        const uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int v = 0; v < D / 8; ++v) reinterpret_cast<uint4*>(orow)[v] = z;
        continue;
      }
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < 2 * my_cnt; ++j, ++g) {
        const uint32_t b = g & 1;
        const uint32_t sc = L::s_col(x, b);
        mbar_wait(&s_full[2 * x + b], (g >> 1) & 1);
        tc_fence_after();
        uint32_t s0[32], s1[32];
        tmem_ld32(trow + sc, s0);
        tmem_ld32(trow + sc + 32, s1);
        tmem_wait_ld();
        auto S = [&](int e) -> float { return __uint_as_float(e < 32 ? s0[e] : s1[e - 32]); };
        if (j == 0) {
          float a = S(0);
#pragma unroll
          for (int i = 1; i < 63; i += 2) a = fmaxf(a, fmaxf(S(i), S(i + 1)));
          m = fmaxf(a, S(63));
        }
        // exponentials against the (stale) reference max, see attn_sm100_db.cu
        float2 acc[2];
        uint32_t pk[32];
        float lmax = -INFINITY;
        auto exps = [&](float mref, bool track) {
          const float2 sc2 = make_float2(sl2, sl2);
          const float2 ng2 = make_float2(-mref * sl2, -mref * sl2);
          acc[0] = acc[1] = make_float2(0.f, 0.f);
          float2 pv_prev[16];
#pragma unroll
          for (int c = 0; c <= 2; ++c) {
            float2 pv_cur[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              if (c < 2) {
                const int e = 32 * c + 2 * i;
                if (track) lmax = fmaxf(lmax, fmaxf(S(e), S(e + 1)));
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
                pk[16 * (c - 1) + i] = pack_bf16v(pv_prev[i].x, pv_prev[i].y);
              }
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) pv_prev[i] = pv_cur[i];
          }
        };
        exps(m, j > 0);
        if (j > 0) {
          const bool need = (lmax - m) * sl2 > 8.0f;
          if (__any_sync(0xFFFFFFFFu, need)) {
            const float alpha = need ? ex2((m - lmax) * sl2) : 1.0f;
            if (need) {
              m = lmax;
              l *= alpha;
            }
            // O_x must hold P(g-1).V before it is rescaled (P(g-2).V retired
            // before S(g) was signalled, so one phase decides)
            mbar_wait(&pv_done[x], (g - 1) & 1);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
              uint32_t o[32];
              tmem_ld32(trow + L::o_col(x) + c * 32, o);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
              tmem_st32(trow + L::o_col(x) + c * 32, o);
            }
            exps(m, false);
          }
        }
        const float2 at = fadd2(acc[0], acc[1]);
        l += at.x + at.y;
        tmem_st32(trow + sc, pk);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[2 * x + b]);
      }
      // epilogue: the tile's last P.V done -> O / l -> bf16 -> global
      mbar_wait(&o_done[x], ucnt & 1);
      ++ucnt;
      tc_fence_after();
      const float inv = 1.0f / l;
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

}  // namespace attn4
}  // namespace rp
