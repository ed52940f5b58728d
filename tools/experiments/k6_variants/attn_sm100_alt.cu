// K6 (v5, "alt"): block-sparse flash-attention forward with the KV steps of
// a query tile alternating between two softmax groups, each with its own
// output accumulator (bf16 in / fp32 softmax, sm_100a).
//
// Same semantics as attn_sm100_db.cu (attention.cpp:50-121, exact mask,
// zero-padded keys attended when their block is active).
//
// Why.  db splits each 128-key step between two warps per row group, so the
// two must agree on the row max every step: a 64-thread named barrier per
// step is its top stall (ncu: 1.27 warps stalled on barrier per issue) and a
// rescale must wait for the previous step's P.V.  Here group x (warps
// 4x..4x+3, thread = one query row, all 128 keys) owns the steps j = x, x+2,
// ... of each unit and accumulates into its own O_x with its own running max
// and sum -- two independent online softmaxes over the even and odd KV
// blocks, merged once per unit in the epilogue:
//   O = (O_0 2^(m_0 - M) + O_1 2^(m_1 - M)) / (l_0 2^(m_0 - M) + l_1 2^(m_1 - M)).
// No per-step exchange, and a rescale of O_x never waits: O_x's last P.V is
// step j-2's, which retired before S(j) was signalled (S(g+2) is issued after
// P(g).V(g)).  Both groups run concurrently on alternate steps, so each SM
// sub-partition still has two softmax warps interleaving MUFU / FMA work.
//   TMEM  S0 cols 0-127 | S1 128-255 | O_0 256-(256+D) | O_1 384-(384+D)
// Q stays in shared memory (two unit buffers; S = Q K^T reads both operands
// from shared memory).  The score tile is double-buffered as in db.
//
//   warps 0-3 softmax group 0 (even steps)   warp 8  TMA producer
//   warps 4-7 softmax group 1 (odd steps)    warp 9  MMA issuer
//   warps 10-11 idle (setmaxnreg group)
#include "common.cuh"

namespace rp {
namespace attn5 {

using attn2::Cursor;
using attn2::Params;

constexpr int kThreads = 384;
constexpr int kBM = 128;
constexpr int kBN = 128;
#ifndef RP_ALT_POLY_MASK
#define RP_ALT_POLY_MASK 0x00u
#endif
constexpr uint32_t kPolyMask = RP_ALT_POLY_MASK;

template <int D>
struct Layout {
  static constexpr int kChunks = D / 64;
  static constexpr int kTileBytes = 128 * D * 2;
  static constexpr int kChunkBytes = 128 * 128;
#ifdef RP_ALT_STAGES
  static constexpr int kStages = RP_ALT_STAGES;
#else
  static constexpr int kStages = D == 128 ? 4 : 8;
#endif
  static constexpr int kSmemData = 2 * kTileBytes + kStages * kTileBytes;
  static constexpr int kNumBars = 2 * kStages + 10;
  static constexpr int kRedBytes = 2 * 2 * 128 * 4;  // (m, l) per group and row
  static constexpr int kSmemBytes = kSmemData + kNumBars * 8 + 16 + kRedBytes + 1024;
  static_assert(kSmemBytes <= 232448, "exceeds the 227 KB opt-in shared memory");
  RP_HD static uint32_t o_col(int x) { return x ? 384u : 256u; }
};

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    bsfa_fwd_alt_kernel(const __grid_constant__ CUtensorMap tq,
                        const __grid_constant__ CUtensorMap tk,
                        const __grid_constant__ CUtensorMap tv, const Params p) {
  using L = Layout<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sq = smem;                       // [2][tile]
  uint8_t* skv = smem + 2 * L::kTileBytes;  // [kStages][tile]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kSmemData);
  uint64_t* kv_full = bars;
  uint64_t* kv_empty = bars + L::kStages;
  uint64_t* q_full = bars + 2 * L::kStages;  // [2]
  uint64_t* q_empty = q_full + 2;            // [2] MMA commit: unit's last S read Q
  uint64_t* s_full = q_full + 4;             // [2] MMA -> softmax: S_b ready
  uint64_t* p_full = q_full + 6;             // [2] softmax group -> MMA: P_b written (4 warps)
  uint64_t* o_done = q_full + 8;             // MMA -> softmax: unit's last P.V retired
  uint64_t* o_free = q_full + 9;             // softmax -> MMA: epilogue read O_0, O_1 (8 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + L::kNumBars);
  float* red = reinterpret_cast<float*>(tmem_slot + 4);  // [group][m, l][128]

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
    }
    mbar_init(o_done, 1);
    mbar_init(o_free, 8);
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
      // Ring order = MMA consumption order: K(0), K(1), then V(g), K(g+2).
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();
      uint32_t kv_it = 0;
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
      Cursor ck, cv;
      ck.start(p);
      cv.start(p);
      auto load_k = [&]() {
        if (ck.j == 0) {  // entering a unit: its Q tile first
          const int qb = ck.ord & 1;
          mbar_wait(&q_empty[qb], ((ck.ord >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx_w(&q_full[qb], L::kTileBytes);
#pragma unroll
          for (int c = 0; c < L::kChunks; ++c)
            tma_load_3d_w(sq + qb * L::kTileBytes + c * L::kChunkBytes, &tq, &q_full[qb], c * 64,
                          ck.h, ck.row * kBM, pol_q);
        }
        load_kv(&tk, ck.h, ck.col(p));
        ck.next(p);
      };
      if (ck.valid) load_k();
      if (ck.valid) load_k();
      while (cv.valid) {
        load_kv(&tv, cv.h, cv.col(p));
        cv.next(p);
        if (ck.valid) load_k();
      }
    } else if (warp == 9) {
      // ----------------------------------------------------- MMA issuer ---
      const uint32_t idesc_qk = idesc_bf16(128, 128, false, false);
      const uint32_t idesc_pv = idesc_bf16(128, D, false, true);
      const uint32_t sq_addr = smem_u32(sq);
      const uint32_t skv_addr = smem_u32(skv);
      uint32_t kv_it = 0, gs = 0, gp = 0;
      Cursor cs, cp;
      cs.start(p);
      cp.start(p);
      // S(gs) = Q . K(gs)^T into buffer gs % 2 (both operands in shared memory)
      auto issue_s = [&]() {
        const int qb = cs.ord & 1;
        if (cs.j == 0) mbar_wait(&q_full[qb], (cs.ord >> 1) & 1);
        const uint32_t st = kv_it % L::kStages;
        mbar_wait(&kv_full[st], (kv_it / L::kStages) & 1);
        tc_fence_after();
        const uint32_t qa = sq_addr + qb * L::kTileBytes;
        const uint32_t kb = skv_addr + st * L::kTileBytes;
        const uint32_t dst = tmem + (gs & 1) * 128;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk / 4) * L::kChunkBytes + (kk % 4) * 32;
          umma_ss_w(dst, smem_desc_sw128(qa + off, 0, 1024), smem_desc_sw128(kb + off, 0, 1024),
                    idesc_qk, kk > 0);
        }
        umma_commit_w(&kv_empty[st]);
        umma_commit_w(&s_full[gs & 1]);
        if (cs.j == cs.n - 1) umma_commit_w(&q_empty[qb]);  // Q(unit) read for the last time
        ++kv_it;
        ++gs;
        cs.next(p);
      };
      if (cs.valid) issue_s();
      if (cs.valid) issue_s();
      while (cp.valid) {
        const uint32_t b = gp & 1;
        mbar_wait(&p_full[b], (gp >> 1) & 1);
        if (cp.j == 0 && cp.ord > 0) mbar_wait(o_free, (cp.ord - 1) & 1);
        const uint32_t st = kv_it % L::kStages;
        mbar_wait(&kv_full[st], (kv_it / L::kStages) & 1);
        tc_fence_after();
        // O_(j % 2) (+)= P(gp) . V(gp): P bf16 pairs in TMEM columns [128b, 128b+64)
        const uint32_t vb = skv_addr + st * L::kTileBytes;
        const uint32_t oc = L::o_col(cp.j & 1);
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk)
          umma_ts_w(tmem + oc, tmem + b * 128 + kk * 8,
                    smem_desc_sw128(vb + kk * 16 * 128, L::kChunkBytes, 1024), idesc_pv,
                    (cp.j >= 2) || kk > 0);
        umma_commit_w(&kv_empty[st]);
        if (cp.j == cp.n - 1) umma_commit_w(o_done);
        ++kv_it;
        ++gp;
        cp.next(p);
        if (cs.valid) issue_s();  // S(gp + 1) into the buffer P(gp - 1) just released
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;" ::: "memory");
    // ------------------------------------------------------- softmax -----
    const int x = warp / 4;   // group: steps j = x, x + 2, ...
    const int wq = warp % 4;  // TMEM lane quarter
    const int r = wq * 32 + lane;
    const uint32_t trow = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    const float sl2 = p.scale_log2;
    uint32_t gbase = 0;  // global step index of the unit's first block
    int ord = 0;
    for (long long u = blockIdx.x; u < p.n_units; u += gridDim.x) {
      const int h = static_cast<int>(u / p.n_rows);
      const int ri = static_cast<int>(u % p.n_rows);
      const int row = p.row_order ? __ldg(p.row_order + ri) : ri;
      const int beg = __ldg(p.row_ptr + row);
      const int n = __ldg(p.row_ptr + row + 1) - beg;
      __nv_bfloat16* orow = p.out + (static_cast<long long>(row) * kBM + r) * p.out_tok_stride +
                            h * p.out_head_stride + x * (D / 2);
      if (n == 0) {  // no active block: defined output (zeros); no pipeline traffic
        const uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int v = 0; v < D / 16; ++v) reinterpret_cast<uint4*>(orow)[v] = z;
        continue;
      }
      float m = -INFINITY;  // this group's running max (raw logits), possibly stale
      float l = 0.f;        // this group's row sum
      for (int j = x; j < n; j += 2) {
        const uint32_t g = gbase + j;
        const uint32_t b = g & 1;
        const uint32_t sb = b * 128;
        mbar_wait(&s_full[b], (g >> 1) & 1);
        tc_fence_after();
        uint32_t s0[32], s1[32], s2[32], s3[32];
        tmem_ld32(trow + sb + 0, s0);
        tmem_ld32(trow + sb + 32, s1);
        tmem_ld32(trow + sb + 64, s2);
        tmem_ld32(trow + sb + 96, s3);
        tmem_wait_ld();
        auto S = [&](int e) -> float {
          const uint32_t v = e < 32 ? s0[e] : e < 64 ? s1[e - 32] : e < 96 ? s2[e - 64] : s3[e - 96];
          return __uint_as_float(v);
        };
        const bool first = j == x;
        if (first) {
          float a = S(0);
#pragma unroll
          for (int i = 1; i < 127; i += 2) a = fmaxf(a, fmaxf(S(i), S(i + 1)));
          m = fmaxf(a, S(127));
        }
        // exponentials against the (stale) reference max, 16-key chunks: a
        // chunk's exponentials overlap the packing and TMEM store of the
        // previous one; this block's max is folded in alongside
        float2 acc[2];
        float lmax = -INFINITY;
        auto exps = [&](float mref, bool track) {
          const float2 sc2 = make_float2(sl2, sl2);
          const float2 ng2 = make_float2(-mref * sl2, -mref * sl2);
          acc[0] = acc[1] = make_float2(0.f, 0.f);
          float2 pv_prev[8];
#pragma unroll
          for (int c = 0; c <= 8; ++c) {
            float2 pv_cur[8];
            uint32_t pk[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (c < 8) {
                const int e = 16 * c + 2 * i;
                if (track) lmax = fmaxf(lmax, fmaxf(S(e), S(e + 1)));
                const float2 xv = ffma2v(make_float2(S(e), S(e + 1)), sc2, ng2);
                if (kPolyMask & (1u << i)) {
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
            if (c > 0) tmem_st8(trow + sb + 8 * (c - 1), pk);
#pragma unroll
            for (int i = 0; i < 8; ++i) pv_prev[i] = pv_cur[i];
          }
        };
        exps(m, false);
        // rescale guard from the row sum (see attn_sm100_db.cu)
        const float2 at0 = fadd2(acc[0], acc[1]);
        if (!first && __any_sync(0xFFFFFFFFu, !(at0.x + at0.y <= 256.0f))) {
          float a = S(0);
#pragma unroll
          for (int i = 1; i < 127; i += 2) a = fmaxf(a, fmaxf(S(i), S(i + 1)));
          lmax = fmaxf(a, S(127));
          const bool need = (lmax - m) * sl2 > 8.0f;
          if (__any_sync(0xFFFFFFFFu, need)) {
            // rebase O_x and l on the new max: O_x is stable (its last P.V,
            // step j-2, retired before S(j) was signalled)
            const float alpha = need ? ex2((m - lmax) * sl2) : 1.0f;
            if (need) {
              m = lmax;
              l *= alpha;
            }
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
              uint32_t o[32];
              tmem_ld32(trow + L::o_col(x) + c * 32, o);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
              tmem_st32(trow + L::o_col(x) + c * 32, o);
            }
            tmem_wait_st();
            exps(m, false);
          }
        }
        const float2 at = fadd2(acc[0], acc[1]);
        l += at.x + at.y;
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[b]);
      }
      gbase += n;
      // epilogue: merge the two groups' (m, l) per row, then this group's
      // D/2 output columns from both accumulators
      red[(x * 2 + 0) * 128 + r] = m;
      red[(x * 2 + 1) * 128 + r] = l;
      mbar_wait(o_done, ord & 1);
      tc_fence_after();
      asm volatile("bar.sync %0, 64;" ::"r"(1 + wq) : "memory");
      const float mo = red[((1 - x) * 2 + 0) * 128 + r];
      const float lo = red[((1 - x) * 2 + 1) * 128 + r];
      const float m0 = x ? mo : m, l0 = x ? lo : l;
      const float m1 = x ? m : mo, l1 = x ? l : lo;
      const float M = fmaxf(m0, m1);
      const float f0 = l0 > 0.f ? ex2((m0 - M) * sl2) : 0.f;  // group 1 may have no step
      const float f1 = l1 > 0.f ? ex2((m1 - M) * sl2) : 0.f;
      const float inv = 1.0f / (l0 * f0 + l1 * f1);
      const float a0 = f0 * inv, a1 = f1 * inv;
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        const uint32_t col = x * (D / 2) + c * 32;
        uint32_t o0[32], o1[32];
        tmem_ld32(trow + L::o_col(0) + col, o0);
        tmem_ld32(trow + L::o_col(1) + col, o1);
        tmem_wait_ld();
        uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
        auto v = [&](int i) {
          // O_1 is uninitialised when the unit has a single block (a1 = 0)
          const float b1 = a1 != 0.f ? __uint_as_float(o1[i]) * a1 : 0.f;
          return __uint_as_float(o0[i]) * a0 + b1;
        };
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          uint4 pkt;
          pkt.x = pack_bf16(v(8 * q4 + 0), v(8 * q4 + 1));
          pkt.y = pack_bf16(v(8 * q4 + 2), v(8 * q4 + 3));
          pkt.z = pack_bf16(v(8 * q4 + 4), v(8 * q4 + 5));
          pkt.w = pack_bf16(v(8 * q4 + 6), v(8 * q4 + 7));
          dst[q4] = pkt;
        }
      }
      tc_fence_before();
      // red is rewritten next unit only after both groups passed this barrier
      asm volatile("bar.sync %0, 64;" ::"r"(1 + wq) : "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(o_free);
      ++ord;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace attn5
}  // namespace rp
