// K6 (v8, "mc"): db (one query tile per CTA, S double-buffered, Q in TMEM,
// cta_group::1 MMAs) on CTA PAIRS whose shared K/V tiles are TMA-MULTICAST
// (bf16 in / fp32 softmax, sm_100a, head_dim 128).
//
// Same semantics as attn_sm100_db.cu (attention.cpp:50-121).
//
// Why.  With the natural unit order the db kernel streams ~8.4 TB/s of K/V
// tiles from L2 into the SMs, close to the L2 throughput cap.  The CTAs of a
// cluster pair own block rows (2p, 2p+1) of one head, whose lists share ~72 %
// of their union (Wan config-3 mask): each tile both rows hold is read from
// L2 once and multicast into both SMs' shared memory.  Unlike rp / cta2 no
// work is wasted on blocks outside a row's own list -- each CTA computes
// only its own steps, exactly as db does.
//
// Coupling.  Both CTAs walk the UNION in the same ring order (db's order:
// K(0), K(1), V(0), K(2), V(1), ... over union entries), so a ring slot holds
// the same tile in both SMs.  Per slot: the leader issues the multicast TMA
// for common tiles, a CTA loads its own single-member tiles, and the other
// CTA just arrives (0 bytes) on its full barrier and releases the slot
// without touching it.  A slot is free for the next tile when BOTH CTAs'
// consumers released it (kv_empty count 2: MMA commits are multicast to both
// CTAs, skips arrive locally and remotely with relaxed arrivals).
#include "common.cuh"

#define RP_TR_NONE(ev, idx) \
  do {                  \
  } while (0)

namespace rp {
namespace attn8 {

using attn3::decode;
using attn3::Params;
using attn3::Unit;
using attn7::cluster_count;
using attn7::cluster_id;
using attn7::cluster_rank;
using attn7::cluster_sync_all;

constexpr int kThreads = 384;
constexpr int kBM = 128;
constexpr int kBN = 128;
// Pairs (of every 8) whose exp2 runs as a polynomial on the FMA pipe.
#ifndef RP_MC_POLY_MASK
#define RP_MC_POLY_MASK 0x01u
#endif
constexpr uint32_t kPolyMask = RP_MC_POLY_MASK;

template <int D>
struct Layout {
  static constexpr int kChunks = D / 64;          // 128-byte K chunks per row
  static constexpr int kTileBytes = 128 * D * 2;  // one 128-row bf16 tile
  static constexpr int kChunkBytes = 128 * 128;
#ifdef RP_MC_STAGES
  static constexpr int kStages = RP_MC_STAGES;
#else
  static constexpr int kStages = D == 128 ? 4 : 8;  // 2 Q tiles + ring <= 227 KB
#endif
  static constexpr int kSmemData = 2 * kTileBytes + kStages * kTileBytes;
  static constexpr int kNumBars = 2 * kStages + 13 + 2;
  static constexpr int kRedBytes = (2 * 2 * 128 + 2 * 128 + 2 * 2 * 128) * 4;
  static constexpr int kSmemBytes = kSmemData + kNumBars * 8 + 16 + kRedBytes + 1024;
  static_assert(kSmemBytes <= 232448, "exceeds the 227 KB opt-in shared memory");
  static constexpr uint32_t kO = 256;  // TMEM column of O
  // Q tiles as the A operand of S = Q K^T live in TMEM (bf16 pairs, D/2
  // columns each, double-buffered by unit): the tensor core then reads only
  // K from shared memory for S, which cuts the step's shared-memory traffic
  // (Q 32 KB + K 32 KB + V 32 KB reads + 64 KB TMA writes) by a fifth.
  RP_HD static uint32_t qt_col(int b) { return 384u + (b ? 64u : 0u); }
};

// shared::cluster address of `bar` in CTA `rank`
RP_DEV uint32_t peer_addr(uint64_t* bar, uint32_t rank) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(bar)), "r"(rank));
  return a;
}
// commit: arrive on the barrier at this offset in both CTAs once this
// thread's prior tcgen05 ops retired
RP_DEV void umma_commit_both_w(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b16 m;\n\t"
      "mov.b16 m, 3;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], m;\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
// TMA multicast into both CTAs (same smem offset, each CTA's barrier)
RP_DEV void tma_mc_load_3d_w(void* smem_dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1,
                             int c2, uint64_t policy) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b16 msk;\n\t"
      "mov.b16 msk, 3;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::"
      "cluster.L2::cache_hint [%0], [%1, {%3, %4, %5}], [%2], msk, %6;\n\t}" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "l"(policy)
      : "memory");
}

// Stream of union entries over this cluster's pair-units (warp-uniform).
struct MCursor {
  long long u;
  int e, n, beg, h;
  int own_cnt, own_ord, d;  // this CTA's list length, ordinal among own-nonempty units, own index
  bool valid;
  RP_DEV void load(const Params& p) {
    valid = false;
    for (; u < p.n_units; u += cluster_count()) {
      const Unit w = decode(p, u, true);
      if (w.n > 0) {
        n = w.n;
        beg = w.beg;
        h = w.h;
        own_cnt = cluster_rank() ? w.cnt[1] : w.cnt[0];
        e = 0;
        d = 0;
        valid = true;
        return;
      }
    }
  }
  RP_DEV void start(const Params& p) {
    u = cluster_id();
    own_ord = 0;
    load(p);
  }
  RP_DEV uint32_t flag(const Params& p) const {
    return static_cast<uint32_t>(shfl0(__ldg(p.pflag + beg + e)));
  }
  RP_DEV int col(const Params& p) const { return shfl0(__ldg(p.pcol + beg + e)); }
  RP_DEV void next(const Params& p, bool mine) {
    if (mine) ++d;
    if (++e < n) return;
    if (own_cnt > 0) ++own_ord;
    u += cluster_count();
    load(p);
  }
};

template <int D>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    bsfa_fwd_mc_kernel(const __grid_constant__ CUtensorMap tq,
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
  uint64_t* q_empty = q_full + 2;            // [2]
  uint64_t* s_full = q_full + 4;             // [2] MMA -> softmax: S_b ready
  uint64_t* p_full = q_full + 6;             // [2] softmax -> MMA: P_b written (8 warps)
  uint64_t* pv_done = q_full + 8;            // MMA -> softmax: a P.V retired
  uint64_t* o_done = q_full + 9;             // MMA -> softmax: unit's last P.V retired
  uint64_t* o_free = q_full + 10;            // softmax -> MMA: epilogue read O (8 warps)
  uint64_t* qt_full = q_full + 11;           // [2] softmax -> MMA: Q in TMEM (8 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + L::kNumBars);
  float* red_max = reinterpret_cast<float*>(tmem_slot + 4);  // [2 slots][2 halves][128]
  float* red_l = red_max + 2 * 2 * 128;                       // [2 halves][128]
  float* red_sum = red_l + 2 * 128;                           // [2 slots][2 halves][128]

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    for (int s = 0; s < L::kStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 2);  // both CTAs release every slot
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(&q_full[x], 1);
      mbar_init(&q_empty[x], 8);  // the softmax warps release Q after copying it to TMEM
      mbar_init(&qt_full[x], 8);
      mbar_init(&s_full[x], 1);
      mbar_init(&p_full[x], 8);
    }
    mbar_init(pv_done, 1);
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
  cluster_sync_all();  // both CTAs' barriers initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t crank = cluster_rank();
  const bool leader = crank == 0;

  if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;" ::: "memory");
    if (warp == 8) {
      // ---------------------------------------------------- TMA producer --
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();
      uint32_t kv_it = 0;
      auto load_pos = [&](const MCursor& c, const CUtensorMap* m) {
        const uint32_t st = kv_it % L::kStages;
        mbar_wait(&kv_empty[st], ((kv_it / L::kStages) & 1) ^ 1);
        const uint32_t fl = c.flag(p);
        const int blk = c.col(p);
        uint8_t* dst = skv + st * L::kTileBytes;
        if (fl == 3u) {  // both rows hold it: one L2 read for both SMs
          mbar_arrive_expect_tx_w(&kv_full[st], L::kTileBytes);
          if (leader) {
#pragma unroll
            for (int ch = 0; ch < L::kChunks; ++ch)
              tma_mc_load_3d_w(dst + ch * L::kChunkBytes, m, &kv_full[st], ch * 64, c.h, blk * kBN,
                               pol_kv);
          }
        } else if ((fl >> crank) & 1u) {  // only this CTA's row holds it
          mbar_arrive_expect_tx_w(&kv_full[st], L::kTileBytes);
#pragma unroll
          for (int ch = 0; ch < L::kChunks; ++ch)
            tma_load_3d_w(dst + ch * L::kChunkBytes, m, &kv_full[st], ch * 64, c.h, blk * kBN,
                          pol_kv);
        } else {  // the partner's tile: keep the ring in step, no bytes
          if (lane == 0) mbar_arrive(&kv_full[st]);
          __syncwarp();
        }
        ++kv_it;
      };
      MCursor ck, cv;
      ck.start(p);
      cv.start(p);
      auto load_k = [&]() {
        if (ck.e == 0 && ck.own_cnt > 0) {  // entering a unit this CTA computes: its Q
          const Unit w = decode(p, ck.u, true);
          const int row = crank ? w.row[1] : w.row[0];
          const int qb = ck.own_ord & 1;
          mbar_wait(&q_empty[qb], ((ck.own_ord >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx_w(&q_full[qb], L::kTileBytes);
#pragma unroll
          for (int ch = 0; ch < L::kChunks; ++ch)
            tma_load_3d_w(sq + qb * L::kTileBytes + ch * L::kChunkBytes, &tq, &q_full[qb],
                          ch * 64, ck.h, row * kBM, pol_q);
        }
        load_pos(ck, &tk);
        ck.next(p, false);
      };
      if (ck.valid) load_k();
      if (ck.valid) load_k();
      while (cv.valid) {
        load_pos(cv, &tv);
        cv.next(p, false);
        if (ck.valid) load_k();
      }
    } else if (warp == 9) {
      // ----------------------------------------------------- MMA issuer ---
      // Consumes ring positions in the producer's order; own entries issue
      // S / P.V as db does, the partner's are released untouched.
      const uint32_t idesc_qk = idesc_bf16(128, 128, false, false);
      const uint32_t idesc_pv = idesc_bf16(128, D, false, true);
      const uint32_t skv_addr = smem_u32(skv);
      uint32_t kv_it = 0, gs = 0, gp = 0;
      uint32_t empty_peer[L::kStages];
#pragma unroll
      for (int s = 0; s < L::kStages; ++s) empty_peer[s] = peer_addr(&kv_empty[s], crank ^ 1u);
      auto release = [&](uint32_t st) {  // a slot this CTA does not read
        if (lane == 0) {
          mbar_arrive(&kv_empty[st]);
          attn7::arrive_cluster(empty_peer[st]);
        }
        __syncwarp();
      };
      MCursor cs, cp;
      cs.start(p);
      cp.start(p);
      auto consume_k = [&]() {
        const uint32_t st = kv_it % L::kStages;
        mbar_wait(&kv_full[st], (kv_it / L::kStages) & 1);
        const bool mine = (cs.flag(p) >> crank) & 1u;
        if (!mine) {
          release(st);
        } else {
          const int qb = cs.own_ord & 1;
          if (cs.d == 0) mbar_wait(&qt_full[qb], (cs.own_ord >> 1) & 1);
          tc_fence_after();
          const uint32_t kb = skv_addr + st * L::kTileBytes;
          const uint32_t dst = tmem + (gs & 1) * 128;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk / 4) * L::kChunkBytes + (kk % 4) * 32;
            umma_ts_w(dst, tmem + L::qt_col(qb) + kk * 8, smem_desc_sw128(kb + off, 0, 1024),
                      idesc_qk, kk > 0);
          }
          umma_commit_both_w(&kv_empty[st]);
          umma_commit_w(&s_full[gs & 1]);
          ++gs;
        }
        ++kv_it;
        cs.next(p, mine);
      };
      auto consume_v = [&]() {
        const uint32_t st = kv_it % L::kStages;
        const bool mine = (cp.flag(p) >> crank) & 1u;
        if (!mine) {
          mbar_wait(&kv_full[st], (kv_it / L::kStages) & 1);
          release(st);
        } else {
          const uint32_t b = gp & 1;
          mbar_wait(&p_full[b], (gp >> 1) & 1);
          if (cp.d == 0 && cp.own_ord > 0) mbar_wait(o_free, (cp.own_ord - 1) & 1);
          mbar_wait(&kv_full[st], (kv_it / L::kStages) & 1);
          tc_fence_after();
          const uint32_t vb = skv_addr + st * L::kTileBytes;
#pragma unroll
          for (int kk = 0; kk < kBN / 16; ++kk)
            umma_ts_w(tmem + L::kO, tmem + b * 128 + kk * 8,
                      smem_desc_sw128(vb + kk * 16 * 128, L::kChunkBytes, 1024), idesc_pv,
                      (cp.d > 0) || kk > 0);
          umma_commit_both_w(&kv_empty[st]);
          umma_commit_w(pv_done);
          if (cp.d == cp.own_cnt - 1) umma_commit_w(o_done);
          ++gp;
        }
        ++kv_it;
        cp.next(p, mine);
      };
      if (cs.valid) consume_k();
      if (cs.valid) consume_k();
      while (cp.valid) {
        consume_v();
        if (cs.valid) consume_k();
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;" ::: "memory");
    // ------------------------------------------------------- softmax -----
    const int half = warp / 4;  // key half / O column half
    const int wq = warp % 4;    // TMEM lane quarter
    const int r = wq * 32 + lane;
    const uint32_t trow = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    const float sl2 = p.scale_log2;
    const bool tr = lane == 0 && wq == 0 && half == 0;
    uint32_t g = 0;
    int ord = 0;
    // Copy the Q tile of non-empty unit `o` (shared-memory buffer o % 2,
    // 128B-swizzled by TMA) into its TMEM buffer: this thread's row, half of
    // the head dimension, bf16 pairs -- the layout P uses as an A operand.
    auto q_to_tmem = [&](int o) {
      const int qb = o & 1;
      mbar_wait(&q_full[qb], (o >> 1) & 1);
      constexpr int kUnits = D / 16;  // 16-byte units per half row
      uint32_t v[2 * kUnits * 2];
      const uint8_t* base = sq + qb * L::kTileBytes + r * 128;
#pragma unroll
      for (int t = 0; t < kUnits; ++t) {
        const int unit = half * kUnits + t;  // along the row
        const int chunk = unit / 8, uu = unit % 8;
        const uint4 x = *reinterpret_cast<const uint4*>(base + chunk * L::kChunkBytes +
                                                         ((uu ^ (r & 7)) * 16));
        v[4 * t + 0] = x.x;
        v[4 * t + 1] = x.y;
        v[4 * t + 2] = x.z;
        v[4 * t + 3] = x.w;
      }
      if constexpr (D == 128) {
        tmem_st32(trow + L::qt_col(qb) + half * 32, *reinterpret_cast<const uint32_t(*)[32]>(v));
      } else {
        tmem_st16(trow + L::qt_col(qb) + half * 16, v);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&qt_full[qb]);
        mbar_arrive(&q_empty[qb]);  // the shared-memory copy is free again
      }
    };
    // Non-empty units of this CTA, in order (the producer / MMA Cursor skips
    // empty rows the same way).
    // Pair-units of this cluster in order; this CTA computes its own row
    // (2p + rank) over its own list.  Own-nonempty units take the Q / O
    // pipeline slots (the producer and MMA count them the same way).
    auto own_of = [&](long long u, int& row, int& cnt, int& hh) {
      const Unit w = decode(p, u, false);
      row = crank ? w.row[1] : w.row[0];
      cnt = crank ? w.cnt[1] : w.cnt[0];
      hh = w.h;
    };
    auto next_nonempty = [&](long long u) -> long long {
      for (; u < p.n_units; u += cluster_count()) {
        int row, cnt, hh;
        own_of(u, row, cnt, hh);
        if (row < p.n_rows && cnt > 0) return u;
      }
      return p.n_units;
    };
    long long nx = next_nonempty(cluster_id());
    if (nx < p.n_units) q_to_tmem(0);
    for (long long u = cluster_id(); u < p.n_units; u += cluster_count()) {
      int row, n, h;
      own_of(u, row, n, h);
      if (row >= p.n_rows) continue;
      __nv_bfloat16* orow = p.out + (static_cast<long long>(row) * kBM + r) * p.out_tok_stride +
                            h * p.out_head_stride + half * (D / 2);
      if (n == 0) {  // no active block: defined output (zeros); no pipeline traffic
        uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int v = 0; v < D / 16; ++v) reinterpret_cast<uint4*>(orow)[v] = z;
        continue;
      }
      float m = -INFINITY;  // running max (raw logits), possibly stale
      float l = 0.f;        // this half's row sum
      for (int j = 0; j < n; ++j, ++g) {
        const uint32_t b = g & 1;
        const uint32_t sb = b * 128;
        const float dlt = 0.f;
        if (tr) RP_TR_NONE(0, g);
        mbar_wait(&s_full[b], (g >> 1) & 1);
        if (tr) RP_TR_NONE(1, g);
        tc_fence_after();
        uint32_t s0[32], s1[32];
        tmem_ld32(trow + sb + 64 * half, s0);
        tmem_ld32(trow + sb + 64 * half + 32, s1);
        tmem_wait_ld();
        if (tr) RP_TR_NONE(10, g);
        auto S = [&](int e) -> float { return __uint_as_float(e < 32 ? s0[e] : s1[e - 32]); };
        // Row max of the two halves, combined through shared memory (slot
        // g % 2 keeps the partner's read of this step ahead of our write two
        // steps later).
        auto exchange_max = [&](float mine) -> float {
          float* slot = red_max + b * 256;
          slot[half * 128 + r] = mine;
          asm volatile("bar.sync %0, 64;" ::"r"(1 + wq) : "memory");
          return fmaxf(slot[r], slot[128 + r]);
        };
        if (j == 0) {  // first block of the unit: the reference max comes first
          float a = S(0);
#pragma unroll
          for (int i = 1; i < 63; i += 2) a = fmaxf(a, fmaxf(S(i), S(i + 1)));
          m = exchange_max(fmaxf(a, S(63)) + dlt);
        }
        // p = 2^((s - m) * scale * log2 e) against the running reference m
        // (stale: the max of the previous blocks, so the exponentials do not
        // wait for this block's max).  32 pairs, chunked so a chunk's
        // exponentials overlap the packing of the previous one; this block's
        // max is folded in alongside and checked afterwards.
        float2 acc[2];
        uint32_t pk[32];
        float lmax = -INFINITY;
        auto exps = [&](float mref, bool track) {
          const float2 sc2 = make_float2(sl2, sl2);
          const float nb = (dlt - mref) * sl2;
          const float2 ng2 = make_float2(nb, nb);
          acc[0] = acc[1] = make_float2(0.f, 0.f);
          float2 pv_prev[16];
#pragma unroll
          for (int c = 0; c <= 2; ++c) {
            float2 pv_cur[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              if (c < 2) {
                const int e = 32 * c + 2 * i;
#ifdef RP_ABL_NOEXP
                // ablation (timing only): no exponentials -- P = raw scores
                pv_cur[i] = make_float2(S(e), S(e + 1));
                (void)sc2;
                (void)ng2;
#else
                if (track) lmax = fmaxf(lmax, fmaxf(S(e), S(e + 1)));
                const float2 xv = ffma2v(make_float2(S(e), S(e + 1)), sc2, ng2);
                if (kPolyMask & (1u << (i & 7))) {
                  pv_cur[i] = ex2_poly2(xv);
                } else {
                  pv_cur[i].x = ex2v(xv.x);
                  pv_cur[i].y = ex2v(xv.y);
                }
#endif
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
        exps(m, false);
        // rescale guard from the exchanged row sum (see attn_sm100_db.cu)
        const float2 at0 = fadd2(acc[0], acc[1]);
        float tot = 0.f;
        if (j > 0) {
          float* slot = red_sum + b * 256;
          slot[half * 128 + r] = at0.x + at0.y;
          asm volatile("bar.sync %0, 64;" ::"r"(1 + wq) : "memory");
          tot = slot[r] + slot[128 + r];
        }
        if (j > 0 && __any_sync(0xFFFFFFFFu, !(tot <= 256.0f))) {
          float a = S(0);
#pragma unroll
          for (int i = 1; i < 63; i += 2) a = fmaxf(a, fmaxf(S(i), S(i + 1)));
          lmax = fmaxf(a, S(63));
          const float mx = exchange_max(lmax + dlt);
          const bool need = (mx - m) * sl2 > 8.0f;
          if (__any_sync(0xFFFFFFFFu, need)) {
            const float alpha = need ? ex2((m - mx) * sl2) : 1.0f;
            if (need) {
              m = mx;
              l *= alpha;
            }
            // O must hold P(g-1).V(g-1) before it is rescaled
            mbar_wait(pv_done, (g - 1) & 1);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < D / 64; ++c) {
              uint32_t o[32];
              const uint32_t oc = trow + L::kO + half * (D / 2) + c * 32;
              tmem_ld32(oc, o);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
              tmem_st32(oc, o);
            }
            exps(m, false);
          }
        }
        if (tr) RP_TR_NONE(11, g);
        const float2 at = fadd2(acc[0], acc[1]);
        l += at.x + at.y;
        tmem_st32(trow + sb + 32 * half, pk);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[b]);
        if (tr) RP_TR_NONE(2, g);
      }
      // the next unit's Q goes to TMEM before this unit's epilogue: the MMA
      // warp issues the next unit's first S ahead of this unit's last P.V
      if (next_nonempty(u + cluster_count()) < p.n_units) q_to_tmem(ord + 1);
      // epilogue: wait for the unit's last P.V, combine the halves' sums,
      // O / l -> bf16 -> global (this half's D/2 columns)
      red_l[half * 128 + r] = l;
      mbar_wait(o_done, ord & 1);
      tc_fence_after();
      asm volatile("bar.sync %0, 64;" ::"r"(1 + wq) : "memory");
      const float inv = 1.0f / (red_l[r] + red_l[128 + r]);
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        uint32_t o[32];
        tmem_ld32(trow + L::kO + half * (D / 2) + c * 32, o);
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
      // red_l is rewritten next unit only after this barrier pair's next
      // use, which both warps reach after reading it here
      asm volatile("bar.sync %0, 64;" ::"r"(1 + wq) : "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(o_free);
      ++ord;
    }
  }

  tc_fence_before();
  cluster_sync_all();  // no CTA exits while its partner may still arrive remotely
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace attn8
}  // namespace rp
