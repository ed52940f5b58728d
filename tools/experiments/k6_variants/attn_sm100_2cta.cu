// K6 (v7, "cta2"): block-sparse flash-attention forward on CTA PAIRS
// (tcgen05.mma.cta_group::2, M = 256), bf16 in / fp32 softmax, sm_100a,
// head_dim 128.
//
// Same semantics as attn_sm100_db.cu (attention.cpp:50-121, exact mask,
// zero-padded keys attended when their block is active).
//
// Why.  Timing ablations of db (tools/build_variant.sh, Wan shape): without
// exponentials 64 % of peak, without exponentials AND K/V reloads 80 %.  The
// reloads cost shared-memory bandwidth: at M = 128 the tensor core reads its
// B operand (K for S, V for P.V) at 64 B/clk and TMA writes the next tiles
// at ~59 B/clk, against ~128 B/clk per SM.  A CTA pair on one TPC issues
// M = 256 MMAs in which each SM holds and reads only HALF of B (keys
// 64c..64c+63 of K, head-dim columns 64c..64c+63 of V), so both the reads and
// the TMA writes per SM halve (and L2 -> SM traffic with them).
//
// Pairing.  The pair owns block rows (2p, 2p+1) of one head: CTA c computes
// row 2p+c (its Q tile, its TMEM S / P / O), both walk the UNION of the two
// rows' block lists (rp's pair lists), and a CTA whose row does not hold a
// union entry writes P = 0 for it (exact: the block contributes nothing;
// Wan config-3 mask: 86 % of the union work is useful).
//
// Per CTA: TMEM S0 | S1 | O | QT0 | QT1 exactly as db (Q copied into TMEM by
// the softmax warps, S double-buffered); the leader (cluster rank 0) issues
// every MMA; commits are multicast to both CTAs' barriers; the peer's
// softmax warps arrive on the leader's p_full / qt_full / o_free remotely;
// both CTAs' producers TMA their halves with the 2-SM form, which completes
// on the leader's kv_full.
//
//   warps 0-7 softmax / epilogue (db's two-halves-per-row split)
//   warp 8 TMA producer, warp 9 MMA issuer (leader) / TMEM owner (both)
#include "common.cuh"

namespace rp {
namespace attn7 {

using attn3::decode;
using attn3::Params;
using attn3::Unit;

constexpr int kThreads = 384;
constexpr int kBM = 128;
constexpr int kD = 128;
constexpr uint32_t kPolyMask = 0x01u;

struct Layout {
  static constexpr int kTileBytes = 128 * kD * 2;  // Q tile
  static constexpr int kHalfBytes = 16384;         // K half (2 x 8 KB chunks) or V half
  static constexpr int kKChunk = 64 * 128;         // 64 key rows x 128 B
  static constexpr int kVChunk = 128 * 128;        // 128 key rows x 128 B (64 d)
  static constexpr int kStages = 8;
  static constexpr int kSmemData = 2 * kTileBytes + kStages * kHalfBytes;
  static constexpr int kNumBars = 2 * kStages + 16;
  static constexpr int kRedBytes = (2 * 2 * 128 + 2 * 128 + 2 * 2 * 128) * 4;
  static constexpr int kSmemBytes = kSmemData + kNumBars * 8 + 16 + kRedBytes + 1024;
  static_assert(kSmemBytes <= 232448, "exceeds the 227 KB opt-in shared memory");
  static constexpr uint32_t kO = 256;
  RP_HD static uint32_t qt_col(int b) { return 384u + (b ? 64u : 0u); }
};

// ---- cluster / 2-SM primitives --------------------------------------------
RP_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
RP_DEV uint32_t cluster_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
RP_DEV uint32_t cluster_count() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
RP_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// shared::cluster address of `bar` in the leader CTA (rank 0)
RP_DEV uint32_t leader_addr(uint64_t* bar) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(a) : "r"(smem_u32(bar)));
  return a;
}
// Relaxed: nothing in generic memory flows between the two CTAs (P and Q go
// through TMEM, ordered by tcgen05.wait::st + tcgen05.fence), and a
// release.cluster arrive costs a GPU-scope MEMBAR per call (ncu: the top
// stall of the first version).
RP_DEV void arrive_cluster(uint32_t addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(addr)
               : "memory");
}
// Barriers that receive the peer CTA's (relaxed) arrivals are waited on with
// the plain CTA-scope try_wait: any cluster-scope try_wait (even .relaxed)
// compiles to an L1 invalidate (CCTL.IVALL) after every successful poll.
RP_DEV void mbar_wait_cl(uint64_t* bar, uint32_t parity) { mbar_wait(bar, parity); }
RP_DEV void umma2_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// commit to the barrier at this offset in both CTAs of the pair
RP_DEV void umma2_commit_both_w(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b16 m;\n\t"
      "mov.b16 m, 3;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], m;\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
// 2-SM TMA: this CTA's half, completing on the leader's barrier
RP_DEV void tma2_load_3d_w(void* smem_dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1,
                           int c2, uint64_t policy) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::"
      "bytes.L2::cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6;\n\t}" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1),
      "r"(c2), "l"(policy)
      : "memory");
}
RP_DEV void tmem_alloc2_512(uint32_t* smem_dst) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                   smem_u32(smem_dst))
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
RP_DEV void tmem_dealloc2_512(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(taddr)
               : "memory");
}

// Walks the pair-units of this cluster and their union entries (warp-uniform).
struct PCursor {
  long long u;
  int ord, e, n, beg, h;
  bool valid;
  RP_DEV void seek(const Params& p) {
    valid = false;
    for (; u < p.n_units; u += cluster_count()) {
      const Unit w = decode(p, u, true);
      if (w.n > 0) {
        n = w.n;
        beg = w.beg;
        h = w.h;
        e = 0;
        valid = true;
        return;
      }
    }
  }
  RP_DEV void start(const Params& p) {
    u = cluster_id();
    ord = 0;
    seek(p);
  }
  RP_DEV void next(const Params& p) {
    if (++e < n) return;
    u += cluster_count();
    ++ord;
    seek(p);
  }
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    bsfa_fwd_2cta_kernel(const __grid_constant__ CUtensorMap tq,
                         const __grid_constant__ CUtensorMap tk64,
                         const __grid_constant__ CUtensorMap tv, const Params p) {
  using L = Layout;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sq = smem;                       // [2][Q tile]
  uint8_t* skv = smem + 2 * L::kTileBytes;  // [kStages][half tile]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kSmemData);
  uint64_t* kv_full = bars;                  // leader: both halves landed
  uint64_t* kv_empty = bars + L::kStages;    // both: stage consumed (multicast commit)
  uint64_t* q_full = bars + 2 * L::kStages;  // [2] local Q TMA
  uint64_t* q_empty = q_full + 2;            // [2] local: Q copied to TMEM (8 warps)
  uint64_t* qt_full = q_full + 4;            // [2] leader: both CTAs' Q in TMEM (16 warps)
  uint64_t* s_full = q_full + 6;             // [2] both (multicast)
  uint64_t* p_full = q_full + 8;             // [2] leader: both CTAs' P written (16 warps)
  uint64_t* pv_done = q_full + 10;           // both (multicast)
  uint64_t* o_done = q_full + 11;            // both (multicast)
  uint64_t* o_free = q_full + 12;            // leader: both epilogues read O (16 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + L::kNumBars);
  float* red_max = reinterpret_cast<float*>(tmem_slot + 4);  // [2 slots][2 halves][128]
  float* red_l = red_max + 2 * 2 * 128;                       // [2 halves][128]
  float* red_sum = red_l + 2 * 128;                           // [2 slots][2 halves][128]

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t crank = cluster_rank();
  const bool leader = crank == 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < L::kStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(&q_full[x], 1);
      mbar_init(&q_empty[x], 8);
      mbar_init(&qt_full[x], 16);
      mbar_init(&s_full[x], 1);
      mbar_init(&p_full[x], 16);
    }
    mbar_init(pv_done, 1);
    mbar_init(o_done, 1);
    mbar_init(o_free, 16);
    fence_barrier_init();
  }
  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&tq);
    tma_prefetch_desc(&tk64);
    tma_prefetch_desc(&tv);
  }
  if (warp == 9) tmem_alloc2_512(tmem_slot);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;" ::: "memory");
    if (warp == 8) {
      // ---------------------------------------------------- TMA producer --
      // Both CTAs: own Q tile (local barrier), own halves of K / V (2-SM
      // form, leader's barrier).  Ring order = MMA order: K(0), K(1), V(g), K(g+2).
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();
      uint32_t kv_it = 0;
      auto load_half = [&](bool is_v, int h, int blk) {
        const uint32_t st = kv_it % L::kStages;
        mbar_wait(&kv_empty[st], ((kv_it / L::kStages) & 1) ^ 1);
        if (leader) mbar_arrive_expect_tx_w(&kv_full[st], 2 * L::kHalfBytes);
        uint8_t* dst = skv + st * L::kHalfBytes;
        if (is_v) {
          tma2_load_3d_w(dst, &tv, &kv_full[st], 64 * static_cast<int>(crank), h, blk * 128,
                         pol_kv);
        } else {
#pragma unroll
          for (int c = 0; c < 2; ++c)
            tma2_load_3d_w(dst + c * L::kKChunk, &tk64, &kv_full[st], c * 64, h,
                           blk * 128 + 64 * static_cast<int>(crank), pol_kv);
        }
        ++kv_it;
      };
      PCursor ck, cv;
      ck.start(p);
      cv.start(p);
      auto load_k = [&]() {
        if (ck.e == 0) {  // entering a unit: this CTA's Q tile first
          const Unit w = decode(p, ck.u, true);
          const int row = crank ? w.row[1] : w.row[0];
          const int qb = ck.ord & 1;
          mbar_wait(&q_empty[qb], ((ck.ord >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx_w(&q_full[qb], L::kTileBytes);
#pragma unroll
          for (int c = 0; c < 2; ++c)
            tma_load_3d_w(sq + qb * L::kTileBytes + c * (128 * 128), &tq, &q_full[qb], c * 64,
                          ck.h, row * kBM, pol_q);
        }
        load_half(false, ck.h, shfl0(__ldg(p.pcol + ck.beg + ck.e)));
        ck.next(p);
      };
      if (ck.valid) load_k();
      if (ck.valid) load_k();
      while (cv.valid) {
        load_half(true, cv.h, shfl0(__ldg(p.pcol + cv.beg + cv.e)));
        cv.next(p);
        if (ck.valid) load_k();
      }
    } else if (warp == 9 && leader) {
      // ------------------------------------------- MMA issuer (leader) ----
      const uint32_t idesc_qk = idesc_bf16(256, 128, false, false);
      const uint32_t idesc_pv = idesc_bf16(256, kD, false, true);
      const uint32_t skv_addr = smem_u32(skv);
      uint32_t kv_it = 0, gs = 0, gp = 0;
      PCursor cs, cp;
      cs.start(p);
      cp.start(p);
      auto issue_s = [&]() {
        const int qb = cs.ord & 1;
        if (cs.e == 0) mbar_wait_cl(&qt_full[qb], (cs.ord >> 1) & 1);
        const uint32_t st = kv_it % L::kStages;
        mbar_wait_cl(&kv_full[st], (kv_it / L::kStages) & 1);
        tc_fence_after();
        const uint32_t kb = skv_addr + st * L::kHalfBytes;
        const uint32_t dst = tmem + (gs & 1) * 128;
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const uint32_t off = (kk / 4) * L::kKChunk + (kk % 4) * 32;
          umma2_ts_w(dst, tmem + L::qt_col(qb) + kk * 8, smem_desc_sw128(kb + off, 0, 1024),
                     idesc_qk, kk > 0);
        }
        umma2_commit_both_w(&kv_empty[st]);
        umma2_commit_both_w(&s_full[gs & 1]);
        ++kv_it;
        ++gs;
        cs.next(p);
      };
      if (cs.valid) issue_s();
      if (cs.valid) issue_s();
      while (cp.valid) {
        const uint32_t b = gp & 1;
        mbar_wait_cl(&p_full[b], (gp >> 1) & 1);
        if (cp.e == 0 && cp.ord > 0) mbar_wait_cl(o_free, (cp.ord - 1) & 1);
        const uint32_t st = kv_it % L::kStages;
        mbar_wait_cl(&kv_full[st], (kv_it / L::kStages) & 1);
        tc_fence_after();
        const uint32_t vb = skv_addr + st * L::kHalfBytes;
#pragma unroll
        for (int kk = 0; kk < 128 / 16; ++kk)
          umma2_ts_w(tmem + L::kO, tmem + b * 128 + kk * 8,
                     smem_desc_sw128(vb + kk * 16 * 128, L::kVChunk, 1024), idesc_pv,
                     (cp.e > 0) || kk > 0);
        umma2_commit_both_w(&kv_empty[st]);
        umma2_commit_both_w(pv_done);
        if (cp.e == cp.n - 1) umma2_commit_both_w(o_done);
        ++kv_it;
        ++gp;
        cp.next(p);
        if (cs.valid) issue_s();
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;" ::: "memory");
    // ------------------------------------------------------- softmax -----
    const int half = warp / 4;
    const int wq = warp % 4;
    const int r = wq * 32 + lane;
    const uint32_t trow = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    const float sl2 = p.scale_log2;
    // arrivals that gate the leader's MMA warp
    const uint32_t pf_addr[2] = {leader_addr(&p_full[0]), leader_addr(&p_full[1])};
    const uint32_t qt_addr[2] = {leader_addr(&qt_full[0]), leader_addr(&qt_full[1])};
    const uint32_t of_addr = leader_addr(o_free);
    uint32_t g = 0;
    int ord = 0;
    auto q_to_tmem = [&](int o) {
      const int qb = o & 1;
      mbar_wait(&q_full[qb], (o >> 1) & 1);
      constexpr int kUnits = kD / 16;
      uint32_t v[2 * kUnits * 2];
      const uint8_t* base = sq + qb * L::kTileBytes + r * 128;
#pragma unroll
      for (int t = 0; t < kUnits; ++t) {
        const int unit = half * kUnits + t;
        const int chunk = unit / 8, uu = unit % 8;
        const uint4 x = *reinterpret_cast<const uint4*>(base + chunk * (128 * 128) +
                                                         ((uu ^ (r & 7)) * 16));
        v[4 * t + 0] = x.x;
        v[4 * t + 1] = x.y;
        v[4 * t + 2] = x.z;
        v[4 * t + 3] = x.w;
      }
      tmem_st32(trow + L::qt_col(qb) + half * 32, *reinterpret_cast<const uint32_t(*)[32]>(v));
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        arrive_cluster(qt_addr[qb]);
        mbar_arrive(&q_empty[qb]);
      }
    };
    auto next_nonempty = [&](long long u) -> long long {
      for (; u < p.n_units; u += cluster_count()) {
        const Unit w = decode(p, u, false);
        if (w.n > 0) return u;
      }
      return p.n_units;
    };
    if (next_nonempty(cluster_id()) < p.n_units) q_to_tmem(0);
    for (long long u = cluster_id(); u < p.n_units; u += cluster_count()) {
      const Unit w = decode(p, u, false);
      const int my_row = crank ? w.row[1] : w.row[0];
      const int my_cnt = crank ? w.cnt[1] : w.cnt[0];
      const bool my_valid = my_row < p.n_rows;
      __nv_bfloat16* orow = p.out + (static_cast<long long>(my_row) * kBM + r) * p.out_tok_stride +
                            w.h * p.out_head_stride + half * (kD / 2);
      if (w.n == 0) {  // neither row holds a block: zeros, no pipeline traffic
        if (my_valid) {
          const uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
          for (int v = 0; v < kD / 16; ++v) reinterpret_cast<uint4*>(orow)[v] = z;
        }
        continue;
      }
      const uint8_t* flags = p.pflag + w.beg;
      float m = -INFINITY;
      float l = 0.f;
      bool first = true;
      for (int e = 0; e < w.n; ++e, ++g) {
        const uint32_t b = g & 1;
        const uint32_t sb = b * 128;
        const bool member = (__ldg(flags + e) >> crank) & 1;
        mbar_wait(&s_full[b], (g >> 1) & 1);
        tc_fence_after();
        uint32_t pk[32];
        if (member) {
          uint32_t s0[32], s1[32];
          tmem_ld32(trow + sb + 64 * half, s0);
          tmem_ld32(trow + sb + 64 * half + 32, s1);
          tmem_wait_ld();
          auto S = [&](int i) -> float { return __uint_as_float(i < 32 ? s0[i] : s1[i - 32]); };
          auto exchange_max = [&](float mine) -> float {
            float* slot = red_max + b * 256;
            slot[half * 128 + r] = mine;
            asm volatile("bar.sync %0, 64;" ::"r"(1 + wq) : "memory");
            return fmaxf(slot[r], slot[128 + r]);
          };
          if (first) {
            float a = S(0);
#pragma unroll
            for (int i = 1; i < 63; i += 2) a = fmaxf(a, fmaxf(S(i), S(i + 1)));
            m = exchange_max(fmaxf(a, S(63)));
          }
          float2 acc[2];
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
                  const int ei = 32 * c + 2 * i;
                  if (track) lmax = fmaxf(lmax, fmaxf(S(ei), S(ei + 1)));
                  const float2 xv = ffma2v(make_float2(S(ei), S(ei + 1)), sc2, ng2);
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
          exps(m, false);
          // rescale guard from the exchanged row sum (see attn_sm100_db.cu)
          const float2 at0 = fadd2(acc[0], acc[1]);
          float tot = 0.f;
          if (!first) {
            float* slot = red_sum + b * 256;
            slot[half * 128 + r] = at0.x + at0.y;
            asm volatile("bar.sync %0, 64;" ::"r"(1 + wq) : "memory");
            tot = slot[r] + slot[128 + r];
          }
          if (!first && __any_sync(0xFFFFFFFFu, !(tot <= 256.0f))) {
            float a = S(0);
#pragma unroll
            for (int i = 1; i < 63; i += 2) a = fmaxf(a, fmaxf(S(i), S(i + 1)));
            lmax = fmaxf(a, S(63));
            const float mx = exchange_max(lmax);
            const bool need = (mx - m) * sl2 > 8.0f;
            if (__any_sync(0xFFFFFFFFu, need)) {
              const float alpha = need ? ex2((m - mx) * sl2) : 1.0f;
              if (need) {
                m = mx;
                l *= alpha;
              }
              mbar_wait(pv_done, (g - 1) & 1);  // O holds P(g-1).V before the rescale
              tc_fence_after();
#pragma unroll
              for (int c = 0; c < kD / 64; ++c) {
                uint32_t o[32];
                const uint32_t oc = trow + L::kO + half * (kD / 2) + c * 32;
                tmem_ld32(oc, o);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
                tmem_st32(oc, o);
              }
              exps(m, false);
            }
          }
          const float2 at = fadd2(acc[0], acc[1]);
          l += at.x + at.y;
          first = false;
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) pk[i] = 0u;  // block not in this row's list
        }
        tmem_st32(trow + sb + 32 * half, pk);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_cluster(pf_addr[b]);
      }
      if (next_nonempty(u + cluster_count()) < p.n_units) q_to_tmem(ord + 1);
      red_l[half * 128 + r] = l;
      mbar_wait(o_done, ord & 1);
      tc_fence_after();
      asm volatile("bar.sync %0, 64;" ::"r"(1 + wq) : "memory");
      const float lt = red_l[r] + red_l[128 + r];
      const float inv = lt > 0.f ? 1.0f / lt : 0.f;  // a row with no own block: zeros
#pragma unroll
      for (int c = 0; c < kD / 64; ++c) {
        uint32_t o[32];
        tmem_ld32(trow + L::kO + half * (kD / 2) + c * 32, o);
        tmem_wait_ld();
        if (my_valid) {
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
      }
      (void)my_cnt;
      tc_fence_before();
      asm volatile("bar.sync %0, 64;" ::"r"(1 + wq) : "memory");
      __syncwarp();
      if (lane == 0) arrive_cluster(of_addr);
      ++ord;
    }
  }

  tc_fence_before();
  cluster_sync_all();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc2_512(tmem);
  }
}

}  // namespace attn7
}  // namespace rp
