// K6 "ppc": block-sparse flash-attention forward on CTA PAIRS with two
// ping-ponged query tiles per CTA, bf16 in / fp32 softmax, sm_100a, d = 128.
//
// Same semantics as attn_sm100_db.cu (attention.cpp:50-121, exact mask,
// zero-padded keys attended when their block is active, a row without an
// active block is the reference's domain_error: zeros + err_flag).
//
// Why.  The per-step softmax of one 128 x 128 tile (~1.8 k clk) is longer
// than its MMAs (1024 clk at M = 128), so a single tile per SM leaves the
// tensor pipe ~45 % idle (db).  Two independent tiles per CTA ping-pong on
// the tensor core (FA4's structure, measured here as `pp`), but with Q as a
// shared-memory operand an M = 128 CTA is then shared-memory bound (Q 32 KB +
// K 32 KB + V 32 KB reads + 64 KB of TMA writes per step).  A CTA pair on one
// TPC issues M = 256 MMAs (tcgen05 cta_group::2) in which each SM holds and
// reads only HALF of K and V, so a step's shared-memory traffic per SM falls
// from 160 KB to 96 KB and the ping-pong is no longer fed late.
//
// Pairing.  Tile t of the cluster owns a pair of block rows (2p, 2p+1) of
// one head: CTA c computes row 2p + c (its Q tile, its TMEM S / P / O), both
// walk the UNION of the two rows' block lists (union_fill_kernel), and a CTA
// whose row does not hold a union entry writes P = 0 for it (exact: the block
// contributes nothing).  Wan config-3 mask: 85.8 % of the union is useful.
//
// Per CTA, TMEM (512 columns, allocated for the pair): S_0 0-127, S_1
// 128-255, O_0 256-383, O_1 384-511; P_t (bf16) overwrites the first 64
// columns of S_t and is the A operand of P_t V.  The leader (cluster rank 0)
// issues every MMA; commits are multicast to both CTAs' barriers; both
// producers TMA their halves (and their Q tiles) with the 2-SM form, which
// completes on the leader's barriers; both CTAs' softmax warps arrive on the
// leader's p_full.
//
//   warps 0-3 softmax + epilogue of tile 0, warps 4-7 of tile 1 (thread = row)
//   warp 8 TMA producer (both CTAs), warp 9 MMA issuer (leader) / TMEM owner
//   warps 10-11 idle (setmaxnreg donors)
#include "common.cuh"

namespace rp {
namespace attn10 {

constexpr int kThreads = 384;
constexpr int kBM = 128;
constexpr int kD = 128;
// Pairs (of 16 per 32-key chunk) whose exp2 runs as a polynomial on the FMA pipe.
#ifndef RP_PPC_POLY
#define RP_PPC_POLY 0x0000u
#endif
constexpr uint32_t kPolyMask = RP_PPC_POLY;

struct Layout {
  static constexpr int kTileBytes = 128 * kD * 2;  // Q tile (this CTA's 128 rows)
  static constexpr int kQChunk = 128 * 128;        // 128 rows x 128 B (64 d)
  static constexpr int kHalfBytes = 16384;         // K half or V half
  static constexpr int kKChunk = 64 * 128;         // 64 key rows x 128 B (64 d)
  static constexpr int kVChunk = 128 * 128;        // 128 key rows x 128 B (64 d)
#ifdef RP_PPC_STAGES
  static constexpr int kStages = RP_PPC_STAGES;
#else
  static constexpr int kStages = 9;
#endif
  static constexpr int kSmemData = 2 * kTileBytes + kStages * kHalfBytes;
  static constexpr int kNumBars = 2 * kStages + 10;
  static constexpr int kSmemBytes = kSmemData + kNumBars * 8 + 16 + 1024;
  static_assert(kSmemBytes <= 232448, "exceeds the 227 KB opt-in shared memory");
  RP_HD static uint32_t s_col(int t) { return static_cast<uint32_t>(t) * 128u; }
  RP_HD static uint32_t o_col(int t) { return 256u + static_cast<uint32_t>(t) * 128u; }
};

struct Params {
  const int32_t* prow_ptr;  // per row pair: union list offsets
  const int32_t* ucol;      // per union entry: block column
  const uint8_t* uflag;     // bit 0: row 2p holds it, bit 1: row 2p+1 holds it
  int n_rows;               // S_b
  int n_pairs;              // ceil(S_b / 2)
  int heads;
  long long n_units;        // heads * n_pairs, head-major
  __nv_bfloat16* out;
  long long out_tok_stride;
  long long out_head_stride;
  float scale_log2;
  int* err_flag;            // may be null
};

// Union lists of the row pairs (2p, 2p+1): ascending block columns, each with
// the membership bits of the two rows.
__global__ void union_count_kernel(const int32_t* __restrict__ row_ptr,
                                   const int32_t* __restrict__ col, int n_rows, int n_pairs,
                                   int32_t* __restrict__ counts) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pairs) return;
  const int a = 2 * p, b = 2 * p + 1;
  int i = row_ptr[a], ie = row_ptr[a + 1];
  int j = b < n_rows ? row_ptr[b] : 0, je = b < n_rows ? row_ptr[b + 1] : 0;
  int n = 0;
  while (i < ie || j < je) {
    const int ca = i < ie ? col[i] : 0x7FFFFFFF, cb = j < je ? col[j] : 0x7FFFFFFF;
    ++n;
    i += ca <= cb;
    j += cb <= ca;
  }
  counts[p] = n;
}
__global__ void union_fill_kernel(const int32_t* __restrict__ row_ptr,
                                  const int32_t* __restrict__ col, int n_rows, int n_pairs,
                                  const int32_t* __restrict__ prow_ptr, int32_t* __restrict__ ucol,
                                  uint8_t* __restrict__ uflag) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pairs) return;
  const int a = 2 * p, b = 2 * p + 1;
  int i = row_ptr[a], ie = row_ptr[a + 1];
  int j = b < n_rows ? row_ptr[b] : 0, je = b < n_rows ? row_ptr[b + 1] : 0;
  int o = prow_ptr[p];
  while (i < ie || j < je) {
    const int ca = i < ie ? col[i] : 0x7FFFFFFF, cb = j < je ? col[j] : 0x7FFFFFFF;
    ucol[o] = ca < cb ? ca : cb;
    uflag[o] = static_cast<uint8_t>((ca <= cb ? 1 : 0) | (cb <= ca ? 2 : 0));
    ++o;
    i += ca <= cb;
    j += cb <= ca;
  }
}

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
// Relaxed: P goes through TMEM, ordered by tcgen05.wait::st + tcgen05.fence.
RP_DEV void arrive_cluster(uint32_t addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(addr)
               : "memory");
}
RP_DEV void umma2_ss_w(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
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
// 2-SM TMA: this CTA's data, completing on the leader's barrier
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

RP_DEV float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// One tile's stream of non-empty pair units and their union entries
// (warp-uniform: every lookup is broadcast from lane 0).
struct Cursor {
  long long u;
  int ord;  // ordinal among this tile's non-empty units
  int j, n, beg, h, pr;
  bool valid;
  int cb = 0, nb = 0, cbase = -1;

  RP_DEV void seek(const Params& p) {
    valid = false;
    const long long stride = 2ll * cluster_count();
    for (; u < p.n_units; u += stride) {
      const int hh = static_cast<int>(u / p.n_pairs);
      const int q = static_cast<int>(u - static_cast<long long>(hh) * p.n_pairs);
      const int b = shfl0(__ldg(p.prow_ptr + q));
      const int e = shfl0(__ldg(p.prow_ptr + q + 1));
      if (e > b) {
        h = hh;
        pr = q;
        beg = b;
        n = e - b;
        j = 0;
        cbase = -1;
        valid = true;
        return;
      }
    }
  }
  RP_DEV void start(const Params& p, int t) {
    u = 2ll * cluster_id() + t;
    ord = 0;
    seek(p);
  }
  RP_DEV void next(const Params& p) {
    if (++j < n) return;
    u += 2ll * cluster_count();
    ++ord;
    seek(p);
  }
  // block column of entry j: 32 loaded per warp at a time, next 32 prefetched
  RP_DEV int col(const Params& p) {
    const int base = j & ~31;
    if (base != cbase) {
      const int lane = threadIdx.x & 31;
      if (cbase >= 0 && base == cbase + 32)
        cb = nb;
      else
        cb = base + lane < n ? __ldg(p.ucol + beg + base + lane) : 0;
      nb = base + 32 + lane < n ? __ldg(p.ucol + beg + base + 32 + lane) : 0;
      cbase = base;
    }
    return __shfl_sync(0xFFFFFFFFu, cb, j & 31);
  }
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    bsfa_fwd_ppc_kernel(const __grid_constant__ CUtensorMap tq,
                        const __grid_constant__ CUtensorMap tk64,
                        const __grid_constant__ CUtensorMap tv, const Params p) {
  using L = Layout;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sq = smem;                       // [2 tiles][Q tile]
  uint8_t* skv = smem + 2 * L::kTileBytes;  // [kStages][half tile]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kSmemData);
  uint64_t* kv_full = bars;                  // leader: both halves landed
  uint64_t* kv_empty = bars + L::kStages;    // both: stage consumed (multicast commit)
  uint64_t* q_full = bars + 2 * L::kStages;  // [2] leader: both CTAs' Q tiles landed
  uint64_t* q_empty = q_full + 2;            // [2] both: the unit's last S retired
  uint64_t* s_full = q_full + 4;             // [2] both (multicast)
  uint64_t* p_full = q_full + 6;             // [2] leader: both CTAs' P written (8 warps)
  uint64_t* o_done = q_full + 8;             // [2] both: the unit's last P.V retired
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + L::kNumBars);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t crank = cluster_rank();
  const bool leader = crank == 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < L::kStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&q_full[t], 1);
      mbar_init(&q_empty[t], 1);
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], 8);
      mbar_init(&o_done[t], 1);
    }
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
      // Both CTAs: own Q tiles and own halves of K / V (2-SM form, leader's
      // barriers).  Ring order = MMA order: K_0(0), K_1(0), then per tile t
      // in turn V_t(j), K_t(j+1).
      const uint64_t pol_q = policy_evict_first();
#ifdef RP_PPC_KV_NORMAL
      const uint64_t pol_kv = policy_evict_normal();
#else
      const uint64_t pol_kv = policy_evict_last();
#endif
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
      Cursor ck[2], cv[2];
      auto load_k = [&](int t) {
        Cursor& c = ck[t];
        if (c.j == 0) {  // entering a unit: this CTA's Q tile first
          mbar_wait(&q_empty[t], (c.ord & 1) ^ 1);
          if (leader) mbar_arrive_expect_tx_w(&q_full[t], 2 * L::kTileBytes);
          const int row = 2 * c.pr + static_cast<int>(crank);
#pragma unroll
          for (int ch = 0; ch < 2; ++ch)
            tma2_load_3d_w(sq + t * L::kTileBytes + ch * L::kQChunk, &tq, &q_full[t], ch * 64,
                           c.h, row * kBM, pol_q);
        }
        load_half(false, c.h, c.col(p));
        c.next(p);
      };
      for (int t = 0; t < 2; ++t) {
        ck[t].start(p, t);
        cv[t].start(p, t);
      }
      for (int t = 0; t < 2; ++t)
        if (ck[t].valid) load_k(t);
      while (cv[0].valid || cv[1].valid) {
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          if (!cv[t].valid) continue;
          load_half(true, cv[t].h, cv[t].col(p));
          cv[t].next(p);
          if (ck[t].valid) load_k(t);
        }
      }
    } else if (warp == 9 && leader) {
      // ------------------------------------------- MMA issuer (leader) ----
      const uint32_t idesc_qk = idesc_bf16(256, 128, false, false);
      const uint32_t idesc_pv = idesc_bf16(256, kD, false, true);
      const uint32_t skv_addr = smem_u32(skv);
      const uint32_t sq_addr = smem_u32(sq);
      uint32_t kv_it = 0;
      uint32_t gp[2] = {0u, 0u};
      Cursor cs[2], cp[2];
      // S_t = Q_t K^T over the pair (M = 256): Q from each CTA's shared
      // memory, K as each CTA's 64-key half.
      auto issue_s = [&](int t) {
        Cursor& c = cs[t];
        if (c.j == 0) mbar_wait(&q_full[t], c.ord & 1);
        const uint32_t st = kv_it % L::kStages;
        mbar_wait(&kv_full[st], (kv_it / L::kStages) & 1);
        tc_fence_after();
        const uint32_t kb = skv_addr + st * L::kHalfBytes;
        const uint32_t qa = sq_addr + t * L::kTileBytes;
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk)
          umma2_ss_w(tmem + L::s_col(t),
                     smem_desc_sw128(qa + (kk / 4) * L::kQChunk + (kk % 4) * 32, 0, 1024),
                     smem_desc_sw128(kb + (kk / 4) * L::kKChunk + (kk % 4) * 32, 0, 1024),
                     idesc_qk, kk > 0);
        umma2_commit_both_w(&kv_empty[st]);
        if (c.j == c.n - 1) umma2_commit_both_w(&q_empty[t]);
        umma2_commit_both_w(&s_full[t]);
        ++kv_it;
        c.next(p);
      };
      for (int t = 0; t < 2; ++t) {
        cs[t].start(p, t);
        cp[t].start(p, t);
      }
      for (int t = 0; t < 2; ++t)
        if (cs[t].valid) issue_s(t);
      while (cp[0].valid || cp[1].valid) {
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          if (!cp[t].valid) continue;
          // O_t (+)= P_t V over the pair: P from each CTA's TMEM, V as each
          // CTA's 64-column half
          mbar_wait(&p_full[t], gp[t] & 1);
          tc_fence_after();
          const uint32_t st = kv_it % L::kStages;
          mbar_wait(&kv_full[st], (kv_it / L::kStages) & 1);
          tc_fence_after();
          const uint32_t vb = skv_addr + st * L::kHalfBytes;
#pragma unroll
          for (int kk = 0; kk < 128 / 16; ++kk)
            umma2_ts_w(tmem + L::o_col(t), tmem + L::s_col(t) + kk * 8,
                       smem_desc_sw128(vb + kk * 16 * 128, L::kVChunk, 1024), idesc_pv,
                       (cp[t].j > 0) || kk > 0);
          umma2_commit_both_w(&kv_empty[st]);
          if (cp[t].j == cp[t].n - 1) umma2_commit_both_w(&o_done[t]);
          ++kv_it;
          ++gp[t];
          cp[t].next(p);
          // S_t(j+1) into the buffer P_t(j) occupies: the tensor pipe runs the
          // issuing thread's MMAs in order, so P.V has read P before S lands
          if (cs[t].valid) issue_s(t);
        }
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;" ::: "memory");
    // ------------------------------------------------------- softmax -----
    const int t = warp >> 2;  // tile
    const int wq = warp & 3;  // TMEM lane quarter (= SM sub-partition)
    const int r = wq * 32 + lane;
    const uint32_t trow = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    const uint32_t scol = L::s_col(t), ocol = L::o_col(t);
    const float sl2 = p.scale_log2;
    const uint32_t pf_addr = leader_addr(&p_full[t]);
    uint32_t g = 0;
    int ord = 0;
    for (long long u = 2ll * cluster_id() + t; u < p.n_units; u += 2ll * cluster_count()) {
      const int h = static_cast<int>(u / p.n_pairs);
      const int pr = static_cast<int>(u - static_cast<long long>(h) * p.n_pairs);
      const int beg = __ldg(p.prow_ptr + pr);
      const int n = __ldg(p.prow_ptr + pr + 1) - beg;
      const int row = 2 * pr + static_cast<int>(crank);
      const bool row_valid = row < p.n_rows;
      __nv_bfloat16* orow =
          p.out + (static_cast<long long>(row) * kBM + r) * p.out_tok_stride + h * p.out_head_stride;
      if (n == 0) {
        // attention.cpp:85-86 throws domain_error; the output stays defined
        // (zeros) and the flag reaches the caller
        if (row_valid) {
          const uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
          for (int v = 0; v < kD / 8; ++v) reinterpret_cast<uint4*>(orow)[v] = z;
          if (p.err_flag && r == 0) atomicOr(p.err_flag, 1);
        }
        continue;
      }
      float m = -INFINITY;  // reference max (raw logits), may be stale by < 2^8
      float l = 0.f;
      bool first = true;
      uint32_t fl_nxt = __ldg(p.uflag + beg);
      for (int j = 0; j < n; ++j, ++g) {
        const bool member = (fl_nxt >> crank) & 1u;
        if (j + 1 < n) fl_nxt = __ldg(p.uflag + beg + j + 1);
        mbar_wait(&s_full[t], g & 1);
        tc_fence_after();
        if (member) {
          uint32_t s[128];
          tmem_ld32(trow + scol + 0, *reinterpret_cast<uint32_t(*)[32]>(s + 0));
          tmem_ld32(trow + scol + 32, *reinterpret_cast<uint32_t(*)[32]>(s + 32));
          tmem_ld32(trow + scol + 64, *reinterpret_cast<uint32_t(*)[32]>(s + 64));
          tmem_ld32(trow + scol + 96, *reinterpret_cast<uint32_t(*)[32]>(s + 96));
          tmem_wait_ld();
          auto S = [&](int e) -> float { return __uint_as_float(s[e]); };
          float mxs[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) mxs[c] = fmax3(S(16 * c), S(16 * c + 1), S(16 * c + 2));
#pragma unroll
          for (int e = 3; e < 15; e += 2)
#pragma unroll
            for (int c = 0; c < 8; ++c) mxs[c] = fmax3(mxs[c], S(16 * c + e), S(16 * c + e + 1));
#pragma unroll
          for (int c = 0; c < 8; ++c) mxs[c] = fmaxf(mxs[c], S(16 * c + 15));
          const float mx = fmax3(fmax3(mxs[0], mxs[1], mxs[2]), fmax3(mxs[3], mxs[4], mxs[5]),
                                 fmaxf(mxs[6], mxs[7]));
          if (first) {
            // O holds only zero contributions so far (P = 0 entries, or none)
            m = mx;
          } else {
            // Lazy rescale (threshold 2^8, exact: O and l rebased together).
            // O holds P(j-1).V(j-1): S(j) was committed after it.
            const bool need = (mx - m) * sl2 > 8.0f;
            if (__any_sync(0xFFFFFFFFu, need)) {
              const float alpha = need ? ex2((m - mx) * sl2) : 1.0f;
              if (need) {
                m = mx;
                l *= alpha;
              }
#pragma unroll
              for (int c = 0; c < kD / 32; ++c) {
                uint32_t o[32];
                const uint32_t oc = trow + ocol + c * 32;
                tmem_ld32(oc, o);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
                tmem_st32(oc, o);
              }
            }
          }
          first = false;
          const float2 sc2 = make_float2(sl2, sl2);
          const float nb = -m * sl2;
          const float2 ng2 = make_float2(nb, nb);
          float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
          float2 prev[16];
#pragma unroll
          for (int c = 0; c <= 4; ++c) {
            float2 cur[16];
            if (c < 4) {
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const int e = 32 * c + 2 * i;
                const float2 xv = ffma2(make_float2(S(e), S(e + 1)), sc2, ng2);
                if (kPolyMask & (1u << i)) {
                  cur[i] = ex2_poly2(xv);
                } else {
                  cur[i].x = ex2(xv.x);
                  cur[i].y = ex2(xv.y);
                }
              }
            }
            if (c > 0) {
              uint32_t pk[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                if (i & 1)
                  acc1 = fadd2(acc1, prev[i]);
                else
                  acc0 = fadd2(acc0, prev[i]);
                pk[i] = pack_bf16(prev[i].x, prev[i].y);
              }
              tmem_st16(trow + scol + 16 * (c - 1), pk);
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) prev[i] = cur[i];
          }
          const float2 at = fadd2(acc0, acc1);
          l += at.x + at.y;
        } else {
          // block not in this row's list: P = 0
          uint32_t z[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) z[i] = 0u;
          tmem_st32(trow + scol, z);
          tmem_st32(trow + scol + 32, z);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_cluster(pf_addr);
      }
      // epilogue: wait for the unit's last P.V; O / l -> bf16 -> global
      mbar_wait(&o_done[t], ord & 1);
      tc_fence_after();
      const float inv = l > 0.f ? 1.0f / l : 0.f;  // a row with no own block: zeros
      if (row_valid && first && p.err_flag && r == 0) atomicOr(p.err_flag, 1);
#pragma unroll
      for (int c = 0; c < kD / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(trow + ocol + c * 32, o);
        tmem_wait_ld();
        if (row_valid) {
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
      // the next unit's first P.V (which overwrites O) is issued only after
      // this warp's next p_full arrival, which follows these completed loads
      tc_fence_before();
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

}  // namespace attn10
}  // namespace rp
