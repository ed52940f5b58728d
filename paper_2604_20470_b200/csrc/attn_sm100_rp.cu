// K6 (v3): block-sparse flash-attention forward with two query row blocks of
// the same head sharing every K/V tile (bf16 in / fp32 softmax, sm_100a).
//
// Same semantics as attn_sm100_db.cu (attention.cpp:50-121,
// exact mask, zero-padded keys attended when their block is active).
//
// Why.  With one query tile per CTA every KV step streams a 32 KB K tile and
// a 32 KB V tile through L2 -> shared memory for 128 rows of work: at the Wan
// shape that is ~7.6 TB/s of L2 -> SM traffic, near the L2 throughput cap,
// and the tensor core's operand reads compete with the TMA writes for shared
// memory (ablation: skipping the K/V reloads makes the db kernel 16 % faster).
// Neighbouring block rows of a radial mask attend almost the same KV blocks,
// so a CTA here owns the row PAIR (2p, 2p+1) of one head and walks their
// blocks as ENTRIES (pair_fill_kernel): first the blocks both rows hold (one
// K/V load used by both query tiles), then "split" entries pairing A's i-th
// exclusive block with B's (two loads, one per tile), then the leftovers.
// S_A / S_B and P_A V / P_B V are issued only for the tiles an entry holds --
// no masked work -- and every two-tile entry keeps the tiles in ping-pong
// (round 2: split entries instead of the sorted union, Hunyuan stage (d)
// 1076 -> 1135 TFLOP/s).
//
// TMEM (512 columns): S_A 0-127, S_B 128-255, O_A 256-(256+D), O_B 384-(384+D);
// P_x (bf16) overwrites the first 64 columns of S_x and is the A operand of
// P_x V straight from TMEM.  Warps 0-3 / 4-7 run the softmax of tiles A / B
// (thread = row, 128 keys per row); the two tiles ping-pong on the tensor
// core.  MMA order per union entry e:  P_A(e-1) V, S_A(e), P_B(e-1) V, S_B(e)
// (each only if the tile holds that block), so K(e) and V(e-1) are released
// right after their last use and the ring stays FIFO.  Online softmax with a
// stale reference max (see attn_sm100_db.cu), exact lazy rescaling.
#include "common.cuh"

namespace rp {
namespace attn3 {

constexpr int kThreads = 384;
constexpr int kBM = 128;
constexpr int kBN = 128;
// Pairs (of every 8 per 16-key chunk) whose exp2 runs as a polynomial on the
// FMA pipe: 1 of 8 measured +1.1 % at the Hunyuan shape (bench, two
// interleaved runs: 101.5-102.3 vs 102.9-103.4 ms), neutral at Wan; 2 of 8
// was slower.
#ifndef RP_RP_POLY_MASK
#define RP_RP_POLY_MASK 0x01u
#endif
constexpr uint32_t kPolyMask = RP_RP_POLY_MASK;

template <int D>
struct Layout {
  static constexpr int kChunks = D / 64;
  static constexpr int kTileBytes = 128 * D * 2;
  static constexpr int kChunkBytes = 128 * 128;
  static constexpr int kStages = D == 128 ? 5 : 10;
  static constexpr int kSmemData = 2 * kTileBytes + kStages * kTileBytes;
  static constexpr int kNumBars = 2 * kStages + 12;
  static constexpr int kSmemBytes = kSmemData + kNumBars * 8 + 16 + 1024;
  static_assert(kSmemBytes <= 232448, "exceeds the 227 KB opt-in shared memory");
  RP_HD static uint32_t s_col(int x) { return x ? 128u : 0u; }
  RP_HD static uint32_t o_col(int x) { return x ? 384u : 256u; }
};

struct Params {
  const int32_t* row_ptr;   // per block row (own list lengths)
  const int32_t* prow_ptr;  // per row pair: union list offsets
  const int32_t* pcol;      // per entry: (block of row 2p, block of row 2p+1), see pair_fill
  const uint8_t* pflag;     // bit 0: row 2p active, bit 1: row 2p+1 active, bit 2: split
                            // entry (the two rows take DIFFERENT blocks, two K/V loads)
  const int32_t* porder;    // pairs by descending union size (may be null)
  int n_rows;               // S_b
  int n_pairs;              // ceil(S_b / 2)
  int heads;
  long long n_units;        // heads * n_pairs
  __nv_bfloat16* out;
  long long out_tok_stride;
  long long out_head_stride;
  float scale_log2;
  // Soft mask (masked_attention, attention.cpp:59-81; null = exact), as in
  // attn_sm100_db.cu: own lists are dense and a block whose bit is clear
  // gets the raw-logit offset soft_delta.
  const int32_t* col_idx;   // own block lists (CSR, with row_ptr)
  const uint8_t* soft_bits;
  long long soft_row_bytes;
  float soft_delta;
};

// Per-entry metadata (flags, block pair) read 32 entries at a time by the
// whole warp (lane i: entry base + i) with the next 32 prefetched, and
// broadcast per entry: a dependent global load per entry sat on the producer
// and MMA issue paths (~0.5 us each).
struct EntryStream {
  const uint8_t* flags;
  const int2* cols;
  int n, base = -1;
  uint32_t f_cur = 0, f_nxt = 0;
  int2 c_cur = make_int2(0, 0), c_nxt = make_int2(0, 0);
  RP_DEV void load(int b, uint32_t& f, int2& c) const {
    const int e = b + (threadIdx.x & 31);
    f = e < n ? __ldg(flags + e) : 0u;
    c = e < n && cols ? __ldg(cols + e) : make_int2(0, 0);
  }
  RP_DEV void at(int e, uint32_t* fl, int* ca, int* cb) {
    const int b = e & ~31;
    if (b != base) {
      if (base >= 0 && b == base + 32) {
        f_cur = f_nxt;
        c_cur = c_nxt;
      } else {
        load(b, f_cur, c_cur);
      }
      load(b + 32, f_nxt, c_nxt);
      base = b;
    }
    *fl = __shfl_sync(0xFFFFFFFFu, f_cur, e & 31);
    if (ca) *ca = __shfl_sync(0xFFFFFFFFu, c_cur.x, e & 31);
    if (cb) *cb = __shfl_sync(0xFFFFFFFFu, c_cur.y, e & 31);
  }
};

struct Unit {
  int h, p, row[2], beg, n, cnt[2];
  bool has[2];
};

RP_DEV Unit decode(const Params& p, long long u, bool warp_uniform) {
  Unit w;
  w.h = static_cast<int>(u / p.n_pairs);
  const int pi = static_cast<int>(u % p.n_pairs);
  int pp = p.porder ? __ldg(p.porder + pi) : pi;
  int beg = __ldg(p.prow_ptr + pp);
  int end = __ldg(p.prow_ptr + pp + 1);
  if (warp_uniform) {
    pp = shfl0(pp);
    beg = shfl0(beg);
    end = shfl0(end);
  }
  w.p = pp;
  w.beg = beg;
  w.n = end - beg;
  for (int x = 0; x < 2; ++x) {
    w.row[x] = 2 * pp + x;
    w.has[x] = w.row[x] < p.n_rows;
    int c = w.has[x] ? __ldg(p.row_ptr + w.row[x] + 1) - __ldg(p.row_ptr + w.row[x]) : 0;
    if (warp_uniform) c = shfl0(c);
    w.cnt[x] = c;
    w.has[x] = w.has[x] && c > 0;
  }
  return w;
}

// Union lists of the row pairs: counts, then fill (one thread per pair; the
// two lists are sorted, so a linear merge).
__global__ void pair_count_kernel(const int32_t* __restrict__ row_ptr,
                                  const int32_t* __restrict__ col, int n_rows, int n_pairs,
                                  int32_t* __restrict__ counts) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pairs) return;
  const int a = 2 * p, b = 2 * p + 1;
  int i = row_ptr[a], ie = row_ptr[a + 1];
  int j = b < n_rows ? row_ptr[b] : 0, je = b < n_rows ? row_ptr[b + 1] : 0;
  int nc = 0, na = 0, nb = 0;
  while (i < ie || j < je) {
    const int ca = i < ie ? col[i] : 0x7FFFFFFF, cb = j < je ? col[j] : 0x7FFFFFFF;
    if (ca == cb) ++nc;
    else if (ca < cb) ++na;
    else ++nb;
    i += ca <= cb;
    j += cb <= ca;
  }
  counts[p] = nc + (na > nb ? na : nb);  // entries: common, split pairs, leftovers
}

// Entry order of a row pair (A = 2p, B = 2p+1): first the blocks both rows
// hold (ascending; one K/V load feeds both tiles), then the exclusive blocks
// as SPLIT entries (A's i-th exclusive block with B's i-th: two K/V loads,
// one per tile), then the leftover exclusive blocks of the longer list.
// Online softmax is order-independent up to rounding; the order decides the
// schedule.  In every entry with both tiles active the MMA warp issues
// P_A.V, S_A, P_B.V, S_B, so the two tiles' softmax and MMAs ping-pong; in
// the sorted union order used before, runs of one-tile entries exposed a
// tile's softmax -> P.V -> S chain (Wan: 16.5 % of the tile steps).
__global__ void pair_fill_kernel(const int32_t* __restrict__ row_ptr,
                                 const int32_t* __restrict__ col, int n_rows, int n_pairs,
                                 const int32_t* __restrict__ prow_ptr, int32_t* __restrict__ pcol,
                                 uint8_t* __restrict__ pflag) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pairs) return;
  const int a = 2 * p, b = 2 * p + 1;
  const int ia = row_ptr[a], iae = row_ptr[a + 1];
  const int ib = b < n_rows ? row_ptr[b] : 0, ibe = b < n_rows ? row_ptr[b + 1] : 0;
  int nc = 0, na = 0, nb = 0;
  for (int i = ia, j = ib; i < iae || j < ibe;) {
    const int ca = i < iae ? col[i] : 0x7FFFFFFF, cb = j < ibe ? col[j] : 0x7FFFFFFF;
    if (ca == cb) ++nc;
    else if (ca < cb) ++na;
    else ++nb;
    i += ca <= cb;
    j += cb <= ca;
  }
  const int o = prow_ptr[p];
  const int m = na < nb ? na : nb;
  for (int e = nc; e < nc + (na > nb ? na : nb); ++e) {  // split / leftover entries
    pcol[2 * (o + e)] = -1;
    pcol[2 * (o + e) + 1] = -1;
    pflag[o + e] = 0;
  }
  int kc = 0, ka = 0, kb = 0;
  for (int i = ia, j = ib; i < iae || j < ibe;) {
    const int ca = i < iae ? col[i] : 0x7FFFFFFF, cb = j < ibe ? col[j] : 0x7FFFFFFF;
    if (ca == cb) {
      pcol[2 * (o + kc)] = ca;
      pcol[2 * (o + kc) + 1] = ca;
      pflag[o + kc] = 3;
      ++kc;
    } else if (ca < cb) {
      const int e = o + nc + (ka < m ? ka : m + (ka - m));
      pcol[2 * e] = ca;
      pflag[e] |= ka < m ? 1 | 4 : 1;
      ++ka;
    } else {
      const int e = o + nc + (kb < m ? kb : m + (kb - m));
      pcol[2 * e + 1] = cb;
      pflag[e] |= kb < m ? 2 | 4 : 2;
      ++kb;
    }
    i += ca <= cb;
    j += cb <= ca;
  }
}

// The same entry lists as pair_count_kernel / pair_fill_kernel, one WARP per
// row pair: the two rows' blocks go into shared-memory bitmaps, common /
// A-only / B-only blocks come out of the bitmap words in ascending order
// (per-lane word ranges + a warp scan), so the lists are identical while a
// pair no longer costs one thread's serial merge of both lists.  kWords
// bounds S_b (32 * kWords blocks); larger grids use the per-thread kernels.
constexpr int kPairWords = 64;     // S_b <= 2048
constexpr int kPairWarps = 8;
template <bool FILL>
__global__ void __launch_bounds__(32 * kPairWarps)
    pair_lists_warp_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                           int n_rows, int n_pairs, int32_t* __restrict__ counts,
                           const int32_t* __restrict__ prow_ptr, int32_t* __restrict__ pcol,
                           uint8_t* __restrict__ pflag) {
  __shared__ uint32_t bm[kPairWarps][2][kPairWords];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p = blockIdx.x * kPairWarps + w;
  if (p >= n_pairs) return;
  const int nw = (n_rows + 31) >> 5;
  uint32_t* A = bm[w][0];
  uint32_t* B = bm[w][1];
  for (int x = lane; x < nw; x += 32) {
    A[x] = 0u;
    B[x] = 0u;
  }
  __syncwarp();
  const int a = 2 * p, b = 2 * p + 1;
  for (int i = row_ptr[a] + lane; i < row_ptr[a + 1]; i += 32) {
    const int c = col[i];
    atomicOr(&A[c >> 5], 1u << (c & 31));
  }
  if (b < n_rows)
    for (int i = row_ptr[b] + lane; i < row_ptr[b + 1]; i += 32) {
      const int c = col[i];
      atomicOr(&B[c >> 5], 1u << (c & 31));
    }
  __syncwarp();
  // lane l owns words [l * per, (l + 1) * per)
  const int per = (nw + 31) >> 5;
  const int w0 = lane * per, w1 = min(nw, w0 + per);
  int mc = 0, ma = 0, mb = 0;
  for (int x = w0; x < w1; ++x) {
    mc += __popc(A[x] & B[x]);
    ma += __popc(A[x] & ~B[x]);
    mb += __popc(B[x] & ~A[x]);
  }
  int ic = mc, ia = ma, ib = mb;  // inclusive scans
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int yc = __shfl_up_sync(0xFFFFFFFFu, ic, o);
    const int ya = __shfl_up_sync(0xFFFFFFFFu, ia, o);
    const int yb = __shfl_up_sync(0xFFFFFFFFu, ib, o);
    if (lane >= o) {
      ic += yc;
      ia += ya;
      ib += yb;
    }
  }
  const int nc = __shfl_sync(0xFFFFFFFFu, ic, 31);
  const int na = __shfl_sync(0xFFFFFFFFu, ia, 31);
  const int nb = __shfl_sync(0xFFFFFFFFu, ib, 31);
  if (!FILL) {
    if (lane == 0) counts[p] = nc + (na > nb ? na : nb);
    return;
  }
  const int o = prow_ptr[p];
  const int m = na < nb ? na : nb;
  int kc = ic - mc, ka = ia - ma, kb = ib - mb;
  for (int x = w0; x < w1; ++x) {
    for (uint32_t v = A[x] & B[x]; v; v &= v - 1) {
      const int c = 32 * x + __ffs(v) - 1;
      pcol[2 * (o + kc)] = c;
      pcol[2 * (o + kc) + 1] = c;
      pflag[o + kc] = 3;
      ++kc;
    }
    for (uint32_t v = A[x] & ~B[x]; v; v &= v - 1) {
      const int c = 32 * x + __ffs(v) - 1;
      const int e = o + nc + ka;  // split (ka < m) or leftover (then na > nb)
      pcol[2 * e] = c;
      if (ka < m) {
        pflag[e] = 1 | 2 | 4;
      } else {
        pcol[2 * e + 1] = -1;
        pflag[e] = 1;
      }
      ++ka;
    }
    for (uint32_t v = B[x] & ~A[x]; v; v &= v - 1) {
      const int c = 32 * x + __ffs(v) - 1;
      const int e = o + nc + kb;
      pcol[2 * e + 1] = c;
      if (kb >= m) {
        pcol[2 * e] = -1;
        pflag[e] = 2;
      }
      ++kb;
    }
  }
}

template <int D, bool SOFT = false>
__global__ void __launch_bounds__(kThreads, 1)
    bsfa_fwd_rp_kernel(const __grid_constant__ CUtensorMap tq,
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
  uint64_t* q_full = bars + 2 * L::kStages;  // [2]
  uint64_t* q_empty = q_full + 2;
  uint64_t* s_full = q_full + 4;
  uint64_t* p_full = q_full + 6;
  uint64_t* o_done = q_full + 8;
  uint64_t* o_free = q_full + 10;
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
      // ring order = MMA consumption order: K(0), then V(e-1), K(e), ...,
      // V(n-1); every union entry is held by at least one of the two rows
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
        // ring order per entry e: V of entry e-1 (A's, then B's if split),
        // then K of entry e (likewise) -- the MMA warp's consumption order
        EntryStream es{p.pflag + w.beg, reinterpret_cast<const int2*>(p.pcol) + w.beg, w.n};
        int pa = 0, pb = 0;
        uint32_t pfl = 0;
        for (int e = 0; e <= w.n; ++e) {
          if (e > 0) {
            if (pfl & 4) {
              load_kv(&tv, w.h, pa);
              load_kv(&tv, w.h, pb);
            } else {
              load_kv(&tv, w.h, (pfl & 1) ? pa : pb);
            }
          }
          if (e < w.n) {
            uint32_t fl;
            int ca, cb;
            es.at(e, &fl, &ca, &cb);
            if (fl & 4) {
              load_kv(&tk, w.h, ca);
              load_kv(&tk, w.h, cb);
            } else {
              load_kv(&tk, w.h, (fl & 1) ? ca : cb);
            }
            pa = ca;
            pb = cb;
            pfl = fl;
          }
        }
      }
    } else if (warp == 9) {
      // ----------------------------------------------------- MMA issuer ---
      const uint32_t idesc_qk = idesc_bf16(128, 128, false, false);
      const uint32_t idesc_pv = idesc_bf16(128, D, false, true);
      const uint32_t sq_addr = smem_u32(sq);
      const uint32_t skv_addr = smem_u32(skv);
      uint32_t kv_it = 0;
      uint32_t ucnt[2] = {0, 0};
      uint32_t pcnt[2] = {0, 0};
      for (long long u = blockIdx.x; u < p.n_units; u += gridDim.x) {
        const Unit w = decode(p, u, true);
        if (w.n == 0) continue;
        EntryStream es{p.pflag + w.beg, nullptr, w.n};
        int done_s[2] = {0, 0}, done_pv[2] = {0, 0};
        uint32_t prev_fl = 0;
        for (int e = 0; e <= w.n; ++e) {
          uint32_t fl = 0u;
          if (e < w.n) es.at(e, &fl, nullptr, nullptr);
          // ring slots: V of entry e-1 (two if it was split), then K of entry e
          uint32_t v_st[2] = {0, 0}, k_st[2] = {0, 0};
          auto take = [&]() {
            const uint32_t st = kv_it % L::kStages;
            mbar_wait(&kv_full[st], (kv_it / L::kStages) & 1);
            ++kv_it;
            return st;
          };
          if (e > 0) {
            v_st[0] = take();
            v_st[1] = (prev_fl & 4) ? take() : v_st[0];
          }
          if (e < w.n) {
            k_st[0] = take();
            k_st[1] = (fl & 4) ? take() : k_st[0];
          }
          tc_fence_after();
          // a shared slot is released by its last user (B if B uses it); a
          // split entry's slots have one user each
          const int last_pv = ((prev_fl & 2) && !(prev_fl & 4)) ? 1 : 0;
          const int last_s = ((fl & 2) && !(fl & 4)) ? 1 : 0;
#pragma unroll
          for (int x = 0; x < 2; ++x) {
            if (e > 0 && (prev_fl >> x) & 1) {
              // O_x (+)= P_x(e-1) V(e-1)
              mbar_wait(&p_full[x], pcnt[x] & 1);
              ++pcnt[x];
              if (done_pv[x] == 0) mbar_wait(&o_free[x], (ucnt[x] & 1) ^ 1);
              tc_fence_after();
              const uint32_t vb = skv_addr + v_st[x] * L::kTileBytes;
#pragma unroll
              for (int kk = 0; kk < kBN / 16; ++kk)
                umma_ts_w(tmem + L::o_col(x), tmem + L::s_col(x) + kk * 8,
                          smem_desc_sw128(vb + kk * 16 * 128, L::kChunkBytes, 1024), idesc_pv,
                          done_pv[x] > 0 || kk > 0);
              ++done_pv[x];
              if (done_pv[x] == w.cnt[x]) umma_commit_w(&o_done[x]);
              if ((prev_fl & 4) || x == last_pv) umma_commit_w(&kv_empty[v_st[x]]);
            }
            if (e < w.n && (fl >> x) & 1) {
              // S_x(e) = Q_x K(e)^T (overwrites P_x of its previous block,
              // whose P.V was issued above / earlier)
              if (done_s[x] == 0) mbar_wait(&q_full[x], ucnt[x] & 1);
              tc_fence_after();
              const uint32_t qa = sq_addr + x * L::kTileBytes;
              const uint32_t kb = skv_addr + k_st[x] * L::kTileBytes;
#pragma unroll
              for (int kk = 0; kk < D / 16; ++kk) {
                const uint32_t off = (kk / 4) * L::kChunkBytes + (kk % 4) * 32;
                umma_ss_w(tmem + L::s_col(x), smem_desc_sw128(qa + off, 0, 1024),
                          smem_desc_sw128(kb + off, 0, 1024), idesc_qk, kk > 0);
              }
              ++done_s[x];
              umma_commit_w(&s_full[x]);
              if (done_s[x] == w.cnt[x]) umma_commit_w(&q_empty[x]);
              if ((fl & 4) || x == last_s) umma_commit_w(&kv_empty[k_st[x]]);
            }
          }
          prev_fl = fl;
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
    uint32_t scnt = 0, ucnt = 0;
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
      const int my_beg = SOFT ? __ldg(p.row_ptr + my_row) : 0;
      for (int j = 0; j < my_cnt; ++j) {
        float dlt = 0.f;  // soft-mask offset of this block (0: exact mode / active)
        if constexpr (SOFT) {
          const int c = __ldg(p.col_idx + my_beg + j);
          const uint8_t by = __ldg(p.soft_bits + my_row * p.soft_row_bytes + (c >> 3));
          dlt = ((by >> (c & 7)) & 1) ? 0.f : p.soft_delta;
        }
        mbar_wait(&s_full[x], scnt & 1);
        ++scnt;
        tc_fence_after();
        uint32_t s0[32], s1[32], s2[32], s3[32];
        tmem_ld32(trow + L::s_col(x) + 0, s0);
        tmem_ld32(trow + L::s_col(x) + 32, s1);
        tmem_ld32(trow + L::s_col(x) + 64, s2);
        tmem_ld32(trow + L::s_col(x) + 96, s3);
        tmem_wait_ld();
        auto S = [&](int e) -> float {
          const uint32_t v = e < 32 ? s0[e] : e < 64 ? s1[e - 32] : e < 96 ? s2[e - 64] : s3[e - 96];
          return __uint_as_float(v);
        };
        if (j == 0) {
          float a = S(0);
#pragma unroll
          for (int i = 1; i < 127; i += 2) a = fmaxf(a, fmaxf(S(i), S(i + 1)));
          m = fmaxf(a, S(127)) + dlt;
        }
        // exponentials against the (stale) reference max, 32-key chunks:
        // a chunk's exponentials overlap the packing and TMEM store of the
        // previous one; this block's max is folded in alongside
        float2 acc[2];
        float lmax = -INFINITY;
        auto exps = [&](float mref, bool track) {
          const float2 sc2 = make_float2(sl2, sl2);
          const float nb = (dlt - mref) * sl2;
          const float2 ng2 = make_float2(nb, nb);
          acc[0] = acc[1] = make_float2(0.f, 0.f);
          float2 pv_prev[8];
#pragma unroll
          for (int c = 0; c <= 8; ++c) {  // 16-key chunks (register budget)
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
            if (c > 0) tmem_st8(trow + L::s_col(x) + 8 * (c - 1), pk);
#pragma unroll
            for (int i = 0; i < 8; ++i) pv_prev[i] = pv_cur[i];
          }
        };
        exps(m, false);
        // rescale guard from the row sum (see attn_sm100_db.cu): a block
        // whose exponentials sum to <= 2^8 cannot hold a max more than 2^8
        // above the reference; only otherwise is the block max computed
        const float2 at0 = fadd2(acc[0], acc[1]);
        if (j > 0 && __any_sync(0xFFFFFFFFu, !(at0.x + at0.y <= 256.0f))) {
          float a = S(0);
#pragma unroll
          for (int i = 1; i < 127; i += 2) a = fmaxf(a, fmaxf(S(i), S(i + 1)));
          lmax = fmaxf(a, S(127)) + dlt;
          const bool need = (lmax - m) * sl2 > 8.0f;
          if (__any_sync(0xFFFFFFFFu, need)) {
            // rebase on the new max: O_x is stable here (S_x(j) was issued
            // after P_x(j-1) V and its commit covers every earlier MMA)
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
        if (lane == 0) mbar_arrive(&p_full[x]);
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

}  // namespace attn3
}  // namespace rp
