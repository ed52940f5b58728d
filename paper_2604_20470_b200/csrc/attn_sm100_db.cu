// K6 (v2): block-sparse flash-attention forward, bf16 in / fp32 softmax,
// sm_100a, with the score tile double-buffered in TMEM.
//
// Replaces radialplan::masked_attention_exact (attention.cpp:50-121) on the
// tensor cores, with the reference's exact-mask semantics: only the row's CSR
// blocks are attended (-inf elsewhere, constant per B x B block), and rows
// >= S are TMA out-of-bounds zeros that take part as keys with logit 0
// whenever their block is active (attention.cpp:43-48, 66-68).
//
// Why this design.  In the first (since removed) two-head ping-pong kernel each head's score
// tile S lives in one TMEM buffer that P overwrites, so S(j+1) can only be
// computed after P(j).V(j) has read P(j): every KV step pays softmax latency
// + MMA latency in series (measured: 2.1k + 1.4k clk per step, tensor pipe
// ~58 % busy).  Here a CTA owns ONE 128-row query tile with two S buffers:
//   TMEM  S0 cols 0-127 | S1 cols 128-255 | O cols 256-(256+D)
// The MMA warp issues S(g+2) right after P(g).V(g), so S(g+1) is already in
// TMEM when the softmax of step g finishes: the softmax runs back to back and
// the tensor core works underneath it.
//
// Softmax: 8 warps (two per SM sub-partition, so their MUFU / FMA work
// interleaves).  Warps w and w+4 share TMEM lanes 32(w%4)..+31 (the same 32
// query rows) and split the 128 keys: half h = w/4 owns keys [64h, 64h+64),
// P columns [32h, 32h+32) of the step's buffer, and O columns [hD/2, hD/2+D/2).
// The row max is combined through shared memory with a 64-thread named
// barrier per row group; the row sums stay per half until the epilogue.
// Lazy rescaling (threshold 2^8, exact: O and l are rebased together); a rescale waits
// for the previous step's P.V to retire before touching O.
//
//   warps 0-7   softmax / epilogue       warp 8  TMA producer (whole warp)
//   warp  9     MMA issuer (whole warp)  warps 10-11 idle (setmaxnreg group)
#include "common.cuh"

namespace rp {
namespace attn2 {

constexpr int kThreads = 384;
constexpr int kBM = 128;
constexpr int kBN = 128;
// Pairs (of every 8) whose exp2 runs as a polynomial on the FMA pipe.  None
// by default: single launches are ~equal at 0 or 1 of 8, but under sustained
// (power-capped) load the extra FMA-pipe instructions cost more than the MUFU
// relief (tools/ab_k6.py: 22.86 vs 23.05 ms; 2 of 8: 23.46 ms).
#ifndef RP_DB_POLY_MASK
#define RP_DB_POLY_MASK 0x00u
#endif
constexpr uint32_t kPolyMask = RP_DB_POLY_MASK;

template <int D>
struct Layout {
  static constexpr int kChunks = D / 64;          // 128-byte K chunks per row
  static constexpr int kTileBytes = 128 * D * 2;  // one 128-row bf16 tile
  static constexpr int kChunkBytes = 128 * 128;
#ifdef RP_DB_STAGES
  static constexpr int kStages = RP_DB_STAGES;
#else
  static constexpr int kStages = D == 128 ? 4 : 8;  // 2 Q tiles + ring <= 227 KB
#endif
  static constexpr int kSmemData = 2 * kTileBytes + kStages * kTileBytes;
  static constexpr int kNumBars = 2 * kStages + 13 + 2;
  // row max x2 slots, row sums, block sums x2 slots, lagged block sums x4
  // slots, per-row |Q|^2 halves x2 Q buffers
  static constexpr int kRedBytes =
      (2 * 2 * 128 + 2 * 128 + 2 * 2 * 128 + 4 * 2 * 128 + 2 * 2 * 128) * 4;
  static constexpr int kSmemBytes = kSmemData + kNumBars * 8 + 16 + kRedBytes + 1024;
  static_assert(kSmemBytes <= 232448, "exceeds the 227 KB opt-in shared memory");
  static constexpr uint32_t kO = 256;  // TMEM column of O
  // Q tiles as the A operand of S = Q K^T live in TMEM (bf16 pairs, D/2
  // columns each, double-buffered by unit): the tensor core then reads only
  // K from shared memory for S, which cuts the step's shared-memory traffic
  // (Q 32 KB + K 32 KB + V 32 KB reads + 64 KB TMA writes) by a fifth.
  RP_HD static uint32_t qt_col(int b) { return 384u + (b ? 64u : 0u); }
};

struct Params {
  const int32_t* row_ptr;
  const int32_t* col_idx;
  const int32_t* row_order;  // may be null
  int n_rows;                // S_b
  int heads;
  long long n_units;         // heads * n_rows
  __nv_bfloat16* out;
  long long out_tok_stride;
  long long out_head_stride;
  float scale_log2;
  // Per-head max_t |k_t| (may be null): enables the exchange-free rescale
  // protocol for units whose logits provably stay within 2^64 of the first
  // block's max (see the softmax below).
  const float* kmax_head;
  // Soft mask (masked_attention, attention.cpp:59-81; null = exact mask):
  // the row lists are dense and a block whose bit is clear gets the logit
  // offset soft_delta = (log eps - log1p eps) / scale (raw-logit units; the
  // common log1p eps of active blocks cancels in the softmax).
  const uint8_t* soft_bits;
  long long soft_row_bytes;
  float soft_delta;
  // B = 64 masks (QM kernels): the CSR is over 128 x 128 TILES (pairs of
  // 64-blocks), qmask[entry] holds the tile's four 64 x 64 quadrant bits
  // (bit 2 * row_half + key_half); out_rows = S' of the 64-block axis, rows
  // at or beyond it exist only in the 128-row tile and are not written.
  const uint8_t* qmask;
  long long out_rows;
};

#ifdef RP_TRACE
constexpr int kTraceCtas = 4, kTraceEv = 12, kTraceSteps = 512;
__device__ unsigned long long g_trace[kTraceCtas][kTraceEv][kTraceSteps];
#define RP_TR2(ev, idx)                                                       \
  do {                                                                        \
    if (blockIdx.x < kTraceCtas && (idx) < kTraceSteps)                       \
      g_trace[blockIdx.x][ev][idx] = clock64();                               \
  } while (0)
#else
#define RP_TR2(ev, idx) \
  do {                  \
  } while (0)
#endif

// Walks this CTA's units (head-major: consecutive units of a CTA stride over
// rows of the same head, so concurrently running CTAs share K/V in L2) and
// their KV blocks.  Empty rows are skipped (the softmax warps zero them).
// All fields are warp-uniform (lookups broadcast from lane 0).
struct Cursor {
  long long u;
  int ord;  // ordinal among this CTA's non-empty units
  int j, n, beg, h, row;
  bool valid;

  RP_DEV void seek(const Params& p) {
    valid = false;
    for (; u < p.n_units; u += gridDim.x) {
      const int hh = static_cast<int>(u / p.n_rows);
      const int ri = static_cast<int>(u % p.n_rows);
      const int r = shfl0(p.row_order ? __ldg(p.row_order + ri) : ri);
      const int b = shfl0(__ldg(p.row_ptr + r));
      const int e = shfl0(__ldg(p.row_ptr + r + 1));
      if (e > b) {
        h = hh;
        row = r;
        beg = b;
        n = e - b;
        j = 0;
        cbase = -1;
        valid = true;
        return;
      }
    }
  }
  RP_DEV void start(const Params& p) {
    u = blockIdx.x;
    ord = 0;
    seek(p);
  }
  RP_DEV void next(const Params& p) {
    if (++j < n) return;
    u += gridDim.x;
    ++ord;
    seek(p);
  }
  // KV block index of step j.  The producer used to load it with one
  // dependent global load per tile (~0.5 us on the TMA issue path); now a
  // warp loads 32 indices at once (lane i: index base + i) and prefetches the
  // next 32, so only a unit's first chunk waits on memory.
  int cb = 0, nb = 0, cbase = -1;
  RP_DEV int col(const Params& p) {
    const int base = j & ~31;
    if (base != cbase) {
      const int lane = threadIdx.x & 31;
      if (cbase >= 0 && base == cbase + 32)
        cb = nb;
      else
        cb = base + lane < n ? __ldg(p.col_idx + beg + base + lane) : 0;
      nb = base + 32 + lane < n ? __ldg(p.col_idx + beg + base + 32 + lane) : 0;
      cbase = base;
    }
    return __shfl_sync(0xFFFFFFFFu, cb, j & 31);
  }
};

// max_t |k_t| per head (the logit bound of the exchange-free rescale
// protocol): one thread per (token, head), 16-byte loads, fp32 sum of squares,
// atomicMax on the non-negative float's bits.
// max_t |k_t| per head (the logit bound of the exchange-free rescale
// protocol): one warp per token in a grid-stride loop, lane l owns heads
// l, l + 32 (heads <= 64) and keeps their running max in registers; the
// block then reduces through shared memory and issues one atomicMax per
// (block, head).  One read of K (HBM-bound).
__global__ void kmax_kernel(const __nv_bfloat16* __restrict__ k, long long tokens, int heads,
                            int d, long long ts, long long hs, float* __restrict__ kmax) {
  __shared__ int red[64];
  for (int h = threadIdx.x; h < 64; h += blockDim.x) red[h] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long warps = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
  float m0 = 0.f, m1 = 0.f;
  for (long long t = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
       t < tokens; t += warps) {
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      const int h = lane + 32 * x;
      if (h >= heads) continue;
      const uint4* row = reinterpret_cast<const uint4*>(k + t * ts + h * hs);
      float acc = 0.f;
      for (int c = 0; c < d / 8; ++c) {
        const uint4 u = __ldg(row + c);
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float lo = __uint_as_float(w[e] << 16), hi = __uint_as_float(w[e] & 0xFFFF0000u);
          acc = fmaf(lo, lo, fmaf(hi, hi, acc));
        }
      }
      if (x == 0) m0 = fmaxf(m0, acc);
      else m1 = fmaxf(m1, acc);
    }
  }
  if (lane < heads) atomicMax(&red[lane], __float_as_int(sqrtf(m0)));
  if (lane + 32 < heads) atomicMax(&red[lane + 32], __float_as_int(sqrtf(m1)));
  __syncthreads();
  for (int h = threadIdx.x; h < heads; h += blockDim.x)
    atomicMax(reinterpret_cast<int*>(kmax + h), red[h]);
}

template <int D, bool QM = false>
__global__ void __launch_bounds__(kThreads, 1)
    bsfa_fwd_db_kernel(const __grid_constant__ CUtensorMap tq,
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
  float* red_lag = red_sum + 2 * 2 * 128;                     // [4 slots][2 halves][128]
  float* red_qn = red_lag + 4 * 2 * 128;                      // [2 Q buffers][2 halves][128]

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    for (int s = 0; s < L::kStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
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
#ifdef RP_ABL_NOLOAD
        // ablation (timing only): after the ring's first fill, reuse stale tiles
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
      const uint32_t skv_addr = smem_u32(skv);
      uint32_t kv_it = 0, gs = 0, gp = 0;
      Cursor cs, cp;
      cs.start(p);
      cp.start(p);
      // S(gs) = Q . K(gs)^T into buffer gs % 2 (128 x 128, K = D).
      auto issue_s = [&]() {
        const int qb = cs.ord & 1;
        if (cs.j == 0) mbar_wait(&qt_full[qb], (cs.ord >> 1) & 1);
        const uint32_t st = kv_it % L::kStages;
        mbar_wait(&kv_full[st], (kv_it / L::kStages) & 1);
        tc_fence_after();
        const uint32_t kb = skv_addr + st * L::kTileBytes;
        const uint32_t dst = tmem + (gs & 1) * 128;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk / 4) * L::kChunkBytes + (kk % 4) * 32;
          umma_ts_w(dst, tmem + L::qt_col(qb) + kk * 8, smem_desc_sw128(kb + off, 0, 1024),
                    idesc_qk, kk > 0);
        }
        umma_commit_w(&kv_empty[st]);
        umma_commit_w(&s_full[gs & 1]);
        ++kv_it;
        ++gs;
        cs.next(p);
      };
      if (cs.valid) issue_s();
      if (cs.valid) issue_s();
      while (cp.valid) {
        const uint32_t b = gp & 1;
        RP_TR2(6, gp);
        mbar_wait(&p_full[b], (gp >> 1) & 1);
        RP_TR2(7, gp);
        if (cp.j == 0 && cp.ord > 0) mbar_wait(o_free, (cp.ord - 1) & 1);
        tc_fence_after();
        // O (+)= P(gp) . V(gp): P bf16 pairs in TMEM columns [128b, 128b+64)
        const uint32_t st = kv_it % L::kStages;
        mbar_wait(&kv_full[st], (kv_it / L::kStages) & 1);
        tc_fence_after();
        const uint32_t vb = skv_addr + st * L::kTileBytes;
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk)
          umma_ts_w(tmem + L::kO, tmem + b * 128 + kk * 8,
                    smem_desc_sw128(vb + kk * 16 * 128, L::kChunkBytes, 1024), idesc_pv,
                    (cp.j > 0) || kk > 0);
        umma_commit_w(&kv_empty[st]);
        umma_commit_w(pv_done);
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
      if (p.kmax_head) {  // this half's |q_row|^2 for the unit's logit bound
        float qq = 0.f;
#pragma unroll
        for (int t = 0; t < 2 * kUnits * 2; ++t) {
          const float lo = __uint_as_float(v[t] << 16), hi = __uint_as_float(v[t] & 0xFFFF0000u);
          qq = fmaf(lo, lo, fmaf(hi, hi, qq));
        }
        red_qn[(qb * 2 + half) * 128 + r] = qq;
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
    auto next_nonempty = [&](long long u) -> long long {
      for (; u < p.n_units; u += gridDim.x) {
        const int ri = static_cast<int>(u % p.n_rows);
        const int row = p.row_order ? __ldg(p.row_order + ri) : ri;
        if (__ldg(p.row_ptr + row + 1) > __ldg(p.row_ptr + row)) return u;
      }
      return p.n_units;
    };
    long long nx = next_nonempty(blockIdx.x);
    if (nx < p.n_units) q_to_tmem(0);
    for (long long u = blockIdx.x; u < p.n_units; u += gridDim.x) {
      const int h = static_cast<int>(u / p.n_rows);
      const int ri = static_cast<int>(u % p.n_rows);
      const int row = p.row_order ? __ldg(p.row_order + ri) : ri;
      const int beg = __ldg(p.row_ptr + row);
      const int n = __ldg(p.row_ptr + row + 1) - beg;
      __nv_bfloat16* orow = p.out + (static_cast<long long>(row) * kBM + r) * p.out_tok_stride +
                            h * p.out_head_stride + half * (D / 2);
      const bool row_out = !QM || static_cast<long long>(row) * kBM + r < p.out_rows;
      if (n == 0) {  // no active block: defined output (zeros); no pipeline traffic
        uint4 z = make_uint4(0, 0, 0, 0);
        if (row_out) {
#pragma unroll
          for (int v = 0; v < D / 16; ++v) reinterpret_cast<uint4*>(orow)[v] = z;
        }
        continue;
      }
      float m = -INFINITY;  // running max (raw logits), possibly stale
      float l = 0.f;        // this half's row sum
      // exchange-free mode for this unit (decided at j == 0, identically in
      // both halves): own block sums of the last two steps, the step of the
      // last rebase
      bool lag = false;
      float own1 = 0.f, own2 = 0.f;
      int last_rebase = 0;
      for (int j = 0; j < n; ++j, ++g) {
        const uint32_t b = g & 1;
        const uint32_t sb = b * 128;
        float dlt = 0.f;  // soft-mask offset of this block (0: exact mode / active)
        if (p.soft_bits) {
          const int c = __ldg(p.col_idx + beg + j);
          const uint8_t by = __ldg(p.soft_bits + row * p.soft_row_bytes + (c >> 3));
          dlt = ((by >> (c & 7)) & 1) ? 0.f : p.soft_delta;
        }
        if constexpr (QM) {  // this thread's 64 keys are one 64 x 64 quadrant
          const uint8_t qb = __ldg(p.qmask + beg + j);
          if (!((qb >> ((r >= 64 ? 2 : 0) + half)) & 1)) dlt = -INFINITY;
        }
        if (tr) RP_TR2(0, g);
        mbar_wait(&s_full[b], (g >> 1) & 1);
        if (tr) RP_TR2(1, g);
        tc_fence_after();
        uint32_t s0[32], s1[32];
        tmem_ld32(trow + sb + 64 * half, s0);
        tmem_ld32(trow + sb + 64 * half + 32, s1);
        tmem_wait_ld();
        if (tr) RP_TR2(10, g);
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
        // the two halves' sums of this block's exponentials (own slots: the
        // slow path below may exchange a max in the same step)
        auto exchange_sum = [&](float mine) -> float {
          float* slot = red_sum + b * 256;
          slot[half * 128 + r] = mine;
          asm volatile("bar.sync %0, 64;" ::"r"(1 + wq) : "memory");
          return slot[r] + slot[128 + r];
        };
        // QM: a row may see no active key in its unit's first tiles (its
        // quadrants masked); the reference max is taken from the first tile
        // that has one (until then O and l stay zero).
        if (j == 0 || (QM && __any_sync(0xFFFFFFFFu, m == -INFINITY))) {
          float a = S(0);
#pragma unroll
          for (int i = 1; i < 63; i += 2) a = fmaxf(a, fmaxf(S(i), S(i + 1)));
          const float mx = exchange_max(fmaxf(a, S(63)) + dlt);
          m = (m == -INFINITY) ? mx : m;
          if (p.kmax_head) {
            // s = q.k <= |q||k| <= |q| max_t |k_t|: if that bound is within
            // 2^64 of the first block's max (the reference m only grows),
            // no exponential of this unit can overflow, and rescaling may
            // be decided two steps late from the halves' block sums, which
            // needs no per-step exchange.  Inputs are the same in both
            // halves (m exchanged, |q|^2 halves in shared memory), so both
            // take the same decision.
            const int qb = ord & 1;
            const float qq = red_qn[(qb * 2) * 128 + r] + red_qn[(qb * 2 + 1) * 128 + r];
            const float bound = sqrtf(qq) * __ldg(p.kmax_head + h) * 1.001f + 1e-3f;
            lag = __all_sync(0xFFFFFFFFu, (bound - m) * sl2 < 64.0f);
          }
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
          const float nb = (QM && mref == -INFINITY) ? -INFINITY : (dlt - mref) * sl2;
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
        // O must hold P(g-1).V(g-1) before a rescale
        auto rescale_o = [&](float alpha) {
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
        };
        if (lag) {
          // Lagged rebase: step j-2's block sums (own + partner's, both
          // written before their P(g-2) arrive; S(g) was issued after P(g-2).V,
          // so that barrier phase is complete and this wait acquires them)
          // bound that block's exponentials; if the row's exceeded 2^8,
          // rebase O, l and m by it before this step's exponentials.  Sums
          // from before the last rebase are stale and skipped.
          if (j >= 2 && j - 2 >= last_rebase) {
            mbar_wait(&p_full[(g - 2) & 1], ((g - 2) >> 1) & 1);
            const float T = own2 + red_lag[(((g - 2) & 3) * 2 + (half ^ 1)) * 128 + r];
            const bool need = !(T <= 256.0f);
            if (__any_sync(0xFFFFFFFFu, need)) {
              const float lt = need ? __log2f(T) : 0.f;
              const float alpha = need ? ex2(-lt) : 1.0f;
              if (need) {
                m += lt / sl2;
                l *= alpha;
              }
              rescale_o(alpha);
              last_rebase = j;
            }
          }
          exps(m, false);
          const float2 at0 = fadd2(acc[0], acc[1]);
          own2 = own1;
          own1 = at0.x + at0.y;
          red_lag[((g & 3) * 2 + half) * 128 + r] = own1;
        } else {
        exps(m, false);
        // Rescale guard without a per-element max: if this block's
        // exponentials (against the stale reference m) sum to <= 2^8 over the
        // row, every one of them is <= 2^8, i.e. the block's max is within
        // 2^8 of m and no rescale is due.  Only otherwise (rare after the
        // first blocks) is the block max computed and exchanged, and O / l
        // rebased when it overtook m by more than 2^8 (exact either way).
        // Both halves see the same row sum, so they take the same branch.
        const float2 at0 = fadd2(acc[0], acc[1]);
        const float tot = j > 0 ? exchange_sum(at0.x + at0.y) : 0.f;
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
            rescale_o(alpha);
            exps(m, false);
          }
        }
        }
        if (tr) RP_TR2(11, g);
        const float2 at = fadd2(acc[0], acc[1]);
        l += at.x + at.y;
        tmem_st32(trow + sb + 32 * half, pk);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[b]);
        if (tr) RP_TR2(2, g);
      }
      // the next unit's Q goes to TMEM before this unit's epilogue: the MMA
      // warp issues the next unit's first S ahead of this unit's last P.V
      if (next_nonempty(u + gridDim.x) < p.n_units) q_to_tmem(ord + 1);
      // epilogue: wait for the unit's last P.V, combine the halves' sums,
      // O / l -> bf16 -> global (this half's D/2 columns)
      red_l[half * 128 + r] = l;
      mbar_wait(o_done, ord & 1);
      tc_fence_after();
      asm volatile("bar.sync %0, 64;" ::"r"(1 + wq) : "memory");
      const float lsum = red_l[r] + red_l[128 + r];
      // QM: a row with no active key anywhere (the reference's domain_error,
      // flagged from the 64-block CSR) is written as zeros
      const float inv = QM ? (lsum > 0.f ? 1.0f / lsum : 0.f) : 1.0f / lsum;
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        uint32_t o[32];
        tmem_ld32(trow + L::kO + half * (D / 2) + c * 32, o);
        tmem_wait_ld();
        uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
        if (!row_out) continue;
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
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace attn2
}  // namespace rp
