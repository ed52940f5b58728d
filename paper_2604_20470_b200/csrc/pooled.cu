// the north star's pooled block selector -- stages (b)/(c) as
// BASELINE.json's north_star words them, NOT the reference's semantics (the
// reference scores every token pair of the radial band, selection.cpp:93-185;
// its exact form is the build_mask path in mask_build.cu / mask_score_sm100.cu).
// Its oracle is a CPU restatement in tests/test_pooled_gpu.py (parity against
// the reference is not defined for it).
//
//   classify  block (r, c): forced when it holds a token pair of frames at
//             distance t <= 1 (the reference's tier 0: intra-frame
//             rectangles and full adjacent bands), candidate when it meets
//             the radial band |u - v| <= w(i, j) of a retained frame pair at
//             t >= 2 (radial.cpp:30-54 windows and split rule).
//   pool      block means of the first H_f heads of Q and K over each block's
//             valid tokens: one pass over 2 S H_f d bf16 -- HBM-bound,
//             128-bit loads, fp32 accumulation, shared-memory reduction.
//   scores    s(r, c) = Qp_r . Kp_c / sqrt(d) / H_f for all block pairs as one
//             tiled fp32 GEMM (64 x 64 tiles staged in shared memory, so each
//             pooled key row is read from L2 once per 64 query rows instead of
//             once per row: 1.7 GB -> 0.1 GB of L2 traffic at Hunyuan);
//   select    one CTA per block row: the row's candidate scores, a
//             bitonic sort (score descending, column ascending on ties), then
//             static-ratio top-k (keep max(1, floor(ratio n)) best) or
//             dynamic cumulative softmax mass (smallest prefix whose softmax
//             mass over the candidates reaches tau), and the row's bits.
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "internal.hpp"
#include "plan.hpp"

namespace rp {
namespace pooled {

constexpr int kMaxFeat = 512;  // H_f * d

struct Dist {
  int32_t width;
  int32_t retained;  // frame pair at this distance survives the split rule
};

// 0 none, 1 candidate, 2 forced (32-bit index arithmetic: S < 2^31)
__global__ void classify_kernel(const Dist* __restrict__ tab, int nf, int64_t nt64, int64_t S64,
                                int bs, int64_t nb, uint8_t* __restrict__ state) {
  const int nt = static_cast<int>(nt64), S = static_cast<int>(S64);
  const int r = blockIdx.y;
  const int t0 = r * bs, t1 = min(t0 + bs, S);  // valid query tokens [t0, t1)
  const int fi0 = t0 / nt, fi1 = (t1 - 1) / nt;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nb; c += gridDim.x * blockDim.x) {
    const int k0 = c * bs, k1 = min(k0 + bs, S);
    uint8_t st = 0;
    if (t0 < t1 && k0 < k1) {
      const int fj0 = k0 / nt, fj1 = (k1 - 1) / nt;
      for (int fi = fi0; fi <= fi1; ++fi) {
        const int ua = max(t0, fi * nt) - fi * nt, ub = min(t1 - 1, fi * nt + nt - 1) - fi * nt;
        for (int fj = fj0; fj <= fj1; ++fj) {
          const int va = max(k0, fj * nt) - fj * nt, vb = min(k1 - 1, fj * nt + nt - 1) - fj * nt;
          const int t = fi > fj ? fi - fj : fj - fi;
          if (t <= 1) {
            st = 2;
          } else {
            const Dist dt = tab[t];
            if (dt.retained && !(va - ub > dt.width || ua - vb > dt.width) && st == 0) st = 1;
          }
        }
      }
    }
    state[static_cast<int64_t>(r) * nb + c] = st;
  }
}

// Block means of the first `heads` heads (H_f * d <= 512 values per token).
// blockIdx.x = block, blockIdx.y = 0 (Q) / 1 (K).  256 threads: 32 chunks of
// 8 values (one 16-byte load each) x 8 token groups.
__global__ void __launch_bounds__(256) pool_kernel(const __nv_bfloat16* __restrict__ q,
                                                   const __nv_bfloat16* __restrict__ k,
                                                   int64_t ts, int64_t hs, int heads, int d,
                                                   int64_t S, int bs, float* __restrict__ qp,
                                                   float* __restrict__ kp) {
  const __nv_bfloat16* x = blockIdx.y ? k : q;
  float* out = blockIdx.y ? kp : qp;
  const int64_t b = blockIdx.x;
  const int64_t t0 = b * bs, t1 = min(t0 + bs, S);
  const int F = heads * d, chunks = F / 8;
  __shared__ float red[8][kMaxFeat];
  const int grp = threadIdx.x / 32;
  for (int ch = threadIdx.x % 32; ch < chunks; ch += 32) {
    const int h = (ch * 8) / d, e = (ch * 8) % d;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    // four independent 16-byte loads in flight per thread (memory-level
    // parallelism for the HBM stream); fp32 sums in token order per lane
    int64_t t = t0 + grp;
    for (; t + 24 < t1; t += 32) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        v[u] = __ldg(reinterpret_cast<const uint4*>(x + (t + 8 * u) * ts + h * hs + e));
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          acc[2 * i] += __uint_as_float(w[i] << 16);
          acc[2 * i + 1] += __uint_as_float(w[i] & 0xFFFF0000u);
        }
      }
    }
    for (; t < t1; t += 8) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(x + t * ts + h * hs + e));
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[2 * i] += __uint_as_float(w[i] << 16);
        acc[2 * i + 1] += __uint_as_float(w[i] & 0xFFFF0000u);
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) red[grp][ch * 8 + i] = acc[i];
  }
  __syncthreads();
  const float inv = t1 > t0 ? 1.f / static_cast<float>(t1 - t0) : 0.f;
  for (int f = threadIdx.x; f < F; f += blockDim.x) {
    float s = 0.f;
#pragma unroll
    for (int g = 0; g < 8; ++g) s += red[g][f];
    out[b * F + f] = s * inv;
  }
}

// sc[r][c] = scale * Qp_r . Kp_c, 64 x 64 output tiles, 256 threads x 4 x 4
// (measured against 128 x 128 / 8 x 8 and 32 x 32 / 64-thread tiles: the
// middle size is fastest at both the Wan and the Hunyuan block counts).
constexpr int kT = 64, kKC = 32, kST = 256;
__global__ void __launch_bounds__(kST) scores_kernel(const float* __restrict__ qp,
                                                     const float* __restrict__ kp, int F,
                                                     int64_t nb, float scale,
                                                     float* __restrict__ sc) {
  __shared__ __align__(16) float fa[kKC][kT + 4];
  __shared__ __align__(16) float fb[kKC][kT + 4];
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * kT, c0 = static_cast<int64_t>(blockIdx.x) * kT;
  const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < F; k0 += kKC) {
    __syncthreads();
    for (int idx = tid; idx < kT * kKC; idx += kST) {
      const int row = idx / kKC, kk = idx % kKC;
      const bool in = k0 + kk < F;
      fa[kk][row] = in && r0 + row < nb ? qp[(r0 + row) * F + k0 + kk] : 0.f;
      fb[kk][row] = in && c0 + row < nb ? kp[(c0 + row) * F + k0 + kk] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < kKC; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(&fa[kk][4 * ty]);
      const float4 b = *reinterpret_cast<const float4*>(&fb[kk][4 * tx]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = r0 + 4 * ty + i;
    if (r >= nb) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t c = c0 + 4 * tx + j;
      if (c < nb) sc[r * nb + c] = acc[i][j] * scale;
    }
  }
}

// One CTA (256 threads) per block row.  Dynamic shared memory: cap (score,
// column) pairs (cap a power of two >= the block count) and one flag byte per
// column.  Candidates are compacted with warp ballots + a block scan (no
// shared-memory atomics: a single counter serialised ~1000 atomics per row),
// the bitonic sort runs over the next power of two >= the candidate count,
// and the row's words come from warp ballots (warp w of a pass owns 32
// aligned columns).
__global__ void __launch_bounds__(256) select_kernel(const float* __restrict__ scores,
                                                     const uint8_t* __restrict__ state,
                                                     int64_t nb, int64_t row_bytes, int cap,
                                                     int mode, double param,
                                                     uint8_t* __restrict__ bits) {
  extern __shared__ float sm[];
  float* sc = sm;                                     // [cap]
  int* ci = reinterpret_cast<int*>(sc + cap);         // [cap]
  uint8_t* flag = reinterpret_cast<uint8_t*>(ci + cap);  // [cap]: 2 forced, 1 kept
  __shared__ int wsum[8];
  __shared__ int n_keep;
  __shared__ double red_total;
  const int64_t r = blockIdx.x;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const float* srow = scores + r * nb;
  const uint8_t* strow = state + r * nb;
  // 1. compaction of the candidates in column order
  int n = 0;
  for (int64_t base = 0; base < nb; base += blockDim.x) {
    const int64_t c = base + threadIdx.x;
    const uint8_t st = c < nb ? strow[c] : 0;
    if (c < nb) flag[c] = st == 2 ? 2 : 0;
    const bool cand = st == 1;
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, cand);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    int off = n;
    for (int w = 0; w < warp; ++w) off += wsum[w];
    int tot = 0;
    for (int w = 0; w < 8; ++w) tot += wsum[w];
    if (cand) {
      const int at = off + __popc(bal & ((1u << lane) - 1u));
      sc[at] = srow[c];
      ci[at] = static_cast<int>(c);
    }
    n += tot;
    __syncthreads();
  }
  int cp = 1;
  while (cp < n) cp <<= 1;
  for (int i = n + threadIdx.x; i < cp; i += blockDim.x) {
    sc[i] = -INFINITY;
    ci[i] = 0x7FFFFFFF;
  }
  __syncthreads();
  // 2. bitonic sort: score descending, column ascending
  for (int size = 2; size <= cp; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < cp / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool desc = (lo & size) == 0;
        const float a = sc[lo], bb = sc[hi];
        const int ia = ci[lo], ib = ci[hi];
        const bool a_first = a > bb || (a == bb && ia < ib);
        if (a_first != desc) {
          sc[lo] = bb;
          sc[hi] = a;
          ci[lo] = ib;
          ci[hi] = ia;
        }
      }
      __syncthreads();
    }
  }
  // 3. how many of the best to keep
  if (mode == RP_POOLED_TOPK) {
    if (threadIdx.x == 0) {
      int keep = n > 0 ? static_cast<int>(floor(static_cast<double>(n) * param)) : 0;
      n_keep = n > 0 && keep < 1 ? 1 : keep;
    }
  } else {
    // smallest best-first prefix whose softmax mass reaches param: weights
    // in fp64, a segmented block scan (thread t owns a contiguous segment)
    __shared__ double seg[256];
    const int per = (n + blockDim.x - 1) / blockDim.x;
    const int b0 = threadIdx.x * per, b1 = min(n, b0 + per);
    const double mx = n > 0 ? static_cast<double>(sc[0]) : 0.0;
    double part = 0.0;
    for (int i = b0; i < b1; ++i) part += exp(static_cast<double>(sc[i]) - mx);
    seg[threadIdx.x] = part;
    if (threadIdx.x == 0) n_keep = n;
    __syncthreads();
    if (threadIdx.x == 0) {  // 256 segment sums: sequential exclusive scan
      double run = 0.0;
      for (int t = 0; t < static_cast<int>(blockDim.x); ++t) {
        const double v = seg[t];
        seg[t] = run;
        run += v;
      }
      red_total = run;
    }
    __syncthreads();
    const double target = param * red_total;
    double run = seg[threadIdx.x];
    for (int i = b0; i < b1; ++i) {
      run += exp(static_cast<double>(sc[i]) - mx);
      if (run >= target) {
        atomicMin(&n_keep, i + 1);
        break;
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n_keep; i += blockDim.x) flag[ci[i]] = 1;
  __syncthreads();
  // 4. the row's bits: one ballot per 32 aligned columns
  uint8_t* row = bits + r * row_bytes;
  for (int64_t base = 32 * warp; base < 8 * row_bytes; base += blockDim.x) {
    const int64_t c = base + lane;
    const uint32_t w = __ballot_sync(0xFFFFFFFFu, c < nb && flag[c] != 0);
    const int64_t byte0 = base / 8 + lane;  // lanes 0-3 store the word's bytes
    if (lane < 4 && byte0 < row_bytes) row[byte0] = static_cast<uint8_t>(w >> (8 * lane));
  }
}

}  // namespace pooled
}  // namespace rp

using namespace rp;

extern "C" {

rp_status rp_pooled_select(const rp_grid* g, const rp_config* c, const rp_tensor* q,
                           const rp_tensor* k, int n_score_heads, int mode, double param,
                           uint8_t* mask_bits_dev, rp_stream stream) {
  return guarded([&] {
    require_device();
    check_grid(g);
    if (!c) throw std::invalid_argument("config: null");
    if (!q || !k || !q->data || !k->data || q->dtype != RP_BF16 || k->dtype != RP_BF16)
      throw std::invalid_argument("pooled select: bf16 features required");
    if (n_score_heads < 1 || n_score_heads > q->heads || q->heads != k->heads ||
        q->head_dim != k->head_dim || q->head_stride != k->head_stride ||
        q->token_stride != k->token_stride)
      throw std::invalid_argument("feature batch: queries/keys shape mismatch");
    const int F = n_score_heads * q->head_dim;
    if (F > pooled::kMaxFeat || q->head_dim % 8 || q->head_stride % 8 || q->token_stride % 8)
      throw std::invalid_argument("pooled select: H_f * d <= 512, 16-byte aligned rows");
    if (q->tokens < g->total_tokens || k->tokens < g->total_tokens)
      throw std::invalid_argument("build_mask: feature batch too short");
    if (mode == RP_POOLED_TOPK ? !(param > 0.0 && param <= 1.0) : !(param > 0.0 && param <= 1.0))
      throw std::invalid_argument("pooled select: ratio / mass must be in (0, 1]");
    if (mode != RP_POOLED_TOPK && mode != RP_POOLED_MASS)
      throw std::invalid_argument("pooled select: unknown mode");
    if (!mask_bits_dev) throw std::invalid_argument("build_mask: null mask buffer");
    if (g->padded_tokens >= (int64_t{1} << 31))
      throw std::invalid_argument("pooled select: more than 2^31 tokens");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t nb = g->blocks_per_dim;
    int cap = 2;
    while (cap < nb) cap <<= 1;
    const size_t smem = static_cast<size_t>(cap) * 9;
    if (smem > 200 * 1024) throw std::invalid_argument("pooled select: grid too large");
    // per-distance window and split decisions (radial.cpp:30-54)
    std::vector<pooled::Dist> tab(static_cast<size_t>(g->n_frames));
    for (int t = 0; t < g->n_frames; ++t) {
      tab[t].width = static_cast<int32_t>(plan::window_width(0, t, *c, *g));
      tab[t].retained = plan::frame_retained(t, *c, *g) ? 1 : 0;
    }
    pooled::Dist* d_tab = nullptr;
    uint8_t* d_state = nullptr;
    float *d_qp = nullptr, *d_kp = nullptr, *d_sc = nullptr;
    RP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_tab), sizeof(pooled::Dist) * tab.size(), s));
    RP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_state), static_cast<size_t>(nb * nb), s));
    RP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_qp), sizeof(float) * nb * F, s));
    RP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_kp), sizeof(float) * nb * F, s));
    RP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_sc), sizeof(float) * nb * nb, s));
    RP_CUDA(cudaMemcpyAsync(d_tab, tab.data(), sizeof(pooled::Dist) * tab.size(),
                            cudaMemcpyHostToDevice, s));
    pooled::classify_kernel<<<dim3(static_cast<unsigned>((nb + 255) / 256),
                                   static_cast<unsigned>(nb)), 256, 0, s>>>(
        d_tab, g->n_frames, g->tokens_per_frame, g->total_tokens, g->block_size, nb, d_state);
    RP_LAUNCHED();
    pooled::pool_kernel<<<dim3(static_cast<unsigned>(nb), 2), 256, 0, s>>>(
        static_cast<const __nv_bfloat16*>(q->data), static_cast<const __nv_bfloat16*>(k->data),
        q->token_stride, q->head_stride, n_score_heads, q->head_dim, g->total_tokens,
        g->block_size, d_qp, d_kp);
    RP_LAUNCHED();
    prepare_kernel(reinterpret_cast<const void*>(pooled::select_kernel), 200 * 1024);
    const float scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(q->head_dim)) /
                                           n_score_heads);
    const unsigned tiles = static_cast<unsigned>((nb + pooled::kT - 1) / pooled::kT);
    pooled::scores_kernel<<<dim3(tiles, tiles), pooled::kST, 0, s>>>(d_qp, d_kp, F, nb, scale,
                                                                      d_sc);
    RP_LAUNCHED();
    pooled::select_kernel<<<static_cast<unsigned>(nb), 256, smem, s>>>(
        d_sc, d_state, nb, g->row_bytes, cap, mode, param, mask_bits_dev);
    RP_LAUNCHED();
    RP_CUDA(cudaFreeAsync(d_tab, s));
    RP_CUDA(cudaFreeAsync(d_state, s));
    RP_CUDA(cudaFreeAsync(d_qp, s));
    RP_CUDA(cudaFreeAsync(d_kp, s));
    RP_CUDA(cudaFreeAsync(d_sc, s));
  });
}

rp_status rp_block_mean_pool(const rp_grid* g, const rp_tensor* x, int n_heads, float* out_dev,
                             rp_stream stream) {
  return guarded([&] {
    require_device();
    check_grid(g);
    if (!x || !x->data || x->dtype != RP_BF16)
      throw std::invalid_argument("block mean pool: bf16 features required");
    if (n_heads < 1 || n_heads > x->heads)
      throw std::invalid_argument("block mean pool: n_heads out of range");
    const int F = n_heads * x->head_dim;
    if (F > pooled::kMaxFeat || x->head_dim % 8 || x->head_stride % 8 || x->token_stride % 8)
      throw std::invalid_argument("pooled select: H_f * d <= 512, 16-byte aligned rows");
    if (x->tokens < g->total_tokens)
      throw std::invalid_argument("build_mask: feature batch too short");
    if (!out_dev) throw std::invalid_argument("block mean pool: null output");
    const __nv_bfloat16* p = static_cast<const __nv_bfloat16*>(x->data);
    pooled::pool_kernel<<<dim3(static_cast<unsigned>(g->blocks_per_dim), 1), 256, 0,
                          reinterpret_cast<cudaStream_t>(stream)>>>(
        p, nullptr, x->token_stride, x->head_stride, n_heads, x->head_dim, g->total_tokens,
        g->block_size, out_dev, nullptr);  // gridDim.y = 1: only the Q side
    RP_LAUNCHED();
  });
}

}  // extern "C"

