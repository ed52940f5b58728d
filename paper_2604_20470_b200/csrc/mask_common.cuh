// Device helpers shared by the mask builder kernels (mask_build.cu) and the
// tensor-core scoring engine (mask_score_sm100.cu).
#pragma once

#include "common.cuh"
#include "mask_build.cuh"

namespace rp {
namespace mask {

// ------------------------------------------------------------ helpers -----
RP_DEV void set_block(uint32_t* words, int64_t row_bytes, int64_t r, int64_t c) {
  const int64_t byte = r * row_bytes + c / 8;
  atomicOr(&words[byte >> 2], 1u << (((byte & 3) << 3) + (c & 7)));
}

// Offsets of the canonical row-major band enumeration (radial.cpp:64-79) in
// closed form: off(u) = sum_{x<u} (min(N-1, x+w) - max(0, x-w) + 1).
RP_HD int64_t band_off(int64_t u, int64_t N, int64_t w) {
  int64_t a = N - w;
  if (a < 0) a = 0;
  if (a > u) a = u;
  const int64_t hi = a * (a - 1) / 2 + a * w + (u - a) * (N - 1);
  int64_t c = u - 1 - w;
  if (c < 0) c = 0;
  return hi - c * (c + 1) / 2 + u;
}
// Flat index -> (u, v): largest u with off(u) <= flat (upper_bound - 1),
// searched in [lo, hi) (off(lo) <= flat < off(hi); default the whole band).
// The same offsets in 32-bit arithmetic: exact while N^2 < 2^31 (N <= 46340;
// w is clamped to N, which leaves off(u) unchanged).
RP_HD int32_t band_off32(int32_t u, int32_t N, int32_t w) {
  int32_t a = N - w;
  if (a < 0) a = 0;
  if (a > u) a = u;
  const int32_t hi = a * (a - 1) / 2 + a * w + (u - a) * (N - 1);
  int32_t c = u - 1 - w;
  if (c < 0) c = 0;
  return hi - c * (c + 1) / 2 + u;
}
RP_HD void band_uv(int64_t flat, int64_t N, int64_t w, int64_t* u, int64_t* v, int64_t lo = 0,
                   int64_t hi = -1) {
  if (hi < 0 || hi > N) hi = N;
  if (N <= 46340) {  // frame sizes in practice: the search in 32-bit arithmetic
    const int32_t n32 = static_cast<int32_t>(N);
    const int32_t w32 = static_cast<int32_t>(w < N ? w : N);
    const int32_t f32 = static_cast<int32_t>(flat);
    int32_t l32 = static_cast<int32_t>(lo), h32 = static_cast<int32_t>(hi);
    while (h32 - l32 > 1) {
      const int32_t mid = (l32 + h32) >> 1;
      if (band_off32(mid, n32, w32) <= f32) l32 = mid; else h32 = mid;
    }
    *u = l32;
    *v = (l32 - w32 > 0 ? l32 - w32 : 0) + (f32 - band_off32(l32, n32, w32));
    return;
  }
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (band_off(mid, N, w) <= flat) lo = mid; else hi = mid;
  }
  *u = lo;
  *v = (lo - w > 0 ? lo - w : 0) + (flat - band_off(lo, N, w));
}

RP_DEV void add_count(const DJob& jb, uint32_t* counts, int64_t nt, int bs, int64_t u,
                      int64_t v) {
  const int64_t gr = static_cast<int64_t>(jb.i) * nt + u;
  const int64_t gc = static_cast<int64_t>(jb.j) * nt + v;
  const int64_t rr = gr / bs - jb.r0, cc = gc / bs - jb.c0;
  atomicAdd(&counts[jb.cnt_off + (rr * jb.tc + cc) * bs + gc % bs], 1u);
}

RP_DEV int find_job(const int64_t* __restrict__ off, int n_jobs, int64_t x) {
  int lo = 0, hi = n_jobs;  // off[lo] <= x < off[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (off[mid] <= x) lo = mid; else hi = mid;
  }
  return lo;
}

struct Feat {
  const void* q;
  const void* k;
  int dtype;
  int64_t q_ts, q_hs, k_ts, k_hs;
  int heads, d;
  double inv_sqrt_d;
};

RP_DEV float feat_at(const void* p, int dtype, int64_t idx) {
  return dtype == RP_BF16 ? __bfloat162float(static_cast<const __nv_bfloat16*>(p)[idx])
                          : static_cast<const float*>(p)[idx];
}

// selection.cpp:104-121: per-head dot in double (ascending d), acc +=
// dot * inv_sqrt_d (no contraction), float(acc / heads).  bf16 rows that are
// 16-byte aligned are read 8 values per load; the accumulation order is the
// reference's either way.
RP_DEV float exact_score(const Feat& f, int64_t qrow, int64_t krow) {
  double acc = 0.0;
  for (int h = 0; h < f.heads; ++h) {
    const int64_t qb = qrow * f.q_ts + h * f.q_hs, kb = krow * f.k_ts + h * f.k_hs;
    double dot = 0.0;
    if (f.dtype == RP_BF16 && ((qb | kb | f.d) & 7) == 0) {
      const uint4* qv = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(f.q) + qb);
      const uint4* kv = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(f.k) + kb);
      for (int e = 0; e < f.d / 8; ++e) {
        const uint4 a = __ldg(qv + e), b = __ldg(kv + e);
        const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          dot = __fma_rn(static_cast<double>(__uint_as_float(aw[t] << 16)),
                         static_cast<double>(__uint_as_float(bw[t] << 16)), dot);
          dot = __fma_rn(static_cast<double>(__uint_as_float(aw[t] & 0xFFFF0000u)),
                         static_cast<double>(__uint_as_float(bw[t] & 0xFFFF0000u)), dot);
        }
      }
    } else if (f.dtype == RP_F32 && ((qb | kb | f.d) & 3) == 0) {
      const float4* qv = reinterpret_cast<const float4*>(static_cast<const float*>(f.q) + qb);
      const float4* kv = reinterpret_cast<const float4*>(static_cast<const float*>(f.k) + kb);
      for (int e = 0; e < f.d / 4; ++e) {
        const float4 a = __ldg(qv + e), b = __ldg(kv + e);
        dot = __fma_rn(static_cast<double>(a.x), static_cast<double>(b.x), dot);
        dot = __fma_rn(static_cast<double>(a.y), static_cast<double>(b.y), dot);
        dot = __fma_rn(static_cast<double>(a.z), static_cast<double>(b.z), dot);
        dot = __fma_rn(static_cast<double>(a.w), static_cast<double>(b.w), dot);
      }
    } else {
      for (int e = 0; e < f.d; ++e)
        dot = __fma_rn(static_cast<double>(feat_at(f.q, f.dtype, qb + e)),
                       static_cast<double>(feat_at(f.k, f.dtype, kb + e)), dot);
    }
    acc = __dadd_rn(acc, __dmul_rn(dot, f.inv_sqrt_d));
  }
  return __double2float_rn(__ddiv_rn(acc, static_cast<double>(f.heads)));
}

RP_DEV double zscore(float s, double2 st) {
  return __ddiv_rn(__dsub_rn(static_cast<double>(s), st.x), __dadd_rn(st.y, 1e-8));
}

// Per (job, tile) item with B (<= 1024) threads: one column each.
// mode 0: closed-form full-band counts; mode 1: counts from a buffer.
static __global__ void apply_kernel(const DJob* __restrict__ jobs, const Item* __restrict__ items,
                             const uint32_t* __restrict__ counts, uint32_t* words, int64_t nt,
                             int bs, int64_t row_bytes, int cmin, int amin, int mode) {
  const Item it = items[blockIdx.x];
  const DJob& jb = jobs[it.job];
  __shared__ int active;
  if (threadIdx.x == 0) active = 0;
  __syncthreads();
  int mine = 0;
  for (int k = threadIdx.x; k < bs; k += blockDim.x) {
    uint32_t cnt = 0;
    if (mode == 0) {
      // mask.cpp:132-158: column v of frame j hit by rows [v-w, v+w] of frame i
      const int64_t qi = static_cast<int64_t>(jb.i) * nt, kj = static_cast<int64_t>(jb.j) * nt;
      const int64_t gc = (jb.c0 + it.tc) * bs + k;
      const int64_t lv = gc - kj;
      if (lv >= 0 && lv < nt) {
        const int64_t ulo = lv - jb.width > 0 ? lv - jb.width : 0;
        const int64_t uhi = lv + jb.width < nt - 1 ? lv + jb.width : nt - 1;
        const int64_t R0 = (jb.r0 + it.tr) * bs, R1 = R0 + bs - 1;
        const int64_t lo = qi + ulo > R0 ? qi + ulo : R0;
        const int64_t hi = qi + uhi < R1 ? qi + uhi : R1;
        if (ulo <= uhi && lo <= hi) cnt = static_cast<uint32_t>(hi - lo + 1);
      }
    } else {
      cnt = counts[jb.cnt_off + (static_cast<int64_t>(it.tr) * jb.tc + it.tc) * bs + k];
    }
    mine += cnt >= static_cast<uint32_t>(cmin);
  }
  if (mine) atomicAdd(&active, mine);
  __syncthreads();
  if (threadIdx.x == 0 && active >= amin)
    set_block(words, row_bytes, jb.r0 + it.tr, jb.c0 + it.tc);
}

}  // namespace mask
}  // namespace rp
