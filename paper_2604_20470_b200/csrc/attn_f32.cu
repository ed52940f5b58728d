// K6f: exact-precision block-sparse attention (fp32 inputs), any block size.
//
// Follows masked_attention_exact (attention.cpp:50-121) arithmetic: logits
// are an fp32 dot product (the reference's float GEMM), scaled in double;
// softmax is two-pass in double (row max, then exp(l - max), sum and P.V in
// double); output = float(acc / sum).  Padding rows (token >= S) of Q/K/V
// are zero and padded keys count whenever their block is active.  Used for
// the fp32 parity configs (tolerance 1e-5); the bf16 tensor-core kernel is
// the performance path.
#include "common.cuh"

namespace rp {
namespace attn32 {

constexpr int kRows = 32;     // query rows per CTA
constexpr int kKeys = 16;     // keys per smem tile
constexpr int kThreads = 128; // 4 threads per query row
constexpr int kMaxD = 128;

struct Params {
  const float* q;
  const float* k;
  const float* v;
  float* out;
  long long q_ts, q_hs, k_ts, k_hs, v_ts, v_hs, o_ts, o_hs;  // strides (elements)
  long long tokens;  // S (rows >= S are zero padding)
  long long padded;  // S'
  int block;         // B
  int heads, d;
  const int32_t* row_ptr;
  const int32_t* col_idx;
  double scale;
  int* error_flag;   // set to 1 on an empty row (domain_error)
  // Soft mask (masked_attention, attention.cpp:59-81; null = exact): dense
  // row lists, logit + log1p(eps) on active blocks, + log(eps) elsewhere.
  const uint8_t* soft_bits;
  long long soft_row_bytes;
  double log_active, log_inactive;
};

__global__ void __launch_bounds__(kThreads)
    attn_f32_kernel(const Params p) {
  __shared__ float sq[kRows][kMaxD + 1];
  __shared__ float sk[kKeys][kMaxD + 1];
  __shared__ float sv[kKeys][kMaxD + 1];
  __shared__ double sp[kRows][kKeys + 1];
  __shared__ double smax[kRows][4];

  const int h = blockIdx.y;
  const long long r0 = static_cast<long long>(blockIdx.x) * kRows;
  const int t = threadIdx.x;
  const int r = t / 4, sub = t % 4;
  const int d = p.d;
  const long long row = r0 + r;

  for (int i = t; i < kRows * d; i += kThreads) {
    const int rr = i / d, e = i % d;
    const long long tok = r0 + rr;
    sq[rr][e] = tok < p.tokens ? p.q[tok * p.q_ts + h * p.q_hs + e] : 0.f;
  }
  __syncthreads();

  // All query rows of the CTA lie in block rows [r0/B, (r0+kRows-1)/B]; a
  // CTA never straddles block rows when B >= kRows, and for B < kRows each
  // thread checks its own row's list below.
  const bool row_ok = row < p.padded;
  const long long brow = row_ok ? row / p.block : 0;

  double m = -INFINITY, sum = 0.0;
  double acc[kMaxD / 4];
#pragma unroll
  for (int e = 0; e < kMaxD / 4; ++e) acc[e] = 0.0;

  // Union of the CTA's block rows' lists is walked per distinct block row.
  const long long b_first = r0 / p.block;
  const long long b_last = min(p.padded - 1, r0 + kRows - 1) / p.block;
  for (int pass = 0; pass < 2; ++pass) {
    for (long long br = b_first; br <= b_last; ++br) {
      const int beg = p.row_ptr[br], end = p.row_ptr[br + 1];
      const bool mine = row_ok && br == brow;
      for (int bi = beg; bi < end; ++bi) {
        const int cb = p.col_idx[bi];
        const long long c0 = static_cast<long long>(cb) * p.block;
        double off = 0.0;
        if (p.soft_bits && mine)
          off = ((p.soft_bits[brow * p.soft_row_bytes + (cb >> 3)] >> (cb & 7)) & 1) ? p.log_active
                                                                                  : p.log_inactive;
        for (int k0 = 0; k0 < p.block; k0 += kKeys) {
          const int nk = min(kKeys, p.block - k0);
          __syncthreads();
          for (int i = t; i < nk * d; i += kThreads) {
            const int kk = i / d, e = i % d;
            const long long tok = c0 + k0 + kk;
            const bool real = tok < p.tokens;
            sk[kk][e] = real ? p.k[tok * p.k_ts + h * p.k_hs + e] : 0.f;
            sv[kk][e] = real ? p.v[tok * p.v_ts + h * p.v_hs + e] : 0.f;
          }
          __syncthreads();
          // logits for (r, kk), kk = sub, sub+4, ...
          for (int kk = sub; kk < nk; kk += 4) {
            float lg = 0.f;
            for (int e = 0; e < d; ++e) lg = fmaf(sq[r][e], sk[kk][e], lg);
            const double l = static_cast<double>(lg) * p.scale + off;
            if (pass == 0) {
              if (mine && l > m) m = l;
            } else {
              sp[r][kk] = mine ? exp(l - m) : 0.0;
            }
          }
          if (pass == 1) {
            __syncthreads();
            if (mine) {
              for (int kk = 0; kk < nk; ++kk) {
                const double pk = sp[r][kk];
                if (sub == 0) sum += pk;
                for (int e = sub; e < d; e += 4)
                  acc[e / 4] += pk * static_cast<double>(sv[kk][e]);
              }
            }
          }
        }
      }
    }
    if (pass == 0) {
      smax[r][sub] = m;
      __syncthreads();
      m = fmax(fmax(smax[r][0], smax[r][1]), fmax(smax[r][2], smax[r][3]));
      if (row_ok && m == -INFINITY && sub == 0 && p.error_flag) atomicExch(p.error_flag, 1);
    }
  }
  // sum lives in sub == 0; share it
  __syncthreads();
  if (sub == 0) smax[r][0] = sum;
  __syncthreads();
  sum = smax[r][0];
  if (row_ok && m != -INFINITY) {
    float* o = p.out + row * p.o_ts + h * p.o_hs;
    for (int e = sub; e < d; e += 4) o[e] = static_cast<float>(acc[e / 4] / sum);
  }
}

}  // namespace attn32
}  // namespace rp
