// Test support: a one-CTA probe that pins the UMMA descriptor conventions
// (K-major SS MMA and TMEM-A / MN-major-B MMA, operands staged in the 128B
// swizzled layout TMA produces) independently of TMA; tests/test_attention_gpu.py
// checks it against torch.  (The first stage-(d) design, two heads of one
// block row ping-ponging on the tensor core, lived here; it was superseded by
// attn_sm100_db.cu and removed -- DESIGN.md section 8 keeps its numbers.)
#include "common.cuh"

namespace rp {
namespace attn {

// --------------------------------------------------------------------------
// Descriptor probe (test support): one CTA computes C1 = A . B^T (both
// K-major, SS) and C2 = P . V (P from TMEM, V MN-major) with operands staged
// by plain stores in the same 128B-swizzled layout TMA produces.  Used by the
// GPU tests to pin the UMMA descriptor conventions independently of TMA.
__global__ void __launch_bounds__(128, 1)
    umma_probe_kernel(const __nv_bfloat16* A, const __nv_bfloat16* B,
                      const __nv_bfloat16* P, const __nv_bfloat16* V, float* C1,
                      float* C2) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + 32768;
  uint8_t* sv = smem + 65536;
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int t = threadIdx.x;
  // K-major / MN-major share the physical pattern: row r (128 B per chunk),
  // 16-byte unit XOR (r % 8), chunk c at c * 128 rows * 128 B.
  auto put = [](uint8_t* base, int r, int col, __nv_bfloat16 val) {
    const int chunk = col / 64, b = (col % 64) * 2;
    const int off = chunk * 16384 + r * 128 + (((b / 16) ^ (r % 8)) * 16) + b % 16;
    *reinterpret_cast<__nv_bfloat16*>(base + off) = val;
  };
  for (int i = t; i < 128 * 128; i += 128) {
    const int r = i / 128, c = i % 128;
    put(sa, r, c, A[i]);
    put(sb, r, c, B[i]);
    put(sv, r, c, V[i]);  // row = key, col = d
  }
  if (t == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (t < 32) tmem_alloc<512>(&slot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t idesc_qk = idesc_bf16(128, 128, false, false);
  const uint32_t idesc_pv = idesc_bf16(128, 128, false, true);
  if (t == 0) {
    for (int kk = 0; kk < 8; ++kk) {
      const uint32_t off = (kk / 4) * 16384 + (kk % 4) * 32;
      umma_ss(tmem, smem_desc_sw128(smem_u32(sa) + off, 0, 1024),
              smem_desc_sw128(smem_u32(sb) + off, 0, 1024), idesc_qk, kk > 0);
    }
    umma_commit(&bar);
  }
  // P rows into TMEM columns 256.. (packed bf16 pairs)
  {
    const int wq = t / 32;
    const uint32_t trow = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    uint32_t pk[32];
    for (int half = 0; half < 2; ++half) {
      for (int i = 0; i < 32; ++i) {
        const int k0 = half * 64 + 2 * i;
        __nv_bfloat162 v2;
        v2.x = P[t * 128 + k0];
        v2.y = P[t * 128 + k0 + 1];
        pk[i] = *reinterpret_cast<uint32_t*>(&v2);
      }
      tmem_st32(trow + 256 + half * 32, pk);
    }
    tmem_wait_st();
  }
  mbar_wait(&bar, 0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (t == 0) {
    for (int kk = 0; kk < 8; ++kk)
      umma_ts(tmem + 128, tmem + 256 + kk * 8,
              smem_desc_sw128(smem_u32(sv) + kk * 16 * 128, 16384, 1024), idesc_pv,
              kk > 0);
    umma_commit(&bar);
  }
  mbar_wait(&bar, 1);
  tc_fence_after();
  {
    const int wq = t / 32;
    const uint32_t trow = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    for (int c = 0; c < 8; ++c) {
      uint32_t o[32];
      tmem_ld32(trow + c * 32, o);
      tmem_wait_ld();
      float* dst = c < 4 ? C1 + t * 128 + c * 32 : C2 + t * 128 + (c - 4) * 32;
      for (int i = 0; i < 32; ++i) dst[i] = __uint_as_float(o[i]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (t < 32) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace attn
}  // namespace rp
