// random_batch (attention.cpp:182-204) on the device: the reference's
// counter-based synthetic features, value (role, h, t, d) =
// float(gaussian_at(mix64(mix64(seed, role, h), t, d))) with role 1/2/3 =
// Q/K/V and gaussian_at the pinned Box-Muller of rng.hpp:84-91.  The double
// log / cos / sqrt of CUDA's libdevice and glibc can differ in the last bit;
// the double -> float rounding absorbs that (and the bf16 rounding of the
// bf16 path all the more), which tests/test_features_gpu.py checks against
// the reference's own values.  Inputs for bench.py and the production-scale
// mask tests, so the benched dynamic mask is the reference's golden mask.
#include "common.cuh"

namespace rp {
namespace feat {

RP_DEV double gaussian_at(uint64_t key) {
  const uint64_t a = mix64(key ^ 0x8D5CF3D2A3B1E601ull);
  const uint64_t b = mix64(key ^ 0xC2B2AE3D27D4EB4Full);
  const double u1 = __dmul_rn(static_cast<double>((a >> 11) + 1), 0x1.0p-53);
  const double u2 = __dmul_rn(static_cast<double>(b >> 11), 0x1.0p-53);
  // 2.0 * pi * u2 evaluates left to right in the reference
  const double ang = __dmul_rn(2.0 * 3.141592653589793, u2);
  return __dmul_rn(sqrt(__dmul_rn(-2.0, log(u1))), cos(ang));
}

// One thread per (token, head, 8 consecutive d): 16 B (bf16) / 32 B (f32)
// stores.  out is [tokens, heads, d] with element strides ts / hs.
template <bool kBf16>
__global__ void random_batch_kernel(int64_t tokens, int heads, int d, uint64_t seed,
                                    uint64_t role, int h0, void* out, int64_t ts, int64_t hs) {
  const int dg = d / 8;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= tokens * heads * dg) return;
  const int g = static_cast<int>(i % dg);
  const int64_t th = i / dg;
  const int h = static_cast<int>(th % heads);
  const int64_t t = th / heads;
  const uint64_t base = mix64(mix64(mix64(seed) ^ role) ^ static_cast<uint64_t>(h0 + h));
  const uint64_t bt = mix64(mix64(base) ^ static_cast<uint64_t>(t));
  float v[8];
#pragma unroll
  for (int e = 0; e < 8; ++e)
    v[e] = __double2float_rn(gaussian_at(mix64(bt ^ static_cast<uint64_t>(g * 8 + e))));
  const int64_t off = t * ts + h * hs + g * 8;
  if constexpr (kBf16) {
    uint4 pk;
    pk.x = pack_bf16(v[0], v[1]);
    pk.y = pack_bf16(v[2], v[3]);
    pk.z = pack_bf16(v[4], v[5]);
    pk.w = pack_bf16(v[6], v[7]);
    *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(out) + off) = pk;
  } else {
    float4* o = reinterpret_cast<float4*>(static_cast<float*>(out) + off);
    o[0] = make_float4(v[0], v[1], v[2], v[3]);
    o[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
}

}  // namespace feat
}  // namespace rp
