// Microbenchmark: formulations of the K6 per-row softmax body (128 values).
#include <cstdio>
#include "../../paper_2604_20470_b200/csrc/common.cuh"
using namespace rp;
__device__ __forceinline__ uint32_t ex2_bf16x2(uint32_t x) { uint32_t y; asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ uint32_t ex2_f16x2(uint32_t x) { uint32_t y; asm("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ uint32_t cvt_f16x2(float lo, float hi) { uint32_t d; asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo)); return d; }
template <int MODE, uint32_t PM>
__global__ void __launch_bounds__(256, 1) k(float* out, long long* cyc, int iters, float sl2) {
  uint32_t s[128];
  for (int i = 0; i < 128; ++i) s[i] = __float_as_uint((threadIdx.x * 7 + i * 13) % 97 * 0.01f);
  float m = 0.5f, l = 0.f;
  uint32_t sink = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float mq[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      float a = __uint_as_float(s[32 * c]);
#pragma unroll
      for (int i = 1; i < 31; i += 2) a = fmaxf(a, fmaxf(__uint_as_float(s[32 * c + i]), __uint_as_float(s[32 * c + i + 1])));
      mq[c] = fmaxf(a, __uint_as_float(s[32 * c + 31]));
    }
    m = fmaxf(m, fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3])));
    const float2 sc2 = make_float2(sl2, sl2), ng2 = make_float2(-m * sl2, -m * sl2);
    float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    if (MODE == 0) {  // fp32 MUFU (+ poly on PM pairs), two-phase
      float2 pv[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        const float2 xv = ffma2(make_float2(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])), sc2, ng2);
        if (PM & (1u << (i & 7))) pv[i] = ex2_poly2(xv); else { pv[i].x = ex2(xv.x); pv[i].y = ex2(xv.y); }
      }
#pragma unroll
      for (int i = 0; i < 64; ++i) { acc[i & 1] = fadd2(acc[i & 1], pv[i]); sink ^= pack_bf16(pv[i].x, pv[i].y); }
    } else if (MODE == 1) {  // bf16x2 MUFU: P comes out packed; sums from the bf16 values
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        const float2 xv = ffma2(make_float2(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])), sc2, ng2);
        const uint32_t p = ex2_bf16x2(pack_bf16(xv.x, xv.y));
        sink ^= p;
        acc[i & 1] = fadd2(acc[i & 1], make_float2(__uint_as_float(p << 16), __uint_as_float(p & 0xFFFF0000u)));
      }
    } else {  // f16x2 MUFU, then f16x2 -> f32 -> bf16x2
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        const float2 xv = ffma2(make_float2(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])), sc2, ng2);
        const uint32_t h = ex2_f16x2(cvt_f16x2(xv.x, xv.y));
        const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&h));
        sink ^= pack_bf16(f.x, f.y);
        acc[i & 1] = fadd2(acc[i & 1], f);
      }
    }
    l += acc[0].x + acc[1].x + acc[0].y + acc[1].y;
    s[it & 127] ^= 1;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = l + sink;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int MODE, uint32_t PM>
void run(const char* name, float* out, long long* cyc) {
  for (int w : {4, 8}) {
    cudaMemset(cyc, 0, 8);
    k<MODE, PM><<<148, 32 * w>>>(out, cyc, 200, 0.127f);
    cudaError_t e = cudaGetLastError(); cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-22s warps %d: %6.0f clk per row iteration per warp %s\n", name, w, double(h) / 200, e ? cudaGetErrorString(e) : "");
  }
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 256 * 4); cudaMalloc(&cyc, 148 * 8);
  run<0, 0x00>("f32 mufu", out, cyc);
  run<0, 0x01>("f32 poly 1/8", out, cyc);
  run<0, 0x11>("f32 poly 2/8", out, cyc);
  run<0, 0x25>("f32 poly 3/8", out, cyc);
  run<0, 0x55>("f32 poly 4/8", out, cyc);
  run<1, 0>("bf16x2 mufu", out, cyc);
  run<2, 0>("f16x2 mufu", out, cyc);
}
