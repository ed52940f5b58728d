// Microbenchmark: the K6 per-row softmax body (max, exp2, sum, bf16 pack) from
// registers, one warp per SMSP, to separate its own cost from pipeline effects.
#include <cstdio>
#include "../../paper_2604_20470_b200/csrc/common.cuh"
using namespace rp;
template <int MODE>
__global__ void __launch_bounds__(128, 1) k(float* out, long long* cyc, int iters, float sl2) {
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
    const float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
    m = fmaxf(m, mx);
    const float2 sc2 = make_float2(sl2, sl2), ng2 = make_float2(-m * sl2, -m * sl2);
    float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    if (MODE == 0) {  // two-phase: all exps, then sums/packs
      float2 pv[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        const float2 xv = ffma2(make_float2(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])), sc2, ng2);
        pv[i].x = ex2(xv.x); pv[i].y = ex2(xv.y);
      }
#pragma unroll
      for (int i = 0; i < 64; ++i) { acc[i & 1] = fadd2(acc[i & 1], pv[i]); sink ^= pack_bf16(pv[i].x, pv[i].y); }
    } else if (MODE == 1) {  // exps only
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        const float2 xv = ffma2(make_float2(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])), sc2, ng2);
        acc[i & 1].x += ex2(xv.x); acc[i & 1].y += ex2(xv.y);
      }
    } else {  // MUFU only, independent
#pragma unroll
      for (int i = 0; i < 128; ++i) acc[i & 1].x += ex2(__uint_as_float(s[i]));
    }
    l += acc[0].x + acc[1].x + acc[0].y + acc[1].y;
    s[it & 127] ^= 1;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = l + sink;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 256 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 200;
  for (int mode = 0; mode < 3; ++mode) for (int w : {4, 8}) {
    if (mode == 0) k<0><<<148, 32 * w>>>(out, cyc, iters, 0.127f);
    if (mode == 1) k<1><<<148, 32 * w>>>(out, cyc, iters, 0.127f);
    if (mode == 2) k<2><<<148, 32 * w>>>(out, cyc, iters, 0.127f);
    cudaError_t e = cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("mode %d warps %d: %.0f clk per row-tile iteration (%s)\n", mode, w, double(h) / iters, cudaGetErrorString(e));
  }
}
