// Microbenchmark: MUFU.EX2 / F2FP / FFMA2 issue throughput per SMSP on sm_100a.
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
  float v[32];
  for (int i = 0; i < 32; ++i) v[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  unsigned acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (MODE == 0) v[i] = ex2(v[i]) - 1.0f;       // MUFU + FADD
      if (MODE == 1) { __nv_bfloat162 b = __floats2bfloat162_rn(v[i], v[(i + 1) & 31]); acc += *reinterpret_cast<unsigned*>(&b); v[i] += 1e-7f; }
      if (MODE == 2) v[i] = ex2(v[i]);               // MUFU only (chain per element)
    }
  }
  long long t1 = clock64();
  __syncthreads();
  float s = 0; for (int i = 0; i < 32; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 1000;
  for (int mode = 0; mode < 3; ++mode)
    for (int warps : {4, 8, 16}) {
      if (mode == 0) k<0><<<148, warps * 32>>>(out, cyc, iters);
      if (mode == 1) k<1><<<148, warps * 32>>>(out, cyc, iters);
      if (mode == 2) k<2><<<148, warps * 32>>>(out, cyc, iters);
      cudaDeviceSynchronize();
      long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      double per_warp_instr = double(h) / (iters * 32.0);  // clocks per (op per warp) per warp
      double lanes_per_clk_sm = (double)warps * 32 * iters * 32 / h;
      printf("mode %d (%s) warps %2d: %lld clk, %.2f clk per op-instr per warp, %.1f ops/clk/SM\n", mode,
             mode == 0 ? "ex2+fadd" : mode == 1 ? "f2fp.bf16x2+fadd" : "ex2 chain", warps, h, per_warp_instr, lanes_per_clk_sm);
    }
  return 0;
}
