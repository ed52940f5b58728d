// Microbenchmark: MUFU throughput of ex2.approx.f32 vs ex2.approx.ftz.bf16x2
// and ex2.approx.f16x2 on sm_100a (results per clock per SM), plus the
// bf16x2 / f16x2 accuracy against exp2 in double.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
template <int MODE>
__global__ void k(uint32_t* out, long long* cyc, int iters) {
  uint32_t v[32];
  for (int i = 0; i < 32; ++i) v[i] = 0x3c003c00u ^ (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (MODE == 0) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(__uint_as_float(v[i]))); v[i] = __float_as_uint(y) & 0xBF7FFFFFu; }
      if (MODE == 1) { uint32_t y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(v[i])); v[i] = y & 0xBF7FBF7Fu; }
      if (MODE == 2) { uint32_t y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(v[i])); v[i] = y & 0xBBFFBBFFu; }
    }
  }
  long long t1 = clock64();
  __syncthreads();
  uint32_t s = 0; for (int i = 0; i < 32; ++i) s ^= v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void acc(float* xs, float* e_bf, float* e_h, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float x = xs[i];
  __nv_bfloat162 xb = __floats2bfloat162_rn(x, x);
  uint32_t yb; asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(yb) : "r"(*reinterpret_cast<uint32_t*>(&xb)));
  __half2 xh = __floats2half2_rn(x, x);
  uint32_t yh; asm("ex2.approx.f16x2 %0, %1;" : "=r"(yh) : "r"(*reinterpret_cast<uint32_t*>(&xh)));
  e_bf[i] = __bfloat162float(reinterpret_cast<__nv_bfloat162*>(&yb)->x);
  e_h[i] = __half2float(reinterpret_cast<__half2*>(&yh)->x);
}
int main() {
  uint32_t* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 1000;
  for (int mode = 0; mode < 3; ++mode)
    for (int warps : {8, 16}) {
      if (mode == 0) k<0><<<148, warps * 32>>>(out, cyc, iters);
      if (mode == 1) k<1><<<148, warps * 32>>>(out, cyc, iters);
      if (mode == 2) k<2><<<148, warps * 32>>>(out, cyc, iters);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      double results = (double)warps * 32 * iters * 32 * (mode ? 2 : 1);
      printf("%s warps %2d: %.1f exp2 results/clk/SM\n", mode == 0 ? "f32   " : mode == 1 ? "bf16x2" : "f16x2 ", warps, results / h);
    }
  const int n = 4096; float hx[n]; for (int i = 0; i < n; ++i) hx[i] = -20.0f * i / n;
  float *dx, *db, *dh; cudaMalloc(&dx, n * 4); cudaMalloc(&db, n * 4); cudaMalloc(&dh, n * 4);
  cudaMemcpy(dx, hx, n * 4, cudaMemcpyHostToDevice);
  acc<<<n / 256, 256>>>(dx, db, dh, n); cudaDeviceSynchronize();
  float hb[n], hh[n]; cudaMemcpy(hb, db, n * 4, cudaMemcpyDeviceToHost); cudaMemcpy(hh, dh, n * 4, cudaMemcpyDeviceToHost);
  double wb = 0, wh = 0, sw = 0, mb = 0, mh = 0;
  for (int i = 0; i < n; ++i) { double r = exp2((double)hx[i]); double eb = fabs(hb[i] - r) / r, eh = fabs(hh[i] - r) / r;
    if (hx[i] > -8) { mb = fmax(mb, eb); mh = fmax(mh, eh); } wb += r * eb; wh += r * eh; sw += r; }
  printf("rel err (x in [-8,0]): bf16x2 max %.4f, f16x2 max %.4f; weight-averaged: bf16x2 %.5f, f16x2 %.5f\n", mb, mh, wb / sw, wh / sw);
  return 0;
}
