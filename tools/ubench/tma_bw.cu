// Microbenchmark: achievable L2 -> SM TMA bandwidth on sm_100a with the K6
// access pattern (32 KB K/V tiles = two 64x128 bf16 boxes, 128B swizzle,
// one CTA per SM, an S-stage mbarrier ring, consumer releases at once).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2604_20470_b200/csrc \
//        -I../../include tma_bw.cu -o tma_bw -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
#include "common.cuh"
using namespace rp;

template <int S>
__global__ void __launch_bounds__(64, 1) k(const __grid_constant__ CUtensorMap tm, int n_tiles,
                                           int iters, long long* cyc) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + S * 32768);
  uint64_t* empty = full + S;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  const int warp = threadIdx.x / 32;
  long long t0 = clock64();
  if (warp == 0) {
    const uint64_t pol = policy_evict_last();
    for (int i = 0; i < iters; ++i) {
      const int st = i % S;
      mbar_wait(&empty[st], ((i / S) & 1) ^ 1);
      const int tile = static_cast<int>((static_cast<long long>(blockIdx.x) * 7919 + i * 104729ll) % n_tiles);
      mbar_arrive_expect_tx_w(&full[st], 32768);
      tma_load_3d_w(sm + st * 32768, &tm, &full[st], 0, 0, tile * 128, pol);
      tma_load_3d_w(sm + st * 32768 + 16384, &tm, &full[st], 64, 0, tile * 128, pol);
    }
  } else {
    for (int i = 0; i < iters; ++i) {
      const int st = i % S;
      mbar_wait(&full[st], (i / S) & 1);
      if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[st]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  const long long tokens_big = 8ll * 1024 * 1024;  // 2 GB of bf16 x 128
  void* buf;
  cudaMalloc(&buf, tokens_big * 128 * 2);
  cudaMemset(buf, 0, tokens_big * 128 * 2);
  long long* cyc;
  cudaMalloc(&cyc, 148 * 8);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  for (long long ws_mb : {16ll, 48ll, 96ll, 2048ll}) {
    const long long tokens = ws_mb * 1024 * 1024 / 256;
    CUtensorMap m;
    cuuint64_t dims[3] = {128, 1, static_cast<cuuint64_t>(tokens)};
    cuuint64_t strides[2] = {256, 256};
    cuuint32_t box[3] = {64, 1, 128};
    cuuint32_t es[3] = {1, 1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int n_tiles = static_cast<int>(tokens / 128);
    auto run = [&](auto kern, int S, int ctas_per_sm) {
      const int smem = S * 32768 + 1024 + 256;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      const int iters = 4000;
      const int grid = 148 * ctas_per_sm;
      kern<<<grid, 64, smem>>>(m, n_tiles, iters / 4, cyc);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      kern<<<grid, 64, smem>>>(m, n_tiles, iters, cyc);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      std::vector<long long> h(148);
      cudaMemcpy(h.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost);
      double mean = 0;
      for (auto x : h) mean += x;
      mean /= 148;
      const double bytes = double(grid) * iters * 32768;
      printf("ws %5lld MB stages %d ctas/SM %d: %.2f TB/s, %.1f B/clk/SM (%.0f clk per CTA, err=%s)\n",
             ws_mb, S, ctas_per_sm, bytes / (ms * 1e-3) / 1e12,
             double(iters) * 32768 * ctas_per_sm / mean, mean,
             cudaGetErrorString(cudaGetLastError()));
    };
    run(k<2>, 2, 1);
    run(k<4>, 4, 1);
    run(k<6>, 6, 1);
    run(k<3>, 3, 2);
  }
  return 0;
}
