// K5 and mask utilities: bit-packed block mask -> block-sparse row lists.
//
// The reference stops at the bitmask (mask.hpp:13-35: row-major, LSB-first,
// row_bytes = ceil(S_b/8)); the attention kernels walk per-row lists of
// active block columns, so this step is new.  Also expand_mask
// (mask.cpp:52-66) and the active-block count behind sparsity (mask.cpp:47).
#include "common.cuh"

namespace rp {
namespace csr {

// One warp per block row: popcount of its row_bytes bytes.
__global__ void row_count_kernel(const uint8_t* __restrict__ bits, int64_t n_rows,
                                 int64_t row_bytes, int32_t* __restrict__ counts) {
  const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (row >= n_rows) return;
  int c = 0;
  for (int64_t b = lane; b < row_bytes; b += 32) c += __popc(bits[row * row_bytes + b]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
  if (lane == 0) counts[row] = c;
}

// Single-CTA exclusive scan (S_b is at most a few tens of thousands).
__global__ void scan_kernel(const int32_t* __restrict__ counts, int64_t n,
                            int32_t* __restrict__ row_ptr, int64_t* nnz_out) {
  __shared__ int32_t warp_tot[32];
  __shared__ int32_t carry;
  const int t = threadIdx.x, lane = t % 32, w = t / 32;
  if (t == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < n; base += blockDim.x) {
    const int64_t i = base + t;
    const int32_t v = i < n ? counts[i] : 0;
    int32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (w == 0) {
      int32_t s = lane < (blockDim.x / 32) ? warp_tot[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xFFFFFFFFu, s, o);
        if (lane >= o) s += y;
      }
      warp_tot[lane] = s;  // inclusive over warps
    }
    __syncthreads();
    const int32_t before = carry + (w ? warp_tot[w - 1] : 0) + x - v;
    if (i < n) row_ptr[i] = before;
    __syncthreads();
    if (t == blockDim.x - 1) carry = before + v;
    __syncthreads();
  }
  if (t == 0) {
    row_ptr[n] = carry;
    if (nnz_out) *nnz_out = carry;
  }
}

// One warp per row: emit ascending active columns.
__global__ void fill_kernel(const uint8_t* __restrict__ bits, int64_t n_rows,
                            int64_t row_bytes, const int32_t* __restrict__ row_ptr,
                            int32_t* __restrict__ col_idx, int64_t col_cap) {
  const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (row >= n_rows) return;
  int32_t out = row_ptr[row];
  for (int64_t b0 = 0; b0 < row_bytes; b0 += 32) {
    const int64_t b = b0 + lane;
    const uint32_t byte = b < row_bytes ? bits[row * row_bytes + b] : 0u;
    const int c = __popc(byte);
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= o) x += y;
    }
    int pos = out + x - c;
    for (int k = 0; k < 8; ++k)
      if ((byte >> k) & 1u) {
        const int64_t col = b * 8 + k;
        if (col < n_rows && pos < col_cap) col_idx[pos] = static_cast<int32_t>(col);
        ++pos;
      }
    out += __shfl_sync(0xFFFFFFFFu, x, 31);
  }
}

// rows by descending nnz, ties by ascending row index (a rank computation;
// S_b^2 comparisons, trivial at S_b <= ~10^4).
__global__ void order_kernel(const int32_t* __restrict__ counts, int64_t n,
                             int32_t* __restrict__ order) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t ci = counts[i];
  int64_t rank = 0;
  for (int64_t j = 0; j < n; ++j) {
    const int32_t cj = counts[j];
    rank += (cj > ci) || (cj == ci && j < i);
  }
  order[rank] = static_cast<int32_t>(i);
}

// expand_mask: token row r, token byte tb -> bits of 8 token columns.
__global__ void expand_kernel(const uint8_t* __restrict__ bits, int64_t blocks,
                              int64_t row_bytes, int block, int64_t tokens,
                              int64_t token_row_bytes, uint8_t* __restrict__ out) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = tokens * token_row_bytes;
  if (idx >= total) return;
  const int64_t r = idx / token_row_bytes, tb = idx % token_row_bytes;
  const int64_t br = r / block;
  uint32_t byte = 0;
  for (int k = 0; k < 8; ++k) {
    const int64_t c = tb * 8 + k;
    if (c >= tokens) break;
    const int64_t bc = c / block;
    byte |= ((bits[br * row_bytes + bc / 8] >> (bc % 8)) & 1u) << k;
  }
  out[idx] = static_cast<uint8_t>(byte);
}

__global__ void popcount_kernel(const uint8_t* __restrict__ bits, int64_t n,
                                unsigned long long* out) {
  unsigned long long c = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    c += __popc(bits[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
  if (threadIdx.x % 32 == 0) atomicAdd(out, c);
}

// Dense row lists (every block of every row) for the soft-mask path:
// row_ptr[r] = r * n, col_idx[r * n + c] = c.
__global__ void dense_lists_kernel(int64_t n, int32_t* __restrict__ row_ptr,
                                   int32_t* __restrict__ col_idx) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i <= n) row_ptr[i] = static_cast<int32_t>(i * n);
  if (i < n * n) col_idx[i] = static_cast<int32_t>(i % n);
}

// B = 64 masks on the 128-row tensor-core kernel: the 64-block CSR rows
// (2R, 2R+1) merged into 128 x 128 tile row R (tile column C covers 64-block
// columns 2C, 2C+1) with the tile's quadrant bits (bit 2 * row_half +
// key_half).  One thread per tile row; the lists are sorted, c / 2 too.
template <bool FILL>
__global__ void quad_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                            int64_t nb, int64_t ns, int32_t* __restrict__ counts,
                            const int32_t* __restrict__ srow_ptr, int32_t* __restrict__ scol,
                            uint8_t* __restrict__ qmask) {
  const int64_t R = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (R >= ns) return;
  const int64_t a = 2 * R, b = 2 * R + 1;
  int i = static_cast<int>(row_ptr[a]), ie = static_cast<int>(row_ptr[a + 1]);
  int j = b < nb ? static_cast<int>(row_ptr[b]) : 0, je = b < nb ? static_cast<int>(row_ptr[b + 1]) : 0;
  int n = 0;
  int o = FILL ? srow_ptr[R] : 0;
  while (i < ie || j < je) {
    const int ca = i < ie ? col[i] >> 1 : 0x7FFFFFFF, cb = j < je ? col[j] >> 1 : 0x7FFFFFFF;
    const int C = ca < cb ? ca : cb;
    uint32_t q = 0;
    while (i < ie && (col[i] >> 1) == C) q |= 1u << (col[i++] & 1);
    while (j < je && (col[j] >> 1) == C) q |= 4u << (col[j++] & 1);
    if (FILL) {
      scol[o] = C;
      qmask[o] = static_cast<uint8_t>(q);
      ++o;
    }
    ++n;
  }
  if (!FILL) counts[R] = n;
}

// Flags a row without any active block (the reference's domain_error,
// attention.cpp:85-86) for kernels that zero-fill such rows silently.
__global__ void empty_row_flag_kernel(const int32_t* __restrict__ row_ptr, int64_t n,
                                      int* __restrict__ flag) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n && row_ptr[i + 1] == row_ptr[i]) atomicOr(flag, 1);
}

}  // namespace csr
}  // namespace rp
