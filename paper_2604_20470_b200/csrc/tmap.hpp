// TMA tensor-map construction shared by the attention and scoring kernels.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <mutex>
#include <string>

#include "dynrad.h"
#include "internal.hpp"

namespace rp {

// ------------------------------------------------------------ tensor maps --
inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
  return fn;
}

// 3-D bf16 view {head_dim, heads, tokens} with a {64, 1, box_rows} box, 128B
// swizzle; rows >= tokens read as zero (the reference's zero padding).
inline CUtensorMap make_map_bf16(const rp_tensor& t, unsigned box_rows = 128) {
  CUtensorMap m;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(t.head_dim), static_cast<cuuint64_t>(t.heads),
                        static_cast<cuuint64_t>(t.tokens)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(t.head_stride) * 2,
                           static_cast<cuuint64_t>(t.token_stride) * 2};
  cuuint32_t box[3] = {64, 1, box_rows};
  cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, t.data, dims, strides,
                                 box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return m;
}


}  // namespace rp
