// Shared declarations of the mask builder (mask_build.cu) and its
// tensor-core scoring engine (mask_score_sm100.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "dynrad.h"

namespace rp {
namespace mask {

// Device copy of one frame-pair job (plan.hpp Job + tile geometry of the
// pair's TileCounts rectangle, mask.cpp:92-103).
struct DJob {
  int32_t i, j, kind;
  int32_t r0, c0, tr, tc;  // first block row/col and tile rows/cols
  int32_t pad;
  int64_t width, n, k;
  int64_t cnt_off;         // offset of this job's [tr][tc][B] counts
  double param;            // ratio or tau
  uint64_t seed;           // splitmix64 stream seed of the pair
};

struct Item {  // one (job, tile) of a job's rectangle
  int32_t job, tr, tc;
};



struct Feat;

// Tensor-core scoring engine (mask_score_sm100.cu).  Created once per plan
// (it caches the tile list and device buffers of the plan's scored pairs).
class FastEngine;
struct FastResult {
  int64_t rechecked = 0;   // pairs re-scored exactly in fp64
  int64_t fallbacks = 0;   // frame pairs that took the fallback_k rule
};
bool fast_engine_supported(const rp_grid& g, int head_dim, int heads);
FastEngine* fast_engine_create(const rp_grid& g, const std::vector<DJob>& jobs, int cmin,
                               int amin, int heads, int head_dim, cudaStream_t s);
void fast_engine_destroy(FastEngine* e);
// Adds the selected tiles of every scored frame pair to `words` (the padded
// 32-bit view of the bit-packed mask).
void fast_engine_run(FastEngine* e, const rp_tensor* q, const rp_tensor* k, const Feat& f,
                     uint32_t* words, cudaStream_t s, double delta_floor, int fallback_k,
                     bool want_stats, FastResult* res);

}  // namespace mask
}  // namespace rp
