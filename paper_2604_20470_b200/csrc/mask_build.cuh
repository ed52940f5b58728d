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

struct FastArgs {
  const rp_tensor* q;
  const rp_tensor* k;
  int heads;
  const std::vector<DJob>& jobs;
  const DJob* d_jobs;
  const rp_grid& g;
  int cmin, amin, fallback_k;
  double delta;
  uint32_t* words;
  cudaStream_t s;
  int64_t* rechecked;
  int64_t* fallbacks;
  bool want_stats;
};

bool fast_engine_supported(const rp_grid& g, int head_dim, int heads);
void build_dynamic_fast(const FastArgs& a, const Feat& f);

}  // namespace mask
}  // namespace rp
