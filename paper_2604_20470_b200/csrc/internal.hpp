// Internal plumbing shared by the C-ABI translation units: exception ->
// rp_status mapping (the reference's four exception types, mask.hpp /
// selection.cpp / attention.cpp), CUDA error checking, launch accounting.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <stdexcept>
#include <string>

#include "dynrad.h"

namespace rp {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void set_error(const std::string& msg);
extern std::atomic<long long> g_launches;

inline void count_launch(long long n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

#define RP_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      throw ::rp::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_));   \
  } while (0)

#define RP_LAUNCHED()                                                              \
  do {                                                                             \
    ::rp::count_launch();                                                          \
    cudaError_t e_ = cudaGetLastError();                                           \
    if (e_ != cudaSuccess)                                                         \
      throw ::rp::CudaError(std::string("kernel launch: ") + cudaGetErrorString(e_)); \
  } while (0)

template <class F>
rp_status guarded(F&& f) {
  try {
    f();
    return RP_OK;
  } catch (const CudaError& e) {
    set_error(e.what());
    return RP_CUDA_ERROR;
  } catch (const std::invalid_argument& e) {
    set_error(e.what());
    return RP_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) {
    set_error(e.what());
    return RP_OUT_OF_RANGE;
  } catch (const std::domain_error& e) {
    set_error(e.what());
    return RP_DOMAIN_ERROR;
  } catch (const std::exception& e) {
    set_error(e.what());
    return RP_RUNTIME_ERROR;
  }
}

// Opt a kernel into `smem` bytes of dynamic shared memory on the current
// device (a per-(kernel, device) attribute: set once per device), after
// running `check` (may be null) on it.
void prepare_kernel(const void* fn, int smem, void (*check)(const void*) = nullptr);

// Keep the stream-ordered pool's memory between calls on the current device
// (the default release threshold returns every byte at each synchronize, so
// the multi-GB scratch of a static mask build or a host-buffer layer would be
// re-mapped on every call).
void keep_pool_memory();

// Optional per-stage CUDA-event timing (rp_profile_stages): when enabled,
// library entry points bracket their kernels with events on the launching
// stream; bench.py reads the per-stage device time of the timed region.
enum Stage : int {
  kStageMaskPrep = 0,    // base-mask copy, norms, per-tile max |k|
  kStageScoreStats = 1,  // tensor-core scoring, pass 1 (per-pair mu / sigma)
  kStageJobStats = 2,    // per-frame-pair thresholds
  kStageScoreSelect = 3, // tensor-core scoring, pass 2 (keep / drop / undecided)
  kStageRecheck = 4,     // exact fp64 re-score of undecided pairs + fallback
  kStageApply = 5,       // theta_c / theta_m tile aggregation, mask copy-out
  kStageCsr = 6,         // bitmask -> row lists
  kStageAttention = 7,   // stage (d)
  kStageExactScore = 8,  // exact fp64 scoring engine (all of a10-a12)
  kStageStatic = 9,      // static Fisher-Yates build (first call of a plan)
  kNumStages = 10
};
bool profiling_on();
void stage_begin(int stage, cudaStream_t s);
void stage_end(int stage, cudaStream_t s);

// Every compute entry point first checks that a CUDA device exists: the
// product has no CPU fallback.
void require_device();

inline void check_grid(const rp_grid* g) {
  if (!g) throw std::invalid_argument("grid: null");
  if (g->n_frames < 1) throw std::invalid_argument("grid: n_frames must be >= 1");
  if (g->tokens_per_frame < 1)
    throw std::invalid_argument("grid: tokens_per_frame must be >= 1");
  if (g->block_size < 2 || (g->block_size & (g->block_size - 1)))
    throw std::invalid_argument("grid: block_size must be a power of two >= 2");
}

}  // namespace rp
