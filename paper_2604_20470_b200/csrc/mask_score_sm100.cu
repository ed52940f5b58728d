// Tensor-core dynamic scoring engine (placeholder until the tcgen05 kernel lands).
#include <stdexcept>

#include "mask_build.cuh"

namespace rp {
namespace mask {
bool fast_engine_supported(const rp_grid&, int, int) { return false; }
void build_dynamic_fast(const FastArgs&, const Feat&) {
  throw std::invalid_argument("build_mask: tensor-core scoring engine not available");
}
}  // namespace mask
}  // namespace rp
