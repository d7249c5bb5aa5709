// K5 tensor-core path (placeholder until the tcgen05 kernel lands).
#include "common.cuh"

namespace lvsk {
bool rowsumsq_tc_f32(const float*, int64_t, int64_t, int64_t, const float*, const float*, int64_t, double*, int32_t*,
                     cudaStream_t, int32_t*) {
  return false;
}
}  // namespace lvsk
