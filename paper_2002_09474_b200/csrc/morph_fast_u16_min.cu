// Instantiates the fused kernel variants for u16 / min (split across files for parallel builds).
#include "morph_fast.cuh"

namespace rmgpu {
namespace fast {
cudaError_t dispatch_u16_min(const MorphJob& j, int vv, int hv) { return dispatch_v<uint16_t, MODE_MIN>(j, vv, hv); }
}  // namespace fast
}  // namespace rmgpu
