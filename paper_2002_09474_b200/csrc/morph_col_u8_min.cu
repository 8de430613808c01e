// Instantiates the register-streaming kernel variants for u8 / min (split for parallel builds).
#include "morph_col.cuh"

namespace rmgpu {
namespace col {
cudaError_t dispatch_u8_min(const MorphJob& j, int R) { return col_dispatch<uint8_t, MODE_MIN>(j, R); }
}  // namespace col
}  // namespace rmgpu
