// Instantiates the register-streaming kernel variants for u8 / gradient (split for parallel builds).
#include "morph_col.cuh"

namespace rmgpu {
namespace col {
cudaError_t dispatch_u8_grad(const MorphJob& j, int R) { return col_dispatch<uint8_t, MODE_GRAD>(j, R); }
}  // namespace col
}  // namespace rmgpu
