// Instantiates the register-streaming kernel variants for u16 / gradient (split for parallel builds).
#include "morph_col.cuh"

namespace rmgpu {
namespace col {
cudaError_t dispatch_u16_grad(const MorphJob& j, int R) { return col_dispatch<uint16_t, MODE_GRAD>(j, R); }
}  // namespace col
}  // namespace rmgpu
