// Instantiates the phase kernel variants for u8 / min (split across files for parallel builds).
#include "morph_phase.cuh"

namespace rmgpu {
namespace phase {
cudaError_t dispatch_u8_min(const MorphJob& j, int vb, int hb, int rh, int B, int q, int pf) {
    return phase_dispatch<uint8_t, MODE_MIN>(j, vb, hb, rh, B, q, pf);
}
}  // namespace phase
}  // namespace rmgpu
