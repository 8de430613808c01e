// Instantiates the phase kernel variants for u16 / min (split across files for parallel builds).
#include "morph_phase.cuh"

namespace rmgpu {
namespace phase {
cudaError_t dispatch_u16_min(const MorphJob& j, int vb, int hb, int rh, int B, int q, int pf) {
    return phase_dispatch<uint16_t, MODE_MIN>(j, vb, hb, rh, B, q, pf);
}
}  // namespace phase
}  // namespace rmgpu
