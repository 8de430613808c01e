// morph_sep_h_u16_min.cu -- K3 horizontal-pass instantiations (u16, min); see morph_sep.cuh.
#include "morph_sep.cuh"

namespace rmgpu {
namespace sep {

cudaError_t launch_h_u16_min(const SepParams& p, int C, int bx, dim3 grid, cudaStream_t s) {
    switch (C * 100 + bx) {
#define RM_H(CC, BB)                                                  \
    case CC * 100 + BB:                                               \
        return launch_hk(hpass_kernel<uint16_t, MODE_MIN, CC, BB>, p, grid, s);
        RM_H(8, 0) RM_H(8, 1) RM_H(8, 2) RM_H(8, 3) RM_H(8, 4) RM_H(8, 5) RM_H(8, 6) RM_H(8, 7)
#undef RM_H
    }
    return cudaErrorInvalidValue;
}

// two horizontal passes (this mode, then the other) in one sweep: opening / closing
cudaError_t launch_hh_u16_min(const SepParams& p, int C, int bx, dim3 grid, cudaStream_t s) {
    switch (C * 100 + bx) {
#define RM_H(CC, BB)                                                  \
    case CC * 100 + BB:                                               \
        return launch_hk(hpass_kernel<uint16_t, MODE_MIN, CC, BB, 2>, p, grid, s);
        RM_H(8, 0) RM_H(8, 1) RM_H(8, 2) RM_H(8, 3) RM_H(8, 4) RM_H(8, 5) RM_H(8, 6) RM_H(8, 7)
#undef RM_H
    }
    return cudaErrorInvalidValue;
}

}  // namespace sep
}  // namespace rmgpu
